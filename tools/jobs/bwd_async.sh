cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 120 python tools/vox_c2.py
SPLATCT_BWD_KERNEL=ts2 timeout -s KILL 120 python tools/vox_c2.py --check
timeout -s KILL 120 python tools/vox_c2.py --config c4
SPLATCT_BWD_KERNEL=ts2 timeout -s KILL 120 python tools/vox_c2.py --config c4
timeout -s KILL 600 python -m pytest tests/test_gpu_edges.py -m gpu -q --timeout 300 -p no:cacheprovider -k "variants or outside" 2>&1 | tail -3
SPLATCT_BWD_KERNEL=ts2 timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_bwd_ts2" -c 1 -o gpurun_out/bts2_full python tools/vox_c2.py --reps 1 > gpurun_out/ncu_bts2.log 2>&1; echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/bts2_full.ncu-rep 2>&1 | tail -3
python tools/ncu_lines.py gpurun_out/bts2_full.ncu-rep k_fvr_bwd_ts2 16
