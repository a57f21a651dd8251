cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/vox_c2.py --check
timeout 120 python tools/vox_c2.py --config c4
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_c2_parity.py tests/test_gpu_poison.py -m gpu -q --timeout 600 -p no:cacheprovider 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_bwd" -c 1 -o gpurun_out/bwd_full python tools/vox_c2.py --reps 1 > gpurun_out/ncu_bwd.log 2>&1; echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/bwd_full.ncu-rep 2>&1 | tail -3
python tools/ncu_lines.py gpurun_out/bwd_full.ncu-rep k_fvr_bwd 12
