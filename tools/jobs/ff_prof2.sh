# FFMA forward v2 + ordered backward: check, timings, ncu captures
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/vox_c2.py --check
SPLATCT_BWD_KERNEL=sp timeout 300 python tools/vox_c2.py
timeout 300 python tools/vox_c2.py --config c4
SPLATCT_FWD_KERNEL=mma timeout 300 python tools/vox_c2.py --config c4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_fwd_ff" -c 1 -o gpurun_out/ff2_full python tools/vox_c2.py --reps 1 > gpurun_out/ncu_ff.log 2>&1; echo "ncu rc=$?"
SPLATCT_BWD_KERNEL=sp timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_bwd_sp" -c 1 -o gpurun_out/bsp_full python tools/vox_c2.py --reps 1 > gpurun_out/ncu_bsp.log 2>&1; echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/ff2_full.ncu-rep 2>&1 | tail -3
python tools/ncu_full_summary.py gpurun_out/bsp_full.ncu-rep 2>&1 | tail -3
