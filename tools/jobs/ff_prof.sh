# FFMA forward + ordered backward: checks, timings, one ncu --set full capture each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/vox_c2.py --check
SPLATCT_FWD_KERNEL=mma timeout 300 python tools/vox_c2.py
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q --timeout 900 -p no:cacheprovider -rA > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_new.log | tail -20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_bwd_sp|k_fvr_fwd_ff" -c 2 -o gpurun_out/ff_full python tools/vox_c2.py --reps 1 > gpurun_out/ncu_ff.log 2>&1; echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/ff_full.ncu-rep 2>&1 | tail -12
