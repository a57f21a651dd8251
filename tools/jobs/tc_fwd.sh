# tensor-core forward: check + timings + ncu, then the voxelizer-related tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/vox_c2.py --check
SPLATCT_FWD_KERNEL=mma timeout 120 python tools/vox_c2.py
timeout 120 python tools/vox_c2.py --config c4
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_c2_parity.py tests/test_gpu_tc.py -m gpu -q --timeout 600 -p no:cacheprovider -rA -x > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
grep -E "^(FAILED|ERROR)|passed|failed|^E  " gpurun_out/pytest_new.log | head -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_fwd_tc" -c 1 -o gpurun_out/tc_full python tools/vox_c2.py --reps 1 > gpurun_out/ncu_tc.log 2>&1; echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/tc_full.ncu-rep 2>&1 | tail -3
SPLATCT_FWD_KERNEL=mma timeout 600 python -m pytest tests/test_gpu_c2_parity.py -m gpu -q -k pins -p no:cacheprovider 2>&1 | grep -E "^E  |passed|failed" | head -6
