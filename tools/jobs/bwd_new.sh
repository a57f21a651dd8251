# new backward: parity subset + C2 voxelizer timings of the variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_c2_parity.py tests/test_gpu_fullsize.py -m gpu -q --timeout 900 -p no:cacheprovider -rA > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_new.log | tail -20
timeout 300 python tools/vox_c2.py --check
SPLATCT_BWD_KERNEL=warp timeout 300 python tools/vox_c2.py
SPLATCT_BWD_KERNEL=warp SPLATCT_BWD_NO_TMA=1 timeout 300 python tools/vox_c2.py
timeout 300 python tools/vox_c2.py --config c4
SPLATCT_BWD_KERNEL=warp timeout 300 python tools/vox_c2.py --config c4
