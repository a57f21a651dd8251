cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_fullsize.py tests/test_gpu_c2_parity.py tests/test_gpu_sharded.py -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -5
timeout -s KILL 120 python tools/vox_c2.py | cut -c1-120
timeout -s KILL 120 python tools/vox_c2.py --config c4 | cut -c1-120
