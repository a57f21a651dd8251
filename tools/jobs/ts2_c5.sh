cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 900 python tools/voxel_sweep.py > gpurun_out/c5_warp.jsonl 2>&1; echo "warp rc=$?"
SPLATCT_BWD_KERNEL=ts2 timeout -s KILL 900 python tools/voxel_sweep.py > gpurun_out/c5_ts2.jsonl 2>&1; echo "ts2 rc=$?"
