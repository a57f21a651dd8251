# GPU parity tests + default bench line (+ optional voxel sweep when SWEEP=1).
# usage: gpurun --timeout 2400 -- 'bash tools/jobs/tests_bench.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 30 --warmup 5} > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
if [ "${SWEEP:-0}" = 1 ]; then
  timeout 1200 python tools/voxel_sweep.py > gpurun_out/voxel_sweep.jsonl 2> gpurun_out/voxel_sweep.err; echo "sweep rc=$?"
fi
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; tail -2 gpurun_out/bench.log
