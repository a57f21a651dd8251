cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log; cat gpurun_out/e2e_probe.log | grep -v Warn
