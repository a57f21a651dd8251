# pytest selection ($PYF / $PYK) + one default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest ${PYF:-tests} -m gpu -q --timeout 900 -p no:cacheprovider ${PYK:+-k "$PYK"} -rA > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_new.log | tail -20
timeout 900 python bench.py ${BENCH_ARGS:---steps 30 --warmup 5} > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log | cut -c1-3000
