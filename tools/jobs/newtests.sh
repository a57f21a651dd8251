# Run a pytest selection ($PYK / $PYF) on the GPU box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest ${PYF:-tests} -m gpu -q --timeout 900 -p no:cacheprovider ${PYK:+-k "$PYK"} -rA > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
grep -E "^(PASSED|FAILED|ERROR)|passed|failed" gpurun_out/pytest_new.log | tail -40
