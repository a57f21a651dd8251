# Non-temporal staging copy: A/B of the sinogram staging and the e2e call.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for nt in 0 1; do
  echo "== SPLATCT_STAGE_NT=$nt"
  SPLATCT_STAGE_NT=$nt timeout -s KILL 300 python tools/stage_probe.py 2>&1 | tail -4
  SPLATCT_STAGE_NT=$nt timeout -s KILL 300 python tools/e2e_phases.py 2>&1 | tail -6
done > gpurun_out/stage_nt.log 2>&1
timeout -s KILL 600 python -m pytest tests -q -m gpu -k "e2e or run_reconstruction or optim or dropin" -p no:cacheprovider > gpurun_out/stage_nt_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/stage_nt_pytest.log
cat gpurun_out/stage_nt.log; tail -n 2 gpurun_out/stage_nt_pytest.log
