cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "ssim_value or nonfinite" -p no:cacheprovider > gpurun_out/pytest_fix.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fix.log
timeout 600 python tools/prof_step.py --iters 3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python tools/prof_step.py --iters 3 > gpurun_out/ncu_launch.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_ssim_stats|k_loss_grad|k_csr_spmm|k_fvr_bwd|k_fvr_fwd" -s 0 -c 7 -o gpurun_out/prof_r1 python tools/prof_step.py --iters 1 > gpurun_out/ncu_full.log 2>&1
echo "done rc=$?"; tail -2 gpurun_out/pytest_fix.log; tail -3 gpurun_out/ncu_full.log
