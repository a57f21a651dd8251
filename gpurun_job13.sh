cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/prof_step.py --iters 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_bwd" -s 0 -c 1 -o gpurun_out/prof_r7 python tools/prof_step.py --iters 1 > gpurun_out/ncu_full7.log 2>&1
echo "done rc=$?"
