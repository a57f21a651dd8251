cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/prof_step.py --iters 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_fwd|k_fvr_bwd" -s 1 -c 2 -o gpurun_out/prof_r6 python tools/prof_step.py --iters 1 > gpurun_out/ncu_full6.log 2>&1
echo "done rc=$?"
