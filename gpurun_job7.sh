cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/prof_step.py --iters 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python tools/prof_step.py --iters 2 > gpurun_out/ncu_launch.log 2>&1
echo "done rc=$?"
