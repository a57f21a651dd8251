# Per-launch ncu list (time + DRAM bytes) of eager C2 iterations, after a plain run exits 0.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-launches}
timeout 600 python tools/prof_step.py --iters 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_bytes.sum,l1tex__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/$TAG.csv python tools/prof_step.py --iters 2 > gpurun_out/ncu_launch.log 2>&1
echo "rc=$?"
