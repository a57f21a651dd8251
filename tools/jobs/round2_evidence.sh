# Round-2 evidence: full GPU tests, smoke, default bench (+ reference arm),
# ncu launch list and --set full captures of the step's kernels, C5 sweep.
# usage: gpurun --timeout 3600 -- 'R=r2 bash tools/jobs/round2_evidence.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R=${R:-r2}
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${R}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${R}_pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${R}_smoke.log
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${R}_bench.log
timeout -s KILL 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${R}_bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${R}_bench_ref.log
timeout -s KILL 600 python tools/prof_step.py --iters 2 > gpurun_out/prof_plain.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_bytes.sum,l1tex__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python tools/prof_step.py --iters 2 > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
timeout -s KILL 1800 ncu --set full --clock-control none --import-source on -k regex:"k_bspmm|k_ssim_stats11|k_loss_grad11|k_fvr_fwd|k_fvr_bwd|k_onesweep|k_bin_emit" -c 12 -o gpurun_out/${R}_full python tools/prof_step.py --iters 1 > gpurun_out/ncu_${R}_full.log 2>&1
echo "full rc=$?"
python tools/ncu_full_summary.py gpurun_out/${R}_full.ncu-rep > gpurun_out/${R}_full_summary.txt 2>&1
python tools/ncu_launch_summary.py gpurun_out/${R}_launches.csv > gpurun_out/${R}_launches.txt 2>&1
python tools/ncu_traffic.py gpurun_out/${R}_launches.csv > gpurun_out/${R}_traffic.json 2>&1
timeout -s KILL 1200 python tools/voxel_sweep.py > gpurun_out/${R}_voxel_sweep.jsonl 2> gpurun_out/voxel_sweep.err; echo "sweep rc=$?"
tail -2 gpurun_out/${R}_pytest_gpu.log; tail -1 gpurun_out/${R}_smoke.log; tail -c 800 gpurun_out/${R}_bench.log; tail -c 400 gpurun_out/${R}_bench_ref.log
