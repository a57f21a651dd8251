# ncu --set full of the cone projector pair at C2-cone size (after a plain run exits 0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_cone.py --reps 1 > gpurun_out/prof_cone.log 2>&1 || { echo "plain run failed"; tail gpurun_out/prof_cone.log; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cone_(fwd|adj)" -c 2 -o gpurun_out/${TAG:-cone} python tools/prof_cone.py --reps 1 > gpurun_out/ncu_${TAG:-cone}.log 2>&1
echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/${TAG:-cone}.ncu-rep 2>&1 | head -20
