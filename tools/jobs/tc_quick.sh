cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/vox_c2.py --check
timeout 120 python tools/vox_c2.py --config c4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_fwd_tc" -c 1 -o gpurun_out/tc_full python tools/vox_c2.py --reps 1 > gpurun_out/ncu_tc.log 2>&1; echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/tc_full.ncu-rep 2>&1 | tail -3
python tools/ncu_hotspots.py gpurun_out/tc_full.ncu-rep k_fvr_fwd_tc 30 2>&1 | awk 'NR%2==1' | head -16
