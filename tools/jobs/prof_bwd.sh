cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_bwd" -c 1 -o gpurun_out/bwd_full python tools/vox_c2.py --reps 1 > gpurun_out/ncu_bwd.log 2>&1; echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/bwd_full.ncu-rep 2>&1 | tail -3
python tools/ncu_lines.py gpurun_out/bwd_full.ncu-rep k_fvr_bwd 30
