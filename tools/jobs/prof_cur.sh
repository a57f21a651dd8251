cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fvr_bwd|k_ssim_stats11|k_loss_grad11|k_fvr_fwd" -c 4 -o gpurun_out/cur_full python tools/prof_step.py --iters 1 > gpurun_out/ncu_cur.log 2>&1; echo "ncu rc=$?"
python tools/ncu_full_summary.py gpurun_out/cur_full.ncu-rep 2>&1 | tail -12
for k in k_fvr_bwd k_ssim_stats11 k_loss_grad11; do python tools/ncu_lines.py gpurun_out/cur_full.ncu-rep $k 14; done
