cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
KREGEX="k_ssim_stats11|k_loss_grad11" SKIP=1 COUNT=2 TAG=loss_full bash tools/jobs/ncu_full.sh
python tools/ncu_full_summary.py gpurun_out/loss_full.ncu-rep 2>&1 | tail -12
python tools/ncu_lines.py gpurun_out/loss_full.ncu-rep "k_ssim_stats11" 30
python tools/ncu_lines.py gpurun_out/loss_full.ncu-rep k_loss_grad11 30
