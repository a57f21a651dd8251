cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
KREGEX="k_bin_emit|k_onesweep|k_tile_starts" SKIP=4 COUNT=4 TAG=bins_full bash tools/jobs/ncu_full.sh
python tools/ncu_full_summary.py gpurun_out/bins_full.ncu-rep 2>&1 | tail -12
python tools/ncu_lines.py gpurun_out/bins_full.ncu-rep k_bin_emit 14
python tools/ncu_lines.py gpurun_out/bins_full.ncu-rep k_onesweep 14
