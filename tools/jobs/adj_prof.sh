cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
KREGEX="k_bspmm" SKIP=2 COUNT=1 TAG=adj_full bash tools/jobs/ncu_full.sh
python tools/ncu_full_summary.py gpurun_out/adj_full.ncu-rep 2>&1 | tail -3
python tools/ncu_lines.py gpurun_out/adj_full.ncu-rep k_bspmm 36
