cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export SPLATCT_FWD_GROUPS=band8
KREGEX="k_bspmm_band" COUNT=1 TAG=band_full bash tools/jobs/ncu_full.sh
python tools/ncu_full_summary.py gpurun_out/band_full.ncu-rep 2>&1 | tail -3
python tools/ncu_lines.py gpurun_out/band_full.ncu-rep k_bspmm_band 20
