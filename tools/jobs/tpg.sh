# Forward table builders per Gaussian (FWD_TPG 8 = 32-Gaussian batches, 4 = 64): parity + timeline.
cd $GRAFT_REPO_ROOT
L=paper_2411_04844_b200/_lib
cp $L/libsplatct.so /tmp/base.so
for v in base tpg4 tpg2; do
  [ $v != base ] && cp $L/libsplatct_$v.so $L/libsplatct.so
  echo "== $v"
  timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_c2_parity.py -q -p no:cacheprovider -k "splat or fvr or forward or c2 or flat or clipped or box" 2>&1 | tail -1
  timeout -s KILL 300 python tools/graph_timeline.py 2>&1 | grep -E "k_fvr_fwd|span" | tail -2
  cp /tmp/base.so $L/libsplatct.so
done
