# Voxelizer forward CTAs per SM (FWD_MINB 4 / 3 / 5), persistent grid sized to match.
cd $GRAFT_REPO_ROOT
L=paper_2411_04844_b200/_lib
cp $L/libsplatct.so /tmp/base.so
for v in base fm3 fm5; do
  [ $v != base ] && cp $L/libsplatct_$v.so $L/libsplatct.so
  echo "== $v"
  timeout -s KILL 300 python -m pytest tests -m gpu -q -p no:cacheprovider -k "splat and c2" 2>&1 | tail -1
  timeout -s KILL 300 python tools/graph_timeline.py 2>&1 | grep -E "k_fvr_fwd|span" | tail -2
  cp /tmp/base.so $L/libsplatct.so
done
