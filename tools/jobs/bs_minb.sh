# Projector CTAs per SM (BS_MINB) with the longest-first forward order: graph timeline.
cd $GRAFT_REPO_ROOT
L=paper_2411_04844_b200/_lib
cp $L/libsplatct.so /tmp/base.so
for v in base m5 m7 m8; do
  [ $v != base ] && cp $L/libsplatct_$v.so $L/libsplatct.so
  echo "== $v"; timeout -s KILL 300 python tools/graph_timeline.py 2>&1 | grep -E "k_bspmm|span" | tail -3
  cp /tmp/base.so $L/libsplatct.so
done
