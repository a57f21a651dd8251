# Radix pass keys per thread (SORT_IPT 16 / 8 / 4): bins stage in the graph timeline + bin tests.
cd $GRAFT_REPO_ROOT
L=paper_2411_04844_b200/_lib
cp $L/libsplatct.so /tmp/base.so
for v in base ipt8 ipt4; do
  [ $v != base ] && cp $L/libsplatct_$v.so $L/libsplatct.so
  echo "== $v"
  timeout -s KILL 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bin or row_ordered" 2>&1 | tail -1
  timeout -s KILL 300 python tools/graph_timeline.py 2>&1 | grep -E "k_onesweep|span" | tail -3
  cp /tmp/base.so $L/libsplatct.so
done
