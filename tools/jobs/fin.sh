# Finalize blocks (FIN_BLOCKS_N 32 / 16 / 8; more would outgrow the 97-double scratch): graph timeline.
cd $GRAFT_REPO_ROOT
L=paper_2411_04844_b200/_lib
cp $L/libsplatct.so /tmp/base.so
for v in base fin16 fin8; do
  [ $v != base ] && cp $L/libsplatct_$v.so $L/libsplatct.so
  echo "== $v"
  timeout -s KILL 300 python -m pytest tests -m gpu -q -p no:cacheprovider -k "finalize or trainer_step or c2_four" 2>&1 | tail -1
  timeout -s KILL 300 python tools/graph_timeline.py 2>&1 | grep -E "k_iter_finalize|span" | tail -2
  cp /tmp/base.so $L/libsplatct.so
done
