cd $GRAFT_REPO_ROOT
L=paper_2411_04844_b200/_lib
cp $L/libsplatct.so $L/libsplatct_base.so
for v in base ch1 ch2 ch2c20; do
  cp $L/libsplatct_$v.so $L/libsplatct.so; touch $L/libsplatct.so
  echo "== $v"
  SPLATCT_BWD_KERNEL=ts2 timeout -s KILL 120 python tools/vox_c2.py | cut -c1-120
  SPLATCT_BWD_KERNEL=ts2 timeout -s KILL 120 python tools/vox_c2.py --config c4 | cut -c1-120
done
