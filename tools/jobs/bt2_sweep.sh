cd $GRAFT_REPO_ROOT
L=paper_2411_04844_b200/_lib
cp $L/libsplatct.so $L/libsplatct_base.so
for v in base bt4_2 bt3_2 bt2_4; do
  cp $L/libsplatct_$v.so $L/libsplatct.so 2>/dev/null || cp $L/libsplatct_base.so $L/libsplatct.so
  touch $L/libsplatct.so
  echo "== $v"; timeout 120 python tools/vox_c2.py --check | cut -c1-200; timeout 120 python tools/vox_c2.py --config c4 | cut -c1-120
done
