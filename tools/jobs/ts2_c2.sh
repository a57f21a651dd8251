# ts2 vs warp backward at C2 (stage times from bench's eager profile), unit sizes 4 / 2 / 1 tiles.
cd $GRAFT_REPO_ROOT
L=paper_2411_04844_b200/_lib
cp $L/libsplatct.so /tmp/base.so
run() { timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --extra "" 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$1', d['value'], d['stages_ms']['fvr_backward'])"; }
run warp
SPLATCT_BWD_KERNEL=ts2 run ts2_ch4
for v in ch2 ch1; do cp $L/libsplatct_$v.so $L/libsplatct.so; SPLATCT_BWD_KERNEL=ts2 run ts2_$v; done
cp /tmp/base.so $L/libsplatct.so
