# Cone check: tests + c2cone bench (stage times)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "cone or sharded" > gpurun_out/pytest_cone.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cone.log
tail -3 gpurun_out/pytest_cone.log
timeout 900 python bench.py --config c2cone --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cone.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cone.log
tail -2 gpurun_out/bench_cone.log | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print('value',d['value']); print(d['stages_ms'])"
if [ -n "$AB" ]; then
SPLATCT_CONE_ADJ=1 timeout 900 python bench.py --config c2cone --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cone_b.log 2>&1
tail -1 gpurun_out/bench_cone_b.log | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('B value',d['value']); print(d['stages_ms'])"
fi
