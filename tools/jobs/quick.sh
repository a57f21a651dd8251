# Quick check: a pytest subset ($PYK) + one bench line (no CPU baseline).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider ${PYK:+-k "$PYK"} > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
tail -2 gpurun_out/pytest_quick.log
tail -2 gpurun_out/bench.log | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print('value',d['value'],'e2e',d['e2e']['value'] if d.get('e2e') else None); print(d['stages_ms'])"
