cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -k "fvr or spec or edges or parity or fullsize or trainer" > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log
tail -2 gpurun_out/pytest_q.log
timeout 600 python tools/voxel_sweep.py --grids 256,512,1024 --ns 400000,2000000 > gpurun_out/sweep_q.jsonl 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
python - <<'PY'
import json
for l in open("gpurun_out/sweep_q.jsonl"):
    try: d=json.loads(l)
    except Exception: continue
    print({k:d[k] for k in d if k in ("grid","n","fwd_ms","bwd_ms")})
for l in open("gpurun_out/bench_q.log"):
    try: d=json.loads(l); print("bench", d["value"], d["stages_ms"])
    except Exception: pass
PY
