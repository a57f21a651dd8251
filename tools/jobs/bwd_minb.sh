# backward min-blocks sweep: rebuild with FAST min CTAs per SM = 6, 7, 8
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2411_04844_b200/csrc/fvr.cu /tmp/fvr_orig.cu
for mb in 6 7 8; do
  sed "s/__launch_bounds__(32 \* BG_WARPS, FAST ? 6 : 4)/__launch_bounds__(32 * BG_WARPS, FAST ? $mb : 4)/" /tmp/fvr_orig.cu > paper_2411_04844_b200/csrc/fvr.cu
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo "build fail $mb"
  timeout 600 python tools/voxel_sweep.py --grids 256,512,1024 --ns 400000,2000000 > gpurun_out/sweep_mb$mb.jsonl 2>&1
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_mb$mb.log 2>&1
done
cp /tmp/fvr_orig.cu paper_2411_04844_b200/csrc/fvr.cu
python - <<'PY'
import json
for mb in (6,7,8):
    print("MINB", mb)
    for l in open(f"gpurun_out/sweep_mb{mb}.jsonl"):
        try: d=json.loads(l)
        except Exception: continue
        print({k:d[k] for k in d if k in ("grid","n","bwd_ms")})
    for l in open(f"gpurun_out/bench_mb{mb}.log"):
        try: d=json.loads(l); print("bench", d["value"], d["stages_ms"]["fvr_backward"])
        except Exception: pass
PY
