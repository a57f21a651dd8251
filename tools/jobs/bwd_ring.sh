# backward TMA ring-depth sweep: rebuild with BT_RING = 4, 5, 6
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2411_04844_b200/csrc/fvr.cu /tmp/fvr_orig.cu
for mb in 4 5 6; do
  sed "s/constexpr int BT_RING = 4;/constexpr int BT_RING = $mb;/" /tmp/fvr_orig.cu > paper_2411_04844_b200/csrc/fvr.cu
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo "build fail $mb"
  timeout 600 python tools/voxel_sweep.py --grids 256,512,1024 --ns 400000,2000000 > gpurun_out/sweep_ring$mb.jsonl 2>&1
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ring$mb.log 2>&1
done
cp /tmp/fvr_orig.cu paper_2411_04844_b200/csrc/fvr.cu
python - <<'PY'
import json
for mb in (4,5,6):
    print("RING", mb)
    for l in open(f"gpurun_out/sweep_ring{mb}.jsonl"):
        try: d=json.loads(l)
        except Exception: continue
        print({k:d[k] for k in d if k in ("grid","n","bwd_ms")})
    for l in open(f"gpurun_out/bench_ring{mb}.log"):
        try: d=json.loads(l); print("bench", d["value"], d["stages_ms"]["fvr_backward"])
        except Exception: pass
PY
