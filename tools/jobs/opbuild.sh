# Operator build: segmented march + hash count (tests, cold probe, launch list of the build).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_edges.py -q -k "march_segments or block_build or band or projector" -p no:cacheprovider > gpurun_out/opb_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/opb_pytest.log
timeout -s KILL 900 python -m pytest tests -m gpu -q -k "proj or cone or parity or golden" -p no:cacheprovider > gpurun_out/opb_pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/opb_pytest2.log
timeout -s KILL 300 python tools/cold_probe.py > gpurun_out/opb_cold.log 2>&1
cat > /tmp/opb.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2411_04844_b200 import device as D
cfg = bench.CONFIGS["c2"]
truth, geom, box, cloud = bench.make_problem(cfg)
D.projector_for(geom, 256, 256, 0.5, torch.device("cuda", 0))
torch.cuda.synchronize()
PY
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/opb_launches.csv python /tmp/opb.py > gpurun_out/opb_ncu.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/opb_launches.csv > gpurun_out/opb_launches.txt 2>&1
tail -n 3 gpurun_out/opb_pytest.log gpurun_out/opb_pytest2.log; cat gpurun_out/opb_cold.log; head -14 gpurun_out/opb_launches.txt
