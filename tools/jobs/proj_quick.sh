cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -q --timeout 600 -p no:cacheprovider -k "proj or occupancy or trainer" 2>&1 | tail -2
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --extra "" > gpurun_out/ro.log 2>&1
grep '^{' gpurun_out/ro.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms'], d.get('last_loss'))
" || tail -5 gpurun_out/ro.log
