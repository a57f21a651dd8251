cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_c2_parity.py tests/test_gpu_poison.py -m gpu -q --timeout 600 -p no:cacheprovider -k "proj or occupancy or trainer or c2 or poison or skip" 2>&1 | tail -2
timeout -s KILL 300 python tools/graph_timeline.py 2>&1 | grep -E "k_bspmm|span" | tail -3
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --extra "" 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['last_loss'], d['stages_ms'], d['e2e']['value'], d['e2e']['cold']['value'])"
