# Voxelizer forward: parity / poison / occupancy tests, graph timeline, bench loss.
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "splat or fvr or forward or c2 or occupancy or poison or trainer or coverage" 2>&1 | tail -1
timeout -s KILL 300 python tools/graph_timeline.py 2>&1 | grep -E "k_fvr_fwd|span" | tail -2
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --extra "" 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['last_loss'], d['stages_ms']['fvr_forward'])"
