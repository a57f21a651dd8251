# Longest-first CTA order of the blocked forward: tests, timeline, bench.
cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "cta_order or proj or c2 or trainer or occupancy or poison or dropin" 2>&1 | tail -2
timeout -s KILL 300 python tools/graph_timeline.py 2>&1 | grep -E "k_bspmm|span" | tail -3
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['last_loss'], d['stages_ms'], d['configs']['c4']['value'], d['configs']['c2cone']['value'], d['e2e']['value'], d['e2e']['cold']['value'])"
