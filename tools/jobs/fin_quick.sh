cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --extra "" > gpurun_out/ro.log 2>&1
grep '^{' gpurun_out/ro.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms'], d.get('last_loss'), d['gpu_launches'])
" || tail -5 gpurun_out/ro.log
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -3
