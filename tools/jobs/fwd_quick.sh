cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 120 python tools/vox_c2.py --check | cut -c100-330
timeout -s KILL 120 python tools/vox_c2.py --config c4 | cut -c1-120
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --extra "" > gpurun_out/ro.log 2>&1
grep '^{' gpurun_out/ro.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms'], d.get('last_loss'))
" || tail -5 gpurun_out/ro.log
