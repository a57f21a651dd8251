cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {
  echo "== $*"
  env "$@" timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --extra "" > gpurun_out/band.log 2>&1
  grep '^{' gpurun_out/band.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['stages_ms']['proj_forward'], d.get('last_loss'), d['kernels']['proj_forward']['binding'].get('gathered_bytes'))
"
}
run SPLATCT_FWD_GROUPS=4
run SPLATCT_FWD_GROUPS=band8
run SPLATCT_FWD_GROUPS=band8 SPLATCT_BAND_V2=1
