# One `ncu --set full` capture of the kernels matching $KREGEX (count $COUNT) after a plain run exits 0.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-full}
timeout 600 python tools/prof_step.py --iters 1 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_bspmm}" -s ${SKIP:-0} -c ${COUNT:-1} -o gpurun_out/$TAG python tools/prof_step.py --iters 1 > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?"
