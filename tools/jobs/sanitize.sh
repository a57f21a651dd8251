# compute-sanitizer over smoke() and 2 eager C1 iterations of the training step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OUT=gpurun_out/sanitizer_r02.txt
: > $OUT
for tool in memcheck racecheck synccheck initcheck; do
  for prog in "python -c 'import __graft_entry__ as g; g.smoke()'" "python tools/prof_step.py --config c1 --iters 2"; do
    echo "=== $tool: $prog" >> $OUT
    timeout 900 bash -c "compute-sanitizer --tool $tool --error-exitcode 7 --print-limit 20 $prog" > gpurun_out/san.log 2>&1
    echo "rc=$?" >> $OUT
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= (Invalid|Race|Uninit|Barrier|Error)|smoke ok|loss trace" gpurun_out/san.log | head -20 >> $OUT
  done
done
cat $OUT
