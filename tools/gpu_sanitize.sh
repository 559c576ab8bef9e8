#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over the small configs (summary in gpurun_out/sanitize.log)
cd $GRAFT_REPO_ROOT
L=gpurun_out/sanitize.log
: > $L
for c in ${CASES:-cfg1 cfg2s cfg4s cfg4s_nd}; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python tools/sanitize_run.py $c ${MAXIT:-40} > gpurun_out/san_${c}_${tool}.log 2>&1
    rc=$?
    echo "$c $tool rc=$rc: $(grep -E 'ERROR SUMMARY|iters' gpurun_out/san_${c}_${tool}.log | tr '\n' ' ')" >> $L
  done
done
cat $L
