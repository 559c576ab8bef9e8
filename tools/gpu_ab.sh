#!/bin/bash
# A/B helper: optional pytest selection, then bench lines for configs x env variants.
#   KEXPR="pytest -k expression"  CONFIGS="cfg3 cfg4"  VARIANTS="DGAS_X=0;DGAS_X=1"  (";"-separated env sets, "-" = none)
cd $GRAFT_REPO_ROOT
L=gpurun_out/ab.log
nvidia-smi -L > $L 2>&1
if [ -n "$KEXPR" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu -rA -s -k "$KEXPR" > gpurun_out/ab_tests.log 2>&1; echo "tests rc $?" >> $L
  tail -5 gpurun_out/ab_tests.log >> $L
fi
IFS=';' read -ra VS <<< "${VARIANTS:--}"
for c in ${CONFIGS:-}; do
  for v in "${VS[@]}"; do
    envs=""; [ "$v" != "-" ] && envs="$v"
    out=$(env $envs DGAS_VERBOSE=${VERB:-0} timeout 600 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline 2> gpurun_out/ab_err_${c}.log | tail -1)
    echo "$c [$v] $(echo "$out" | python -c 'import sys,json
try:
  d=json.loads(sys.stdin.read()); k=d["kernels"]
  print("it/s %.1f iters %s K %.4f | " % (d["value"], d["run"]["iters_per_solve"], d["run"]["lanczos_cond"]) + " ".join("%s %.4f" % (n, k[n]["ms"]) for n in k))
except Exception as e: print("FAILED", e)')" >> $L
    grep -i "ND coarse\|error" gpurun_out/ab_err_${c}.log | head -3 >> $L
  done
done
cat $L
