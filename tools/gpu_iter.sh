#!/bin/bash
# iteration helper: selected GPU tests (KEXPR), then bench lines (CONFIGS) with verbose setup logs
cd $GRAFT_REPO_ROOT
L=gpurun_out/iter.log
nvidia-smi -L > $L 2>&1
if [ -n "$KEXPR" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu -x -k "$KEXPR" > gpurun_out/iter_tests.log 2>&1; echo "tests rc $?" >> $L
  tail -15 gpurun_out/iter_tests.log >> $L
fi
for c in ${CONFIGS:-}; do
  DGAS_VERBOSE=1 timeout 600 env $BENV python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > gpurun_out/iter_$c.log 2> gpurun_out/iter_$c.err
  echo "bench $c rc $?" >> $L
  python - "$c" >> $L <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/iter_{c}.log").read().strip().splitlines()[-1]); k = d["kernels"]
    print(c, "it/s %.1f" % d["value"], "iters", d["run"]["iters_per_solve"], "K %.6f" % d["run"]["lanczos_cond"],
          " ".join("%s %.4f" % (n, k[n]["ms"]) for n in k))
except Exception as e:
    print(c, "FAILED", e)
PY
  grep -i "multi-RHS\|class SpMV\|ND coarse\|error" gpurun_out/iter_$c.err | head -5 >> $L
done
cat $L
