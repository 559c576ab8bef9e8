#!/bin/bash
# diagnostic pass: smoke, per-config bench with ND verbose output, eager per-phase timing, GPU tests
cd $GRAFT_REPO_ROOT
L=gpurun_out/diag.log
nvidia-smi -L > $L 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1; echo "smoke rc $?" >> $L
for c in ${DIAG_CONFIGS:-cfg3 cfg4}; do
  DGAS_VERBOSE=1 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/diag_bench_$c.log 2>&1; echo "bench $c rc $?" >> $L
  DGAS_EAGER=1 DGAS_EAGER_TIMING=1 timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/diag_eager_$c.log 2>&1; echo "eager $c rc $?" >> $L
done
if [ -n "$DIAG_TESTS" ]; then
  timeout 2400 python -m pytest tests -q -m gpu -x $DIAG_TESTS > gpurun_out/diag_tests.log 2>&1; echo "tests rc $?" >> $L
  tail -5 gpurun_out/diag_tests.log >> $L
fi
cat $L
