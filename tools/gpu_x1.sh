#!/bin/bash
# one-off: SpMV diagnostic + config-3 fork/batch variants + eager in-situ timings
cd $GRAFT_REPO_ROOT
timeout 900 python tools/diag_spmv.py cart128_p3 cfg3s > gpurun_out/diag_spmv.log 2>&1; echo "diag rc $?"
for c in cfg3 cfg4; do
  DGAS_EAGER=1 DGAS_EAGER_TIMING=1 DGAS_VERBOSE=1 timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/eager_$c.log 2> gpurun_out/eager_$c.err; echo "eager $c rc $?"
done
CONFIGS="cfg3" VARIANTS="-;DGAS_NO_FORK=1;DGAS_MR_B=16;DGAS_MR_B=8;DGAS_MR_S=8;DGAS_ND_PDL=0;DGAS_SPMV_PSPLIT=0" bash tools/gpu_ab.sh > /dev/null 2>&1
cat gpurun_out/ab.log
CONFIGS="cfg4" VARIANTS="-;DGAS_NO_FORK=1" bash tools/gpu_ab.sh > /dev/null 2>&1
cp gpurun_out/ab.log gpurun_out/ab_cfg4.log; cat gpurun_out/ab_cfg4.log
grep -h "eager\|phase\|dgas:" gpurun_out/eager_cfg3.err gpurun_out/eager_cfg4.err | head -60
cat gpurun_out/diag_spmv.log
