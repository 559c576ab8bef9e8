#!/bin/bash
cd $GRAFT_REPO_ROOT
CONFIGS="cfg3" VARIANTS="-;DGAS_MR_NW=4;DGAS_MR_KERNEL=2" bash tools/gpu_ab.sh > /dev/null 2>&1; cp gpurun_out/ab.log gpurun_out/ab1.log
CONFIGS="cfg4 cfg5_p6q6 cfg5_p3q3" VARIANTS="-;DGAS_PRODUCER_NS=32;DGAS_PRODUCER_NS=128;DGAS_PRODUCER_NS=400" bash tools/gpu_ab.sh > /dev/null 2>&1; cp gpurun_out/ab.log gpurun_out/ab2.log
cat gpurun_out/ab1.log gpurun_out/ab2.log | grep -v "ND coarse"
