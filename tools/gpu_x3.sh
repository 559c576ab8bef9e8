#!/bin/bash
# one-off: warp-chain multi-RHS kernel: parity tests, geometry sweep on config 3, class-SpMV occupancy
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -q -m gpu -x -k "local_kernel_variants and cart" > gpurun_out/x3_tests.log 2>&1; echo "tests rc $?"; tail -4 gpurun_out/x3_tests.log
CONFIGS="cfg3" VARIANTS="${XV:--;DGAS_MR_G=2;DGAS_MR_G=8;DGAS_MR_G=2 DGAS_MR_NW=8;DGAS_MR_G=4 DGAS_MR_NW=8;DGAS_MR_G=4 DGAS_MR_NW=2;DGAS_MR_S=4;DGAS_MR_S=16;DGAS_CLS_MINB=2}" VERB=1 bash tools/gpu_ab.sh > /dev/null 2>&1
cat gpurun_out/ab.log
grep -h "multi-RHS\|class SpMV" gpurun_out/ab_err_cfg3.log | tail -2
