#!/bin/bash
# one-off: config-3 batch-size sweep of the multi-RHS local solve + ncu full captures of its hot kernels
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x -k "test_spmv_rhs and cart128 or dedup_is_bitwise" > gpurun_out/x2_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/x2_tests.log
CONFIGS="cfg3" VARIANTS="DGAS_MR_B=4;DGAS_MR_B=6;DGAS_MR_B=8;DGAS_MR_B=10;DGAS_MR_B=12;DGAS_MR_B=16;DGAS_MR_B=20;DGAS_MR_B=24;DGAS_MR_B=8 DGAS_MR_S=8;DGAS_MR_B=8 DGAS_MR_S=2" VERB=1 bash tools/gpu_ab.sh > /dev/null 2>&1
cat gpurun_out/ab.log
grep -h "multi-RHS" gpurun_out/ab_err_cfg3.log | tail -2
CONFIG=cfg3 NCU_KS="k_local_mrhs k_spmv_cls k_restrict_chunk k_prolong" bash tools/gpu_ncu.sh
CONFIG=cfg3 BENV="DGAS_MR_B=8" NCU_KS="k_local_mrhs" bash tools/gpu_ncu.sh
