#!/bin/bash
cd $GRAFT_REPO_ROOT
DGAS_CLS_TC=1 timeout 1200 python -m pytest tests -q -m gpu -x -k "test_spmv_rhs and (cart or cfg3s or cfg1) or dedup or (pcg_parity and (cfg3s or cart or cfg1))" > gpurun_out/x8_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/x8_tests.log
CONFIGS="cfg3" VARIANTS="-;DGAS_CLS_TC=1;DGAS_CLS_TC=1 DGAS_CLS_RUN=32;DGAS_CLS_TC=1 DGAS_CLS_RUN=64;DGAS_CLS_TC=1 DGAS_CLS_RUN=16" VERB=1 bash tools/gpu_ab.sh > /dev/null 2>&1
grep -v "ND coarse" gpurun_out/ab.log
grep -h "class SpMV" gpurun_out/ab_err_cfg3.log | tail -1
