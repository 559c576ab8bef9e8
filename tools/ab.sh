#!/bin/bash
cd $GRAFT_REPO_ROOT
C=${AB_CONFIG:-cfg4}
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ab_${C}_$tag.log 2>&1; echo "$tag rc $?"; }
run base
run sp3_48 DGAS_SPMV_CTAS_PER_SM=3 DGAS_SPMV_BUDGET_KB=48
run sp4_48 DGAS_SPMV_CTAS_PER_SM=4 DGAS_SPMV_BUDGET_KB=48
run sp4_36 DGAS_SPMV_CTAS_PER_SM=4 DGAS_SPMV_BUDGET_KB=36
run sp3_96 DGAS_SPMV_CTAS_PER_SM=3 DGAS_SPMV_BUDGET_KB=96
run nd DGAS_COARSE_MODE=nd
run nd64 DGAS_COARSE_MODE=nd DGAS_ND_LEAF=64
