#!/bin/bash
# A/B sweep of launch/ring parameters on one config (kernel timings; one line per setting)
cd $GRAFT_REPO_ROOT
C=${AB_CONFIG:-cfg4}
run() {  # tag env...
  tag=$1; shift
  env "$@" timeout 600 python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ab_${C}_$tag.log 2>&1
  echo "$tag rc $?"
}
run base
run sp_4_2_48 DGAS_SPMV_CTAS_PER_SM=4 DGAS_SPMV_G=2 DGAS_SPMV_BUDGET_KB=48
run sp_4_4_100 DGAS_SPMV_CTAS_PER_SM=4 DGAS_SPMV_G=4 DGAS_SPMV_BUDGET_KB=50
run sp_8_1_24 DGAS_SPMV_CTAS_PER_SM=8 DGAS_SPMV_G=1 DGAS_SPMV_BUDGET_KB=24
run sp_3_2_64 DGAS_SPMV_CTAS_PER_SM=3 DGAS_SPMV_G=2 DGAS_SPMV_BUDGET_KB=64
run sp_2_2_96 DGAS_SPMV_CTAS_PER_SM=2 DGAS_SPMV_G=2 DGAS_SPMV_BUDGET_KB=96
run lo_27_6 DGAS_APPLY_BUDGET_KB=27 DGAS_APPLY_SLOT_KB=6
run lo_40_8 DGAS_APPLY_BUDGET_KB=40 DGAS_APPLY_SLOT_KB=8
run lo_36_12 DGAS_APPLY_BUDGET_KB=36 DGAS_APPLY_SLOT_KB=12
run lo_80_16 DGAS_APPLY_BUDGET_KB=80 DGAS_APPLY_SLOT_KB=16
run lo_110_24 DGAS_APPLY_BUDGET_KB=110 DGAS_APPLY_SLOT_KB=24
