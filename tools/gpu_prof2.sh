#!/bin/bash
# round-2 profile pass: launch lists of four configs (eager path), ncu --set full of the dominant kernels of
# config 3 (default bench) and config 4
cd $GRAFT_REPO_ROOT
LAUNCH_CONFIGS="cfg2 cfg3 cfg4 cfg5_p6q6" FULL=cfg3 FULL_KERNELS="k_local_mrhs_w|k_spmv_cls" FULL_SKIP=2 FULL_COUNT=2 bash tools/gpu_profile_round.sh > /dev/null 2>&1
cp gpurun_out/profile_round.log gpurun_out/profile_round_a.log
LAUNCH_CONFIGS="" FULL=cfg4 FULL_KERNELS="k_local_panel|k_spmv_ring" FULL_SKIP=2 FULL_COUNT=2 bash tools/gpu_profile_round.sh > /dev/null 2>&1
cat gpurun_out/profile_round_a.log gpurun_out/profile_round.log
