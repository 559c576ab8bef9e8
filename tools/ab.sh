#!/bin/bash
cd $GRAFT_REPO_ROOT
C=${AB_CONFIG:-cfg4}
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ab_${C}_$tag.log 2>&1; echo "$tag rc $?"; }
run base
for b in 31 40 55 80; do for sl in 3 6 12; do run lo_${b}_$sl DGAS_APPLY_BUDGET_KB=$b DGAS_APPLY_SLOT_KB=$sl; done; done
