#!/bin/bash
cd $GRAFT_REPO_ROOT
C=${AB_CONFIG:-cfg4}
run() { tag=$1; shift; env "$@" timeout 600 python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ab_${C}_$tag.log 2>&1; echo "$tag rc $?"; }
run base
run leaf16 DGAS_ND_LEAF=16
run leaf64 DGAS_ND_LEAF=64
run leaf128 DGAS_ND_LEAF=128
