#!/bin/bash
# A/B sweep of env settings: AB_CONFIGS="cfg4 cfg2" AB_SETS="base u2:DGAS_UNROLL=2 u4:DGAS_UNROLL=4"
# prints PCG it/s, ms per solve and the per-kernel ms (spmv, local, coarse, apply_total)
cd $GRAFT_REPO_ROOT
for C in ${AB_CONFIGS:-cfg4}; do
  for set in ${AB_SETS:-base}; do
    tag=${set%%:*}; envs=""
    [ "$set" != "$tag" ] && envs=$(echo ${set#*:} | tr ',' ' ')
    env $envs timeout 600 python bench.py --config $C --steps ${AB_STEPS:-3} --warmup 3 --no-cpu-baseline ${AB_ARGS} > gpurun_out/ab_${C}_$tag.log 2>&1
    echo "$C $tag rc $? $(tail -1 gpurun_out/ab_${C}_$tag.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernels"]; print(round(d["value"],1), round(d["ms_per_step"],3), "spmv", round(k["spmv"]["ms"],4), "local", round(k["local"]["ms"],4), "coarse", round(k["coarse"]["ms"],4), "apply", round(k["apply_total"]["ms"],4))' 2>/dev/null)"
  done
done
