#!/bin/bash
# in-loop phase times (eager path, CUDA events around every phase of every PCG iteration: DGAS_EAGER_TIMING) for
# configs (XC) x env variants (XV, ';'-separated)
cd $GRAFT_REPO_ROOT
IFS=';' read -ra VS <<< "${XV:--}"
for c in ${XC:-cfg3}; do
  for v in "${VS[@]}"; do
    envs=""; [ "$v" != "-" ] && envs="$v"
    env $envs DGAS_EAGER=1 DGAS_EAGER_TIMING=1 timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/eager_$c.log 2> gpurun_out/eager_$c.err
    echo "$c [$v] $(grep -h 'eager timing' gpurun_out/eager_$c.err | tail -1)"
  done
done
