#!/bin/bash
# one ncu --set full capture per kernel regex (NCU_K1, NCU_K2, ...) on CONFIG, after a plain run of the same command
cd $GRAFT_REPO_ROOT
C=${CONFIG:-cfg3}
timeout 600 env $BENV python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_plain_$C.log 2>&1; echo "plain rc $?"
i=0
for K in ${NCU_KS:-k_local_mrhs}; do
  i=$((i+1))
  timeout 900 env $BENV ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${NCU_S:-2} -c ${NCU_C:-1} -o gpurun_out/prof_${C}_$i -f python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_${C}_$i.log 2>&1
  echo "ncu $K rc $?"
done
