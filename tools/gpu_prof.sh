#!/bin/bash
# quick checks + source-level ncu of selected kernels (one ncu tool per call)
cd $GRAFT_REPO_ROOT
L=gpurun_out/prof.log
: > $L
for c in ${BENCH_CONFIGS:-cfg5_p6q6}; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc $?" >> $L
done
C=${NCU_FULL:-cfg4}
timeout 600 python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_full_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNELS:-k_local}" -s ${NCU_SKIP:-4} -c ${NCU_COUNT:-1} -o gpurun_out/prof_$C -f python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_full.log 2>&1
echo "ncu $C rc $?" >> $L
cat $L
