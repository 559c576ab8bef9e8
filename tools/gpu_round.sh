#!/bin/bash
# one gpurun round: smoke, parity tests, benches, optional ncu launch list / full capture
cd $GRAFT_REPO_ROOT
L=gpurun_out/round.log
nvidia-smi -L > $L 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1; echo "smoke rc $?" >> $L
if [ -z "$SKIP_TESTS" ]; then
  timeout 2400 python -m pytest tests/test_gpu_parity.py -q -m gpu --maxfail=25 > gpurun_out/tests.log 2>&1; echo "tests rc $?" >> $L
  tail -3 gpurun_out/tests.log >> $L
fi
for c in ${BENCH_CONFIGS:-cfg4}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc $?" >> $L
done
if [ -n "$NCU_CONFIG" ]; then
  # launch list of the same command; DGAS_EAGER=1 makes every PCG iteration kernel its own launch (ncu
  # does not profile inside the graph's conditional WHILE node); window inside the first solve
  DGAS_EAGER=1 timeout 600 python bench.py --config $NCU_CONFIG --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_plain.log 2>&1 && \
  DGAS_EAGER=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s ${NCU_SKIP:-500} -c ${NCU_COUNT:-80} --csv --log-file gpurun_out/launches_$NCU_CONFIG.csv python bench.py --config $NCU_CONFIG --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu.log 2>&1
  echo "ncu launches rc $?" >> $L
fi
if [ -n "$NCU_FULL" ]; then
  timeout 600 python bench.py --config $NCU_FULL --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_full_plain.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNELS:-k_local|k_spmv3}" -s ${NCU_FSKIP:-6} -c ${NCU_FCOUNT:-2} -o gpurun_out/prof_$NCU_FULL -f python bench.py --config $NCU_FULL --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc $?" >> $L
fi
if [ -n "$PAPER" ]; then
  timeout 1500 python tools/paper_tables.py $PAPER > gpurun_out/paper.log 2>&1; echo "paper rc $?" >> $L
fi
cat $L
