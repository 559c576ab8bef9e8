#!/bin/bash
# one gpurun round: parity tests, smoke, benches, ncu launch list (logs under gpurun_out/)
cd $GRAFT_REPO_ROOT
L=gpurun_out/round.log
nvidia-smi -L > $L 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1; echo "smoke rc $?" >> $L
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -m gpu --maxfail=25 > gpurun_out/tests.log 2>&1; echo "tests rc $?" >> $L
for c in ${BENCH_CONFIGS:-cfg4}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc $?" >> $L
done
if [ -n "$NCU_CONFIG" ]; then
  timeout 600 python bench.py --config $NCU_CONFIG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_spmv2|k_restrict|k_apply|k_prolong" -s 8 -c 40 --csv --log-file gpurun_out/launches_$NCU_CONFIG.csv python bench.py --config $NCU_CONFIG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1
  echo "ncu rc $?" >> $L
fi
tail -3 gpurun_out/tests.log >> $L
cat $L
if [ -n "$NCU_FULL" ]; then
  timeout 600 python bench.py --config $NCU_FULL --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_full_plain.log 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNELS:-k_apply|k_spmv2}" -s 6 -c 2 -o gpurun_out/prof_$NCU_FULL -f python bench.py --config $NCU_FULL --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_full.log 2>&1
  echo "ncu full rc $?" >> $L
  tail -2 $L
fi
