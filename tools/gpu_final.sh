#!/bin/bash
# end-of-round GPU pass: smoke, full parity suite, benches (every config, the fp32-factor variant, the
# reference arm), ncu launch list of the default bench and a full capture of its dominant kernels
cd $GRAFT_REPO_ROOT
L=gpurun_out/final.log
nvidia-smi -L > $L 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1; echo "smoke rc $?" >> $L
if [ -z "$SKIP_TESTS" ]; then
  timeout 2400 python -m pytest tests -q -m gpu -rA -s > gpurun_out/tests_final.log 2>&1; echo "tests rc $?" >> $L
  grep -E "passed|failed" gpurun_out/tests_final.log | tail -2 >> $L
fi
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench default rc $?" >> $L
for c in ${CONFIGS:-cfg1 cfg2 cfg3 cfg4 cfg5_p1q1 cfg5_p2q1 cfg5_p2q2 cfg5_p3q1 cfg5_p3q3 cfg5_p4q1 cfg5_p4q4 cfg5_p5q1 cfg5_p5q5 cfg5_p6q1 cfg5_p6q6}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc $?" >> $L
done
for c in cfg4 cfg3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --local-f32 > gpurun_out/bench_${c}_f32.log 2>&1; echo "bench $c f32 rc $?" >> $L
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "bench reference rc $?" >> $L
if [ -z "$SKIP_NCU" ]; then
  DGAS_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s ${NCU_SKIP:-500} -c 80 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu launches rc $?" >> $L
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_local_mrhs_t|k_spmv_cls_t|k_restrict_chunk|k_prolong" -s 4 -c 4 -o gpurun_out/prof_default -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?" >> $L
fi
cat $L
# config 2 launch list (its setup builds the explicit inverses with ~1,200 launches: skip past them)
if [ -z "$SKIP_NCU" ]; then
  DGAS_EAGER=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s ${NCU_SKIP2:-2200} -c 60 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cfg2.log 2>&1; echo "ncu cfg2 launches rc $?" >> $L
fi
for c in cfg3 cfg4; do
  DGAS_EAGER=1 DGAS_EAGER_TIMING=1 timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/eager_$c.log 2> gpurun_out/eager_$c.err
  echo "in-situ $c: $(grep -h 'eager timing' gpurun_out/eager_$c.err | tail -1)" >> $L
done
tail -4 $L
