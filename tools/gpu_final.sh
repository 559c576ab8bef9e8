#!/bin/bash
# end-of-round GPU pass: smoke, full parity suite, benches (every config, the NEXT-4 variant, the
# reference arm), ncu launch list and full capture of the dominant kernels (cfg4)
cd $GRAFT_REPO_ROOT
L=gpurun_out/final.log
nvidia-smi -L > $L 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1; echo "smoke rc $?" >> $L
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/tests_final.log 2>&1; echo "tests rc $?" >> $L
tail -3 gpurun_out/tests_final.log >> $L
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench default rc $?" >> $L
for c in cfg1 cfg2 cfg3 cfg4 cfg5_p1q1 cfg5_p2q2 cfg5_p3q3 cfg5_p4q4 cfg5_p5q5 cfg5_p6q6 cfg5_p6q1; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc $?" >> $L
done
for c in cfg4 cfg3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --local-f32 > gpurun_out/bench_${c}_f32.log 2>&1; echo "bench $c f32 rc $?" >> $L
done
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "bench reference rc $?" >> $L
DGAS_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 500 -c 80 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu.log 2>&1; echo "ncu launches rc $?" >> $L
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_local_panel|k_spmv_ring" -s 2 -c 2 -o gpurun_out/prof_cfg4 -f python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?" >> $L
cat $L
