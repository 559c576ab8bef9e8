#!/bin/bash
# Profiling round: (1) ncu launch lists (time + DRAM bytes per launch) of the bench command for several
# configs, DGAS_EAGER=1 so each PCG-iteration kernel is its own launch (ncu does not see inside the graph's
# WHILE node); (2) one `ncu --set full` capture of the dominant kernels of the headline config;
# (3) CTAs-per-SM sweep of the panel local-solve kernel (duration, DRAM read, L2 hit rate) on cfg3/cfg4.
cd $GRAFT_REPO_ROOT
L=gpurun_out/profile_round.log
nvidia-smi -L > $L 2>&1
for c in ${LAUNCH_CONFIGS:-cfg2 cfg3 cfg4 cfg5_p6q6}; do
  DGAS_EAGER=1 timeout 600 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$c.log 2>&1 && \
  DGAS_EAGER=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s ${NCU_SKIP:-400} -c ${NCU_COUNT:-60} --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1
  echo "launches $c rc $?" >> $L
done
if [ -n "$FULL" ]; then
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${FULL_KERNELS:-k_local_panel|k_spmv_ring}" \
    -s ${FULL_SKIP:-2} -c ${FULL_COUNT:-2} -o gpurun_out/prof_$FULL -f python bench.py --config $FULL --steps 1 --warmup 1 \
    --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_full_$FULL.log 2>&1
  echo "full $FULL rc $?" >> $L
fi
for c in ${SWEEP_CONFIGS:-}; do
  for cps in ${CPS_LIST:-1 2 3 4 5 6 7}; do
    DGAS_LOCAL_CPS=$cps timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:k_local_panel -s 2 -c 1 --csv --log-file gpurun_out/sweep_${c}_cps${cps}.csv \
      python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --kernel-reps 2 > gpurun_out/sweep_${c}_${cps}.log 2>&1
    echo "sweep $c cps $cps rc $?" >> $L
  done
done
cat $L
