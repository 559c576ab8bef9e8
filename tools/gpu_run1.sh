cd $GRAFT_REPO_ROOT
L=gpurun_out/run1.log
nvidia-smi -L > $L 2>&1
for c in cfg3 cfg4; do
  DGAS_VERBOSE=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2> gpurun_out/bench_$c.err; echo "bench $c rc $?" >> $L
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1; echo "smoke rc $?" >> $L
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/tests.log 2>&1; echo "tests rc $?" >> $L
tail -3 gpurun_out/tests.log >> $L
cat $L
