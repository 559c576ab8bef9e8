#!/bin/bash
# one-off: parity tests of the kernels touched + config 3 / 4 benches (+ optional variants)
cd $GRAFT_REPO_ROOT
timeout 2000 python -m pytest tests -q -m gpu -x -k "${KX:-local_kernel_variants or spmv or dedup or full_size}" > gpurun_out/x4_tests.log 2>&1; echo "tests rc $?"; tail -4 gpurun_out/x4_tests.log
CONFIGS="${XC:-cfg3}" VARIANTS="${XV:--}" VERB=1 bash tools/gpu_ab.sh > /dev/null 2>&1
cat gpurun_out/ab.log
