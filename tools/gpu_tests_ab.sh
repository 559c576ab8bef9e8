#!/bin/bash
# iteration helper: selected parity tests (KX = pytest -k expression), then bench lines for configs (XC) x env
# variants (XV, ';'-separated) through tools/gpu_ab.sh
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -q -m gpu -x -k "${KX:-pcg_parity or local_kernel_variants or eager_path or full_size or nested_dissection}" > gpurun_out/x7_tests.log 2>&1; echo "tests rc $?"; tail -4 gpurun_out/x7_tests.log
CONFIGS="${XC:-cfg3 cfg4 cfg5_p3q3 cfg2}" VARIANTS="${XV:--;DGAS_FUSE_R=0}" bash tools/gpu_ab.sh > /dev/null 2>&1
grep -v "ND coarse" gpurun_out/ab.log
