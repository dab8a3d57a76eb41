#!/bin/bash
# quick iteration: fused timings on cfg2 / target_k4 / cfg1, then the fast-mode GPU tests
mkdir -p gpurun_out
for c in ${CFGS:-cfg2 target_k4_v0.3 cfg1_v0.3}; do python scripts/prof_fused_warm.py $c 200 500 2>&1 | tail -2; done
timeout 1200 python -m pytest -m gpu -q -x ${TESTS:-tests/test_gpu_parity.py tests/test_distributed.py} > gpurun_out/iter_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/iter_tests.log
