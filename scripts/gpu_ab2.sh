#!/bin/bash
# A/B of the current library vs _build/old (built from the previous revision),
# settled timings on several configs, then the fast-mode GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for c in ${CFGS:-cfg2 cfg1_v0.3}; do
  for rep in 1 2; do
    echo "new: $(python scripts/prof_fused_warm.py $c ${W:-200} ${N:-300} 2>&1 | tail -1)"
    echo "old: $(PF_B200_LIB=paper_2605_01748_b200/_build/old/libpf_b200.so python scripts/prof_fused_warm.py $c ${W:-200} ${N:-300} 2>&1 | tail -1)"
  done
done
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest -m gpu -q -x $TESTS > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/ab_tests.log; fi
