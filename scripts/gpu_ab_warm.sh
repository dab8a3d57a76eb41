#!/bin/bash
# A/B after a warm-up (beta settled): CFG W N, current library vs _build/$VARIANT
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for rep in 1 2; do
  echo "new: $(python scripts/prof_fused_warm.py ${CFG:-cfg2} ${W:-1500} ${N:-300} 2>&1 | tail -1)"
  echo "${VARIANT:-old}: $(PF_B200_LIB=paper_2605_01748_b200/_build/${VARIANT:-old}/libpf_b200.so python scripts/prof_fused_warm.py ${CFG:-cfg2} ${W:-1500} ${N:-300} 2>&1 | tail -1)"
done
