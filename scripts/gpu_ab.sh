#!/bin/bash
# A/B of the current library against a variant (PF_B200_LIB), same box, interleaved
# usage: CFGS="cfg1_v0.3 cfg2" ITERS="2000 300" VARIANT=old bash scripts/gpu_ab.sh
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
set -- $ITERS
for c in ${CFGS:-cfg1_v0.3 cfg2}; do
  n=$1; shift
  for rep in 1 2; do
    echo "new $c: $(python scripts/prof_fused.py $c $n 2>&1 | tail -1)"
    echo "${VARIANT:-old} $c: $(PF_B200_LIB=paper_2605_01748_b200/_build/${VARIANT:-old}/libpf_b200.so python scripts/prof_fused.py $c $n 2>&1 | tail -1)"
  done
done
