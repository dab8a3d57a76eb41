#!/bin/bash
# A/B of the in-tree library against _r1/ (a copy of an earlier revision with its
# own library and scripts), settled and from-cold regimes
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for c in ${CFGS:-cfg2}; do
  for r in 1 2; do
    echo "new: $(python scripts/prof_fused_warm.py $c ${W:-200} ${N:-300} 2>&1 | tail -1)"
    echo "r1:  $(python _r1/scripts/prof_fused_warm.py $c ${W:-200} ${N:-300} 2>&1 | tail -1)"
  done
done
