#!/bin/bash
# bitwise check (state digests after 300 iterations) and settled timings of the
# in-tree library against _r1/ (a copy of an earlier revision)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for c in ${DCFGS:-cfg1_v0.3 cfg2}; do
  echo "NEW: $(python scripts/state_digest.py $c 300 2>/dev/null)"
  echo "R1:  $(python _r1/scripts/state_digest.py $c 300 2>/dev/null)"
done
bash scripts/gpu_vs_r1.sh
