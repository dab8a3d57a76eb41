#!/bin/bash
# phase ablation timings of the fused kernel (results are wrong by design; timing only)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python scripts/prof_fused.py cfg2 5 >/dev/null 2>&1
for ab in ${ABL:-0 1 2 3 0}; do
  r=$(PF_FAST_ABLATE=$ab timeout 300 python scripts/prof_fused.py cfg2 40 2>&1 | tail -1)
  echo "ablate=$ab :: $r"
done
