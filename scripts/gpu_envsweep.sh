#!/bin/bash
# timing sweep over environment settings: ENVS="A=1 B=2;A=2;..." (cfg2, 40 iterations)
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
python scripts/prof_fused.py ${CFG:-cfg2} 5 >/dev/null 2>&1
IFS=';' read -ra SETS <<< "$ENVS"
for e in "${SETS[@]}"; do
  r=$(env $e timeout 300 python scripts/prof_fused.py ${CFG:-cfg2} 40 2>&1 | tail -1)
  echo "[$e] :: $r"
done
