#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for c in cfg1 cfg1_v0.3 target_k4_v0.3; do python scripts/prof_fused.py $c 400 2>&1 | tail -1; done
for t in 256 512 1024; do echo "tps=$t"; PF_FAST_TPS=$t python scripts/prof_fused.py cfg1 400 2>&1 | tail -1; done
