#!/bin/bash
# config 1 (small, latency-bound) timing over tile sizes, with and without the phase probe
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for t in ${TPS:-256 512 1024 2048 4096}; do
  echo "tps=$t"; PF_FAST_TPS=$t python scripts/prof_fused.py cfg1_v0.3 2000 2>&1 | tail -1
  PF_FAST_PROBE=1 PF_FAST_TPS=$t python scripts/prof_fused.py cfg1_v0.3 2000 2>&1 | grep probe | tail -1
done
