#!/bin/bash
# the N=2 shared-GPU bench dry run repeated: the sharded time-to-1% quality and
# its single-GPU cross-check each time
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for r in $(seq ${REPS:-3}); do
  NS=2 CFG=${CFG:-cfg1} STEPS=${STEPS:-20} bash scripts/gpu_bench_shared.sh > /dev/null 2>&1
  python - <<'PY'
import json
t = open("gpurun_out/shared_n2.json").read().strip().splitlines()
d = json.loads(t[-1]) if t else {}
x = d.get("time_to_1pct") or {}
print(x.get("optimality_at_k_star_vs_reference_fixed_point"), x.get("single_gpu_check"), d.get("check"), flush=True)
PY
done
