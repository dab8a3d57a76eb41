#!/bin/bash
# bounded config-3 / north-star probes on one B200
free -g | head -2; nvidia-smi --query-gpu=memory.total --format=csv
MEM=$(free -g | awk '/Mem:/{print $2}')
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 300 python -c "
import bench, json
print(json.dumps(bench.time_to_quality('target_k4_v0.3', cpu=False)))
" 2>&1 | tail -2
if [ "$MEM" -ge 96 ]; then
  timeout 900 python scripts/cfg3_probe.py cfg3 20 2>&1 | tail -8
else
  echo "host memory ${MEM} GB: skipping cfg3"
fi
