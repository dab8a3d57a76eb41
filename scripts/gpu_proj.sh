#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "proj" > gpurun_out/projtests.log 2>&1; echo "proj tests rc=$?"; tail -2 gpurun_out/projtests.log
PF_PROJ_STATS=1 python scripts/prof_project.py cfg2 210
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_edge_trim|k_demand_trim|Sort|k_scores|k_edge_gather|k_segment" --csv --log-file gpurun_out/proj_launches.csv python scripts/prof_project.py cfg2 210 > /dev/null 2>&1; echo ncu=$?
