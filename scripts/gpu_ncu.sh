#!/bin/bash
# ncu --set full of the second k_fused launch (10 iterations of cfg2) + source page
TAG=${1:-v6}
CFG=${2:-cfg2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python scripts/prof_fused.py $CFG 10 > gpurun_out/prof_plain_${TAG}.log 2>&1; cat gpurun_out/prof_plain_${TAG}.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 1 -c 1 -f -o gpurun_out/fused_${CFG}_${TAG} python scripts/prof_fused.py $CFG 10 > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_${TAG}.log
