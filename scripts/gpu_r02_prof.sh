#!/bin/bash
mkdir -p gpurun_out
python scripts/diag_smoke.py > gpurun_out/diag_smoke.log 2>&1; echo "diag rc=$?"; cat gpurun_out/diag_smoke.log | cut -c1-600
bash scripts/gpu_ncu.sh r02a cfg2
ncu -i gpurun_out/fused_cfg2_r02a.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/fused_cfg2_r02a_source.csv 2>/dev/null; echo "src rc=$?"
