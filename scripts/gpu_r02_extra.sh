#!/bin/bash
# round-2 evidence: sanitizers (incl. the run-slot layout and the time-to-quality
# snapshot path) and an ncu --set full capture of k_fused at config 3 (run slots)
mkdir -p gpurun_out
bash scripts/gpu_sanitize.sh
for tool in memcheck racecheck; do
  PF_FAST_RS=1 PF_FAST_TPS=512 timeout 900 compute-sanitizer --tool $tool --print-limit 6 python scripts/sanitize_fused.py 90 4 \
    > gpurun_out/san_rs_$tool.log 2>&1
  echo "run slots $tool rc=$? $(grep "ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/san_rs_$tool.log | tail -1)"
done
python scripts/prof_fused.py cfg3 4 > gpurun_out/prof_plain_cfg3.log 2>&1; cat gpurun_out/prof_plain_cfg3.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -s 1 -c 1 -f -o gpurun_out/fused_cfg3_r02 python scripts/prof_fused.py cfg3 4 > gpurun_out/ncu_cfg3.log 2>&1; echo "ncu cfg3 rc=$?"
