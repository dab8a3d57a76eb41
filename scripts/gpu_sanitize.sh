#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel family
# (scripts/sanitize_all.py: fused fast solve, 4-CTA cluster projection, exact
# solve, bitwise projection, validation) and a traced solve
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  PF_PROJ_CLUSTER=4 timeout 900 compute-sanitizer --tool $tool --print-limit 6 python scripts/sanitize_all.py 12 \
    > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(grep "ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/san_$tool.log | tail -1)"
done
timeout 600 compute-sanitizer --tool memcheck python scripts/memcheck_trace.py > gpurun_out/san_trace.log 2>&1
echo "memcheck (trace) rc=$? $(grep "ERROR SUMMARY" gpurun_out/san_trace.log | tail -1)"
