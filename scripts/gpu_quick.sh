#!/bin/bash
# quick GPU check: build, gpu tests, short bench without time-to-quality
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/gputests.log
timeout 600 python bench.py --steps 200 --warmup 10 --no-ttq --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
