#!/bin/bash
# new-test pass: build, smoke, the round-2 parity files, then a short bench + reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest -m gpu -q -rs ${TESTS:-tests/test_parity_scale.py tests/test_reductions_golden.py tests/test_dropin.py tests/test_gpu_parity.py} > gpurun_out/newtests.log 2>&1; echo "tests rc=$?"; tail -40 gpurun_out/newtests.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref.json
timeout 900 python bench.py --steps 20 --warmup 5 --no-ttq --no-extras > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
