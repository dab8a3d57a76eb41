#!/bin/bash
# Round checkpoint: smoke, gpu tests, bench (+ttq, cpu baseline), reference arm,
# the bench's ncu launch list and one ncu --set full capture of k_fused.
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests.log
timeout 1200 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref_${TAG}.json 2>/dev/null; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 20 --warmup 3 --no-ttq --no-cpu-baseline --no-extras > /dev/null 2>&1; echo "ncu launches rc=$?"
bash scripts/gpu_ncu.sh ${TAG} cfg2 > /dev/null 2>&1; echo "ncu full rc=$?"
