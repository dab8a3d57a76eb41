set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -25
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline 2>&1 | tail -3
timeout 600 python scripts/prof_fused.py cfg2 20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 -o gpurun_out/fused_cfg2 python scripts/prof_fused.py cfg2 10 2>&1 | tail -5
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python scripts/prof_fused.py cfg2 10 2>&1 | tail -3
