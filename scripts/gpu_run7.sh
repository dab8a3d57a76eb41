timeout 900 python scripts/ttq_probe.py cfg1_v0.3 cfg1 cfg2_v0.3 target_k4_v0.3 2>&1 | tail -8
timeout 1200 python bench.py --steps 300 --warmup 10 2>&1 | tail -2
