python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25
timeout 900 python bench.py --steps 300 --warmup 10 --ttq cfg1_v0.3 2>&1 | tail -1
timeout 600 python bench.py --impl reference --steps 20 --warmup 2 2>&1 | tail -1
