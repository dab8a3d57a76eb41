"""Run bench.py's multi-GPU code path (distributed.bench_main) at world size 1
(it is what `bench.py --gpus N` runs for N > 1 under torchrun)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
os.environ.setdefault("LOCAL_RANK", "0")
import argparse  # noqa: E402

import bench  # noqa: E402
from paper_2605_01748_b200 import distributed as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--config", default="cfg2")
a = ap.parse_args()
a.gpus = 1
sys.exit(D.bench_main(a, bench))
