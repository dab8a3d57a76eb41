"""Diagnostic: is the single-GPU fused solver bitwise deterministic when two
processes share one GPU (time-sliced)?  Rank 0 first runs alone, then every
rank runs the same K iterations concurrently; each prints a digest of x."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "target_k4_v0.3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
rank, world, local = bench.dist_env()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
if rank == 0:
    bench.build_inputs(name)
dist.barrier()
topo, tab, flat = bench.build_inputs(name)
full = pf.build_instance_flat(topo, tab, flat, device=local)


def once():
    s = pf.Solver(full, pf.SolverConfig(mode="fast", max_iterations=10 ** 9, gamma=1e-12)).init()
    s.run(K)
    r = s.result()
    return f"it={r.iterations} a={r.alpha} b={r.beta:g} x={hashlib.sha256(np.ascontiguousarray(s.x()).tobytes()).hexdigest()[:16]}"


if rank == 0:
    print("solo  :", once(), flush=True)
dist.barrier()
for rep in range(int(os.environ.get("REPS", "2"))):
    d = once()
    print(f"shared rank {rank} rep {rep}:", d, flush=True)
    dist.barrier()
dist.destroy_process_group()
