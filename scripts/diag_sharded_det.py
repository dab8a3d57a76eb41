"""Diagnostic: is the sharded (peer-memory) trajectory deterministic?  N ranks
(torchrun, may share one GPU) run K iterations in one launch, `reps` times;
rank 0 prints a digest of the gathered rates and the controller state per rep
(identical digests = deterministic)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402
from paper_2605_01748_b200.distributed import ShardedSolver  # noqa: E402

name = sys.argv[1]
K = int(sys.argv[2])
reps = int(sys.argv[3])
chunk = int(sys.argv[4]) if len(sys.argv) > 4 else K
rank, world, local = bench.dist_env()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
if rank == 0:
    bench.build_inputs(name)
dist.barrier()
topo, tab, flat = bench.build_inputs(name)
for rep in range(reps):
    sh = ShardedSolver(topo, tab, flat, pf.SolverConfig(mode="fast", gamma=float(os.environ.get("DIAG_GAMMA", "1e-12")), max_iterations=10 ** 9), rank,
                       world, local)
    sh.init()
    dist.barrier()
    done = 0
    while done < K:
        sh.time_loop(min(chunk, K - done))
        done = min(K, done + chunk)
        if os.environ.get("DIAG_VERBOSE"):
            rr = sh.result()
            print(f"  rank {rank} rep {rep}: it={rr.iterations} a={rr.alpha} b={rr.beta:g} conv={rr.converged} "
                  f"st={rr.status}", flush=True)
        if sh.result().converged or sh.result().status:
            break
    r = sh.result()
    xg = sh.gather_x()
    if rank == 0:
        print(f"rep {rep}: it={r.iterations} a={r.alpha} b={r.beta:g} st={r.status} "
              f"x={hashlib.sha256(np.ascontiguousarray(xg).tobytes()).hexdigest()[:16]}", flush=True)
    del sh
    dist.barrier()
dist.destroy_process_group()
