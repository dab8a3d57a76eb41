"""Diagnostic: N ranks (torchrun, may share one GPU) run the north-star
instance for K iterations in ONE launch each (time_loop) vs a single-GPU solver;
prints the controller states, max |dx| and the post-projection quality of both."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402
from paper_2605_01748_b200.distributed import ShardedSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "target_k4_v0.3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4860
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
rank, world, local = bench.dist_env()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
if rank == 0:
    bench.build_inputs(name)
dist.barrier()
topo, tab, flat = bench.build_inputs(name)
meta, opt = bench.oracle_fixed_point(name)
full = pf.build_instance_flat(topo, tab, flat, device=local) if rank == 0 else None
if rank == 0:
    single = pf.Solver(full, pf.SolverConfig(mode="fast", max_iterations=5000)).init()
    single.time_loop(K)
    xs = single.x()
    rs = single.result()
    qs = pf.optimality_from_sums(pf.commodity_sums(full, pf.project(full, xs, int(rs.alpha))), opt,
                                 pf.default_theta(full))
    print(f"single: it={rs.iterations} a={rs.alpha} b={rs.beta:g} q={qs:.6f}", flush=True)
pre = None
if os.environ.get("DIAG_PRE"):  # an earlier sharded solver on another instance, kept alive (the bench's flow)
    t1, b1, f1 = bench.build_inputs(os.environ["DIAG_PRE"])
    pre = ShardedSolver(t1, b1, f1, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9), rank, world,
                        local)
    pre.init()
    pre.time_loop(30)
    if os.environ.get("DIAG_PRE_DEL"):
        del pre
        pre = None
    dist.barrier()
for rep in range(reps):
    sh = ShardedSolver(topo, tab, flat, pf.SolverConfig(mode="fast", max_iterations=5000), rank, world, local)
    sh.init()
    dist.barrier()
    sh.time_loop(K)
    r = sh.result()
    st = [None] * world
    dist.all_gather_object(st, (int(r.iterations), int(r.alpha), float(r.beta), int(r.status)))
    xg = sh.gather_x()
    if rank == 0:
        q = pf.optimality_from_sums(pf.commodity_sums(full, pf.project(full, xg, int(r.alpha))), opt,
                                    pf.default_theta(full))
        d = float(np.max(np.abs(xg - xs)) / max(float(np.max(np.abs(xs))), 1e-300))
        print(f"rep {rep}: ranks {st} q={q:.6f} max|dx|/max|x|={d:.3e}", flush=True)
    del sh
    dist.barrier()
dist.destroy_process_group()
