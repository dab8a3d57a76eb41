"""Diagnostic: sharded (torchrun, ranks may share one GPU) vs single-GPU
trajectory quality on the north-star instance at a few checkpoints."""
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
rank, world, local = bench.dist_env()
torch.cuda.set_device(local)
dist.init_process_group("gloo")
if rank == 0:
    bench.build_inputs(name)
dist.barrier()
topo, tab, flat = bench.build_inputs(name)
meta, opt = bench.oracle_fixed_point(name)
pre = None
if os.environ.get("DIAG_PRE"):  # an earlier sharded solver on another instance (the bench's flow)
    t1, b1, f1 = bench.build_inputs(os.environ["DIAG_PRE"])
    pre = ShardedSolver(t1, b1, f1, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9), rank, world,
                        local)
    pre.init()
    pre.time_loop(30)
    dist.barrier()
sh = ShardedSolver(topo, tab, flat, pf.SolverConfig(mode="fast", max_iterations=5000), rank, world, local)
sh.init()
after = os.environ.get("DIAG_SINGLE_AFTER") == "1"  # rank 0's single-GPU objects only after the sharded run
full = single = theta = None


def make_single():
    global full, single, theta
    full = pf.build_instance_flat(topo, tab, flat, device=local)
    single = pf.Solver(full, pf.SolverConfig(mode="fast", max_iterations=5000)).init()
    theta = pf.default_theta(full)


if rank == 0 and not after:
    make_single()
done = 0
for k in [int(v) for v in os.environ.get("DIAG_KS", "10,100,1000,2500,4860").split(",")]:
    sh.run(k - done)
    if rank == 0:
        if single is None:
            make_single()
            single.run(k)
        else:
            single.run(k - done)
    done = k
    r = sh.result()
    if r.status:
        print(f"rank {rank}: status {r.status} at iteration {r.iterations}", flush=True)
    xg = sh.gather_x()
    if rank == 0:
        rs = single.result()
        xs = single.x()
        qa = pf.optimality_from_sums(pf.commodity_sums(full, pf.project(full, xg, int(r.alpha))), opt, theta)
        qb = pf.optimality_from_sums(pf.commodity_sums(full, pf.project(full, xs, int(rs.alpha))), opt, theta)
        d = np.abs(xg - xs).max() / max(np.abs(xs).max(), 1e-300)
        print(f"k={k}: sharded it={r.iterations} a={r.alpha} b={r.beta:g} q={qa:.6f} | single it={rs.iterations} "
              f"a={rs.alpha} b={rs.beta:g} q={qb:.6f} | max|dx|/max|x| {d:.3e}", flush=True)
dist.barrier()
dist.destroy_process_group()
