"""Two ranks of the peer-memory transport on ONE GPU (two processes, world size
2, both on device 0): exercises the cross-rank exchange (slots, counters,
parities, rank-order sums) for real.  The two cooperative kernels are
time-sliced by the driver, so iterations are slow; the check is correctness:
identical controller state on both ranks and a feasible projected result close
to the single-GPU solve at the same iteration count."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port, iters, q):
    import numpy as np
    import torch.distributed as dist

    import paper_2605_01748_b200 as pf
    from paper_2605_01748_b200 import distributed as D
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    topo = pf.random_topology(24, seed=24)
    tab = pf.gravity_table(topo, 0.3 * float(topo.capacity.sum()))
    flat = pf.k_shortest_paths(topo, tab, 4)
    cfg = pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 6)
    sh = D.ShardedSolver(topo, tab, flat, cfg, rank, world, 0, transport="ipc").init()
    sh.run(iters)
    r = sh.result()
    x = sh.gather_x()
    out = None
    if rank == 0:
        inst = pf.build_instance_flat(topo, tab, flat, device=0)
        single = pf.Solver(inst, cfg).init()
        single.run(iters)
        out = (np.asarray(x), single.x())
    q.put((rank, int(r.iterations), float(r.beta), int(r.alpha), out))
    dist.destroy_process_group()


if __name__ == "__main__":
    import numpy as np
    import torch.multiprocessing as mp
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, iters, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
    res.sort()
    print("ranks:", [(r, it, b, a) for r, it, b, a, _ in res], flush=True)
    assert res[0][1:4] == res[1][1:4], "ranks diverged"
    xg, xs = res[0][4]
    rel = float(np.max(np.abs(xg - xs)) / max(1e-12, float(np.max(np.abs(xs)))))
    print(f"two-rank IPC vs single GPU after {iters} iterations: max |dx| / max|x| = {rel:.2e}", flush=True)
    assert rel < 1e-6, rel
    print("OK", flush=True)
