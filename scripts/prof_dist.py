"""World-1 NCCL timing of the sharded (multi-GPU) solver path: graph-driven vs
host-driven iteration loop, against the single-GPU fused kernel."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402
from paper_2605_01748_b200 import distributed as D  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
s = socket.socket()
s.bind(("127.0.0.1", 0))
port = s.getsockname()[1]
s.close()
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
topo, tab, flat = bench.build_inputs(name)
cfg = pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)
xs = {}
for mode in ("ipc", "graph", "host"):
    if mode == "host":
        os.environ["PF_DIST_NO_GRAPH"] = "1"
    sh = D.ShardedSolver(topo, tab, flat, cfg, 0, 1, 0, transport="ipc" if mode == "ipc" else "nccl").init()
    sh.time_loop(5)
    ms, _ = sh.time_loop(iters)
    st = sh.solver.kernel_stats()
    print(f"{name} dist-{mode}: {iters} its {ms:.2f} ms = {1e3 * ms / iters:.1f} us/iter, launches {st['launches']}",
          flush=True)
    xs[mode] = sh.local_x()
print("graph == host bitwise:", bool(np.array_equal(xs["graph"], xs["host"])))
xs_ipc = xs["ipc"]
inst = pf.build_instance_flat(topo, tab, flat, device=0)
f = pf.Solver(inst, cfg).init()
f.time_loop(5)
ms, _ = f.time_loop(iters)
print(f"{name} fused: {iters} its {ms:.2f} ms = {1e3 * ms / iters:.1f} us/iter", flush=True)
print("ipc == single-GPU fused bitwise:", bool(np.array_equal(xs_ipc, f.x())))
dist.destroy_process_group()
