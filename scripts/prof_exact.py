"""Exact-mode (reference operation order) iterations/s on a config."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
topo, tab, flat = bench.build_inputs(name)
inst = pf.build_instance_flat(topo, tab, flat, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="exact", gamma=1e-12, max_iterations=10 ** 9)).init()
s.run(2)
t = time.perf_counter()
s.run(iters)
dt = time.perf_counter() - t
print(f"{name} exact mode: {iters} iterations {1e3 * dt:.1f} ms = {1e3 * dt / iters:.2f} ms/iter", flush=True)
