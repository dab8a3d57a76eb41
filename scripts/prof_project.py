"""Profile target: GPU projection of a raw cfg2 iterate (after N fused iterations)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 210
topo, tab, flat = bench.build_inputs(name)
inst = pf.build_instance_flat(topo, tab, flat, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
s.run(iters)
x = s.x()
st = s.state()
rep = pf.validate_allocation(inst, np.maximum(x, 0))
print(f"{name}: {iters} its, alpha {st.alpha}, violated edges {int((rep.edge_overload > 1e-9).sum())}, over-demand commodities {int((rep.commodity_excess > 1e-9).sum())}", flush=True)
for k in range(3):
    t = time.perf_counter()
    y = pf.project(inst, x, int(st.alpha))
    print(f"project: {1e3 * (time.perf_counter() - t):.2f} ms (host wall, includes H2D/D2H)", flush=True)
print("feasible:", pf.validate_allocation(inst, y).feasible)
