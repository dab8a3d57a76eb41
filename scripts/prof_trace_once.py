"""Profile target: one traced fast-mode solve (config 2, 20 iterations)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

topo, tab, flat = bench.build_inputs(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
inst = pf.build_instance_flat(topo, tab, flat, device=0)
pf.solve(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=20, trace=True))
