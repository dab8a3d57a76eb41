"""Small traced fast and exact solves + validate_allocation (memcheck target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

topo, tab, flat = bench.build_inputs("cfg1_v0.3")
inst = pf.build_instance_flat(topo, tab, flat, device=0)
for mode in ("fast", "exact"):
    r = pf.solve(inst, pf.SolverConfig(mode=mode, max_iterations=30, trace=True))
    print(mode, r.iterations, r.trace[-1].objective, r.trace[-1].mean_relative_violation)
print(pf.validate_allocation(inst, r.rates).feasible)
