"""Sanitizer target: every kernel family on small instances -- fused fast
solve + cluster projection, exact solve + bitwise projection, validation,
kernel-level entry points.  Run under compute-sanitizer (memcheck / racecheck
/ synccheck)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2605_01748_b200 as pf  # noqa: E402
from b200_helpers import generated  # noqa: E402

its = int(sys.argv[1]) if len(sys.argv) > 1 else 20
topo, tab, ps = generated(40, 4, 1.5)
inst = pf.build_instance(topo, tab, ps, device=0)
r = pf.solve(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=its))
print("fast", r.iterations, pf.validate_allocation(inst, r.rates).feasible, flush=True)
r2 = pf.solve(inst, pf.SolverConfig(mode="exact", gamma=1e-12, max_iterations=its))
print("exact", r2.iterations, pf.validate_allocation(inst, r2.rates).feasible, flush=True)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
s.run(its)
x = s.x()
y = pf.project(inst, x, int(s.state().alpha))
print("project", pf.validate_allocation(inst, y).feasible, float(np.sum(y)), flush=True)
