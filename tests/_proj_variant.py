"""Subprocess helper for test_fast_projection_cluster_variants: the fast-mode
projection of a raw iterate under the PF_PROJ_CLUSTER set in the environment
(read once per process), and PF_PROJ_PIPE (pipelined cluster trim).  Prints a JSON line."""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2605_01748_b200 as pf  # noqa: E402
from b200_helpers import generated  # noqa: E402

n, k, its = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
topo, tab, ps = generated(n, k, 1.5)
inst = pf.build_instance(topo, tab, ps, device=0)
out = {}
for rep in range(2):
    s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
    s.run(its)
    x = s.x()
    alpha = int(s.state().alpha)
    rates, sums = s.finish()
    out.setdefault("digests", []).append(hashlib.sha256(rates.tobytes()).hexdigest())
exact = pf.project(inst, x, alpha)
ex_sums = pf.commodity_sums(inst, exact)
rep0 = pf.validate_allocation(inst, np.maximum(x, 0.0))
out.update(feasible=bool(pf.validate_allocation(inst, rates).feasible), infeasible_before=not rep0.feasible,
           max_edge_paths=int(np.max(np.diff(np.asarray(inst.edge_pair_ptr)))),
           sums_rel=float(np.max(np.abs(sums - ex_sums)) / max(1e-300, float(np.max(np.abs(ex_sums))))),
           deterministic=out["digests"][0] == out["digests"][1])
print(json.dumps(out))
