"""Diagnostic: exact vs fast convergence on the smoke instance (24 nodes, k=4, V=0.3)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_01748_b200 as pf  # noqa: E402
from oracle import oracle as O  # noqa: E402

topo = pf.random_topology(24, seed=24)
tab = pf.gravity_table(topo, 0.3 * float(topo.capacity.sum()))
ps = pf.k_shortest_paths(topo, tab, 4)
inst = pf.build_instance(topo, tab, ps, device=0)
for at in (1, None, 0, 2):
    ex = pf.solve(inst, pf.SolverConfig(mode="exact", alpha_target=at, trace=True))
    fa = pf.solve(inst, pf.SolverConfig(mode="fast", alpha_target=at, trace=True))
    print(f"alpha_target={at}: exact it={ex.iterations} a={ex.alpha} conv={ex.converged}; "
          f"fast it={fa.iterations} a={fa.alpha} conv={fa.converged}")
    for lab, r in (("exact", ex), ("fast", fa)):
        tr = r.trace
        idx = sorted(set([0, 1, 2, 10, 50, 100, 200, 500, 1000, 2000, 4999, len(tr) - 1]) & set(range(len(tr))))
        print("  ", lab, [(tr[i].iteration, tr[i].alpha, f"{tr[i].beta:.3g}", f"{tr[i].s:.2e}", f"{tr[i].r:.2e}") for i in idx])
    want = np.sort(ex.sums)
    got = np.sort(fa.sums)
    print("   max |rel| sorted sums", float(np.max(np.abs(got - want) / np.maximum(want, 1e-12))),
          "scaled", float(np.max(np.abs(got - want))) / float(want.max()))
