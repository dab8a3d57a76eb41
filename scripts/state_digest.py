"""Digest of the fast solver's state after N iterations (compare two library
revisions: python scripts/state_digest.py CFG N vs python _r1/scripts/...)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
topo, tab, flat = bench.build_inputs(name)
inst = pf.build_instance_flat(topo, tab, flat, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
s.run(n)
st = s.state()
h = hashlib.sha256()
for f in ("x", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg"):
    h.update(getattr(st, f).tobytes())
print(name, n, st.beta, h.hexdigest()[:16])
