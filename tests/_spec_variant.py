"""Subprocess helper for test_speculated_rescale_bitwise: a fast solve's raw
iterate after N iterations under the PF_FAST_SPEC set in the environment (read
when the solver is created).  Prints a JSON line with digests."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2605_01748_b200 as pf  # noqa: E402
from b200_helpers import generated  # noqa: E402

n, k, its = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
topo, tab, ps = generated(n, k, 1.5)
inst = pf.build_instance(topo, tab, ps, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 6)).init()
s.run(its)
st = s.state()
dig = {f: hashlib.sha256(getattr(st, f).tobytes()).hexdigest()
       for f in ("x", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg")}
print(json.dumps({"digests": dig, "beta": st.beta, "iteration": st.iteration}))
