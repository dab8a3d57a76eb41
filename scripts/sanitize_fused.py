"""Sanitizer target for the fused kernel's multi-tile path: a generated
instance with several tiles per CTA (set PF_FAST_TPS small), a few iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2605_01748_b200 as pf  # noqa: E402
from b200_helpers import generated  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 90
its = int(sys.argv[2]) if len(sys.argv) > 2 else 4
topo, tab, ps = generated(n, 8, 1.5)
inst = pf.build_instance(topo, tab, ps, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
s.run(its)
print("pairs", inst.num_pairs, "stats", s.kernel_stats(), "beta", s.result().beta, flush=True)
