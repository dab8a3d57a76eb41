"""Fused-loop timing after a warm-up of W untimed iterations (beta settled, so
rollback passes are rare): python scripts/prof_fused_warm.py CFG W N.  Prints
the timing and the beta changes seen in the timed window (trace rows)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

name, W, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
topo, tab, flat = bench.build_inputs(name)
inst = pf.build_instance_flat(topo, tab, flat, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
s.time_loop(W)
b0 = s.result().beta
ms, per = s.time_loop(N)
r = s.result()
print(f"{name}: after {W}, {N} iterations {ms:.3f} ms, {per * 1e3:.1f} us/iter (beta {b0:g} -> {r.beta:g}, "
      f"alpha {r.alpha}; grid {s.kernel_stats()['grid']}, tiles {s.kernel_stats()['tiles']})", flush=True)
