"""Cost of trace=True: pf.solve of config 2 with and without the per-iteration trace."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
topo, tab, flat = bench.build_inputs(name)
inst = pf.build_instance_flat(topo, tab, flat, device=0)
for trace in (False, True, False, True):
    t = time.perf_counter()
    r = pf.solve(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=K, trace=trace))
    dt = time.perf_counter() - t
    print(f"{name} trace={trace}: {K} iterations {1e3 * dt:.1f} ms wall ({1e3 * dt / K:.3f} ms/it), loop "
          f"{r.loop_ms:.1f} ms, rows {len(r.trace) if r.trace else 0}", flush=True)
