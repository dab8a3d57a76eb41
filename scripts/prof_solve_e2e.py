"""Profile target: end-to-end fast-mode pf.solve of config 2 (warm start, K
iterations, fast GPU projection), repeated: the first solve builds the
projection workspace, the later ones are the steady state.  With ncu this
lists every launch of the solves (scripts/launch_sum.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
topo, tab, flat = bench.build_inputs("cfg2")
inst = pf.build_instance_flat(topo, tab, flat, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
s.run(20)
warm = s.x()
for _ in range(reps):
    r = pf.solve(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=K), warm_start=warm)
    print(f"loop {r.loop_ms:.1f} ms projection {r.projection_ms:.2f} ms runtime {1e3 * r.runtime_s:.1f} ms "
          f"feasible {pf.validate_allocation(inst, r.rates).feasible}", flush=True)
import time  # noqa: E402

for _ in range(2):
    t0 = time.perf_counter()
    rep = pf.validate_allocation(inst, r.rates)
    print(f"validate_allocation: {1e3 * (time.perf_counter() - t0):.2f} ms (feasible {rep.feasible})", flush=True)
