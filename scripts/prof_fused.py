"""Profile target: one k_fused launch of N iterations on config 2 (run under ncu)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
topo, tab, flat = bench.build_inputs(name)
inst = pf.build_instance_flat(topo, tab, flat, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
s.time_loop(3)            # launch 2 (k_fused): warm-up
ms, per = s.time_loop(iters)  # launch 3 (k_fused): profiled
print(f"{name}: {iters} iterations, {ms:.3f} ms, {per * 1e3:.1f} us/iter", flush=True)
