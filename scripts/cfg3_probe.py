"""Config 3 probe: native path generation, GPU incidence build and fused-kernel
iterations on one B200 (bounded: prints timings as it goes)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
t = time.perf_counter()
topo, tab, flat = bench.build_inputs(name)
print(f"{name}: generated C={len(tab)} P={len(flat.path_edge_ptr) - 1} NP={len(flat.path_edges)} "
      f"in {time.perf_counter() - t:.1f}s", flush=True)
t = time.perf_counter()
inst = pf.build_instance_flat(topo, tab, flat, device=0)
print(f"build_instance {time.perf_counter() - t:.1f}s: C={inst.num_commodities} P={inst.num_paths} "
      f"E={inst.num_edges} NP={inst.num_pairs}", flush=True)
t = time.perf_counter()
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
print(f"fast solver init (tile layout) {time.perf_counter() - t:.1f}s stats {s.kernel_stats()}", flush=True)
s.time_loop(3)
ms, per = s.time_loop(iters)
b_iter = 36 * inst.num_pairs + 40 * inst.num_paths + 32 * inst.num_commodities + 32 * inst.num_edges
print(f"{name}: {iters} iterations {ms:.1f} ms = {1e3 * ms / iters:.0f} us/iter, "
      f"algorithmic {b_iter / 1e9:.2f} GB/iter -> {b_iter * iters / ms / 1e6:.0f} GB/s", flush=True)
