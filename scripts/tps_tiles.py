"""Tile count and settled per-iteration time for a tile size (PF_FAST_TPS)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
topo, tab, flat = bench.build_inputs(name)
inst = pf.build_instance_flat(topo, tab, flat, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
s.time_loop(1000)
ms, per = s.time_loop(300)
st = s.kernel_stats()
print(f"tps={os.environ.get('PF_FAST_TPS', 'default')} tiles={st['tiles']} grid={st['grid']} "
      f"tiles/cta={st['tiles'] / st['grid']:.2f} {per * 1e3:.1f} us/iter", flush=True)
