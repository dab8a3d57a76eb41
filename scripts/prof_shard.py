"""Per-GPU work of an N-way sharded run, timed on one GPU: the fused loop over
shard `r` of `n` (the commodity range distributed.partition gives rank r)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402
from paper_2605_01748_b200 import distributed as D  # noqa: E402

name, n, r = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 0
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 200
topo, tab, flat = bench.build_inputs(name)
lo, hi = D.partition(D.pair_counts(tab, flat), n)[r]
stab, sflat = D.shard_inputs(tab, flat, lo, hi)
inst = pf.build_instance_flat(topo, stab, sflat, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
s.time_loop(5)
ms, _ = s.time_loop(iters)
st = s.kernel_stats()
print(f"{name} shard {r}/{n}: pairs {inst.num_pairs}, tiles {st['tiles']}, grid {st['grid']}: "
      f"{1e3 * ms / iters:.1f} us/iter", flush=True)
