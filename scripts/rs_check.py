"""Run-slot layout vs the per-CTA edge-table layout on one instance: the fast
trajectories after N iterations (same algorithm, different association of the
per-edge sums: close, not bitwise) and the settled per-iteration times.
    python scripts/rs_check.py CFG N"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 3:  # child: one layout
    sys.path.insert(0, ROOT)
    import bench  # noqa: E402
    import paper_2605_01748_b200 as pf  # noqa: E402
    name, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    topo, tab, flat = bench.build_inputs(name)
    inst = pf.build_instance_flat(topo, tab, flat, device=0)
    s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
    s.time_loop(n)
    x = s.x()
    ms, per = s.time_loop(20)
    st = s.kernel_stats()
    np.save(out, x)
    print(f"{name} PF_FAST_RS={os.environ.get('PF_FAST_RS')}: {per * 1e3:.1f} us/iter settled, "
          f"bytes/iter {st['bytes_per_iter']}, tiles {st['tiles']}, grid {st['grid']}", flush=True)
    sys.exit(0)
name, n = sys.argv[1], int(sys.argv[2])
xs = []
for rs in ("0", "1"):
    out = f"/tmp/rs_{name}_{rs}.npy"
    subprocess.run([sys.executable, __file__, name, str(n), out], env=dict(os.environ, PF_FAST_RS=rs), check=True)
    xs.append(np.load(out))
a, b = xs
d = np.abs(a - b) / np.maximum(np.abs(a), 1e-9)
print(f"{name}: after {n} iterations max rel diff {d.max():.3e}, median {np.median(d):.3e}; "
      f"sum rel diff {abs(a.sum() - b.sum()) / abs(a.sum()):.3e}")
