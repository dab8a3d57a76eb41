"""Where the time of one end-to-end pf.solve goes (config 2, warm start, K iterations)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
topo, tab, flat = bench.build_inputs("cfg2")
inst = pf.build_instance_flat(topo, tab, flat, device=0)
s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
s.run(20)
warm = s.x()
cfg = pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=K)
for _ in range(2):
    pf.solve(inst, cfg, warm_start=warm)
t = time.perf_counter()
r = pf.solve(inst, cfg, warm_start=warm)
tot = time.perf_counter() - t
print(f"pf.solve K={K}: {1e3 * tot:.1f} ms wall; loop {r.loop_ms:.1f} ms, projection {r.projection_ms:.1f} ms, "
      f"runtime_s {1e3 * r.runtime_s:.1f} ms", flush=True)
t = time.perf_counter()
np.all(np.isfinite(warm))
print(f"isfinite(warm): {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)

# split: Python wrapper vs the pf_solve call vs runtime_s
import ctypes as C  # noqa: E402

from paper_2605_01748_b200 import _abi as A  # noqa: E402
from paper_2605_01748_b200._lib import lib  # noqa: E402
from paper_2605_01748_b200.controller import _p  # noqa: E402

keep = []
c = cfg.to_c(keep=keep)
rates = np.empty(inst.num_paths)
sums = np.empty(inst.num_commodities)
res = A.Result()
tb = (A.TraceRow * 1)()
tl = C.c_int64(0)
w = warm.copy()
for rep in range(2):
    t = time.perf_counter()
    rc = lib().pf_solve(inst.handle, C.byref(c), _p(w), _p(rates), _p(sums), C.byref(res), tb, 0, C.byref(tl))
    dt = time.perf_counter() - t
    print(f"pf_solve call: {1e3 * dt:.1f} ms, runtime_s {1e3 * res.runtime_s:.1f} ms, loop {res.loop_ms:.1f}, "
          f"projection {res.projection_ms:.1f} (rc {rc})", flush=True)
