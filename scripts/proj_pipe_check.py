"""Pipelined cluster trim vs the plain cluster trim (PF_PROJ_PIPE=0/1 in two
processes): bitwise-equal fast-mode solves (rates after the GPU projection) at
config 2 after K iterations, and their projection times."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 2:
    sys.path.insert(0, ROOT)
    import bench  # noqa: E402
    import paper_2605_01748_b200 as pf  # noqa: E402
    K, out = int(sys.argv[1]), sys.argv[2]
    topo, tab, flat = bench.build_inputs("cfg2")
    inst = pf.build_instance_flat(topo, tab, flat, device=0)
    s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
    s.run(20)
    warm = s.x()
    for _ in range(3):
        r = pf.solve(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=K), warm_start=warm)
        print(f"PF_PROJ_PIPE={os.environ.get('PF_PROJ_PIPE')}: projection {r.projection_ms:.2f} ms, "
              f"feasible {pf.validate_allocation(inst, r.rates).feasible}", flush=True)
    np.save(out, r.rates)
    sys.exit(0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
xs = []
for v in ("0", "1"):
    o = f"/tmp/pp_{v}.npy"
    subprocess.run([sys.executable, __file__, str(K), o], env=dict(os.environ, PF_PROJ_PIPE=v), check=True)
    xs.append(np.load(o))
print("bitwise equal:", bool(np.array_equal(xs[0], xs[1])))
