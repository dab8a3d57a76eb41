"""Speculated rescale factor vs always-1 (PF_FAST_SPEC=1/0, two processes): the
fast iterates after N iterations must be bitwise equal (a correct prediction
skips the rollback pass, a wrong one falls back to it), and the timings."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 4:
    sys.path.insert(0, ROOT)
    import bench  # noqa: E402
    import paper_2605_01748_b200 as pf  # noqa: E402
    name, n, out = sys.argv[1], int(sys.argv[2]), sys.argv[4]
    topo, tab, flat = bench.build_inputs(name)
    inst = pf.build_instance_flat(topo, tab, flat, device=0)
    s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
    ms, per = s.time_loop(n)
    st = s.state()
    np.savez(out, x=st.x, dcon=st.dual_consensus, dn=st.dual_nonneg, dd=st.dual_demand, dc=st.dual_capacity)
    print(f"{name} PF_FAST_SPEC={os.environ.get('PF_FAST_SPEC')}: {n} its from cold {ms:.2f} ms "
          f"({per * 1e3:.1f} us/it), beta {st.beta:g}", flush=True)
    sys.exit(0)
name, n = sys.argv[1], int(sys.argv[2])
vals = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1"]
outs = []
for v in vals:
    o = f"/tmp/spec_{len(outs)}.npz"
    subprocess.run([sys.executable, __file__, name, str(n), "child", o], env=dict(os.environ, PF_FAST_SPEC=v),
                   check=True)
    outs.append(np.load(o))
for i in range(1, len(outs)):
    print(name, vals[0], "vs", vals[i], "bitwise equal:", all(np.array_equal(outs[0][k], outs[i][k]) for k in outs[0].files),
          {k: float(np.max(np.abs(outs[0][k] - outs[i][k]))) for k in outs[0].files})
