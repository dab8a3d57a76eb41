"""The reference algorithm's own fixed points on the benchmarked instances
(SURVEY 8(d) time-to-1%), computed with the C oracle (oracle/pf_oracle.c:
the reference's exact fp64 operation order, pinned to the reference by
tests/golden/make_golden.py).

For each instance (cfg1 / the north-star 500-node k=4 / config 2, all at
V = 0.3 x total capacity, the reference's default SolverConfig, 5,000-iteration cap):

* the oracle solve (controller.py:197-284): iterations, alpha, converged, the
  digest of the raw iterate and of the projected rates, and the post-projection
  commodity sums = OPT_ref (stored verbatim: bench.py's time-to-1% and the GPU
  parity tests read them);
* the oracle trajectory's own k*: the first iteration k whose post-projection
  optimality_from_sums(S_k, OPT_ref, default_theta) >= 0.99
  (oracles.py:51-53, 244-254; controller.py:173-194), found on checkpoints
  every 50 iterations and bisected inside the crossing interval;
* the optimality curve at the checkpoints.

Instances are built with this package's generators (random_topology /
gravity_table pinned bitwise, the native KSP pinned to networkx on all of
config 2 by tests/golden/golden_ksp.json).  Run here (CPU; ~1 h on 8 cores):

    python tests/golden/make_golden_fixed_points.py [names...]

Output: tests/golden/golden_fixed_points.npz (+ .json).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
import paper_2605_01748_b200 as pf  # noqa: E402  (generators + metrics only)

INSTANCES = {"cfg1_v0.3": (40, 4, 0.3), "target_k4_v0.3": (500, 4, 0.3), "cfg2_v0.3": (500, 8, 0.3)}
CK = 50
OUT_NPZ = os.path.join(HERE, "golden_fixed_points.npz")
OUT_JSON = os.path.join(HERE, "golden_fixed_points.json")


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        a = a + 0.0
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]


def oracle_instance(n, k, vol):
    topo = pf.random_topology(n, seed=n)
    tab = pf.gravity_table(topo, vol * float(topo.capacity.sum()))
    flat = pf.k_shortest_paths(topo, tab, k)
    return O.build_instance(topo.capacity, tab.demand, flat.com_path_ptr, flat.path_edge_ptr, flat.path_edges)


def quality(I, x, alpha, opt, theta):
    return pf.optimality_from_sums(O.commodity_sums(I, O.project(I, x, alpha)), opt, theta)


def run(name):
    n, k, vol = INSTANCES[name]
    t0 = time.perf_counter()
    I = oracle_instance(n, k, vol)
    cfg = O.make_config(max_iterations=5000)
    loop = O.Loop(I, cfg)
    snaps = []  # (iteration, x, alpha)
    while not loop.stopped:
        it0 = loop.state().iteration if snaps else 0
        loop.step(CK)
        st = loop.state()
        if st.iteration == it0:
            break
        snaps.append((st.iteration, st.x, st.alpha))
        if st.iteration >= cfg.max_iterations:
            break
    st = loop.state()
    rates = O.project(I, st.x, st.alpha)
    opt = O.commodity_sums(I, rates)
    theta = 1e-6 * (float(I.demand.max()) if I.num_commodities else 1.0)
    print(f"[{name}] solve: {st.iteration} its alpha={st.alpha} stopped={loop.stopped} "
          f"{time.perf_counter() - t0:.0f}s", flush=True)
    curve = []
    hi = None
    for it, x, a in snaps:
        q = quality(I, x, a, opt, theta)
        curve.append((it, q))
        if q >= 0.99:
            hi = it
            break
    lo = 0 if hi is None or len(curve) < 2 else curve[-2][0]
    kstar = hi
    if hi is not None and hi - lo > 1:
        # replay to lo, keep every iterate of (lo, hi], bisect (quality is monotone in practice)
        loop2 = O.Loop(I, cfg)
        if lo:
            loop2.step(lo)
        xs = {}
        for it in range(lo + 1, hi + 1):
            loop2.step(1)
            s2 = loop2.state()
            xs[it] = (s2.x, s2.alpha)
        a_, b_ = lo, hi
        while b_ - a_ > 1:
            mid = (a_ + b_) // 2
            if quality(I, xs[mid][0], xs[mid][1], opt, theta) >= 0.99:
                b_ = mid
            else:
                a_ = mid
        kstar = b_
    meta = {"nodes": n, "k": k, "volume_fraction": vol, "commodities": I.num_commodities, "paths": I.num_paths,
            "pairs": I.num_pairs, "edges": I.num_edges, "iterations": int(st.iteration), "alpha": int(st.alpha),
            "converged": bool(loop.stopped), "cap_limited": not bool(loop.stopped), "k_star": kstar,
            "theta": theta, "raw_x_digest": digest(st.x), "rates_digest": digest(rates),
            "opt_digest": digest(opt), "oracle_threads": O.num_threads(),
            "seconds": time.perf_counter() - t0}
    print(f"[{name}] k*={kstar} ({time.perf_counter() - t0:.0f}s)", flush=True)
    return meta, opt, np.array(curve, np.float64)


def main(argv):
    names = argv or list(INSTANCES)
    arrays = dict(np.load(OUT_NPZ)) if os.path.exists(OUT_NPZ) else {}
    meta = json.load(open(OUT_JSON)) if os.path.exists(OUT_JSON) else {}
    for name in names:
        m, opt, curve = run(name)
        meta[name] = m
        arrays[f"{name}/opt_sums"] = opt
        arrays[f"{name}/curve"] = curve
        np.savez_compressed(OUT_NPZ, **arrays)
        with open(OUT_JSON, "w") as fh:
            json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
