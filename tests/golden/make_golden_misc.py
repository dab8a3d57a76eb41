"""Golden vectors for the standalone reduction entry points, from the
UNMODIFIED reference:

* model.commodity_sums / edge_loads / edge_loads_from_pairs (model.py:297-319),
* _reduce.det_diff_norm (_reduce.py:118-128),
* projection.score_paths (projection.py:22-32) for alpha in {0, 1, 2},

on seeded inputs (uniform, with exact zeros and negative entries) over the
small builders and config 1 (cfg1_v0.3 instance from golden_arrays.npz), and
det_diff_norm over lengths that straddle its 32-element chunks and
4096-element blocks.  Run HERE (the reference imports):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden_misc.py

Output: tests/golden/golden_misc.npz.  Verbatim arrays (float64) -- the
tests compare bitwise.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from pathfair import _reduce, model, projection  # noqa: E402
import make_golden as MG  # noqa: E402

OUT = os.path.join(HERE, "golden_misc.npz")
DDN_LENGTHS = (0, 1, 31, 32, 33, 1000, 4095, 4096, 4097, 20011)


def inputs(rng, P, NP):
    x = rng.uniform(-0.5, 20.0, P)
    x[rng.random(P) < 0.15] = 0.0
    pv = rng.uniform(-1.0, 5.0, NP)
    return x, pv


def main():
    out = {}
    insts = {name: MG.instance_from_builder(fn, kw) for name, (fn, kw) in MG.small_instances().items()}
    A = dict(np.load(os.path.join(HERE, "golden_arrays.npz")))
    topo, coms, ps, _ = MG.gen_instance(40, 4, 0.3)
    insts["cfg1_v0.3"] = model.build_instance(topo, coms, ps)
    assert np.array_equal(insts["cfg1_v0.3"].capacity, A["cfg1_v0.3/in/capacity"])
    for tag, inst in insts.items():
        rng = np.random.default_rng(17 + len(tag))
        for trial in range(3):
            x, pv = inputs(rng, inst.num_paths, inst.num_pairs)
            if trial == 2:  # a feasible-ish point: scale down so few edges are violated
                x = np.abs(x) * 0.05
            key = f"{tag}/t{trial}"
            out[f"{key}/x"] = x
            out[f"{key}/pv"] = pv
            out[f"{key}/commodity_sums"] = model.commodity_sums(inst, x)
            out[f"{key}/edge_loads"] = model.edge_loads(inst, x)
            out[f"{key}/edge_loads_from_pairs"] = model.edge_loads_from_pairs(inst, pv)
            for a in (0, 1, 2):
                out[f"{key}/score_a{a}"] = projection.score_paths(inst, x, a)
    rng = np.random.default_rng(23)
    for n in DDN_LENGTHS:
        a = rng.normal(0, 1e3, n)
        b = a + rng.normal(0, 1.0, n) * (rng.random(n) < 0.5)
        out[f"ddn/{n}/a"] = a
        out[f"ddn/{n}/b"] = b
        out[f"ddn/{n}/out"] = np.array([_reduce.det_diff_norm(a, b)])
    np.savez_compressed(OUT, **out)
    print(f"wrote {len(out)} arrays to {OUT}")


if __name__ == "__main__":
    main()
