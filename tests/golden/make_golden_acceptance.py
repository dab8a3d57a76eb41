"""Goldens for acceptance criteria 2 and 7 (reference tests/test_acceptance.py:
117-166 and 331-365): the reference's exhaustive grid oracle
`oracles.exact_bruteforce_tiny` (oracles.py:158) on the reference's own
instance families, with the instances' flat inputs, so the GPU tests can run
the same checks at the same thresholds without the reference present.

Run HERE (the reference imports):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden_acceptance.py

Output: tests/golden/golden_acceptance.npz.
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

import test_acceptance as TA  # noqa: E402  (the reference's acceptance suite: builders only)
from pathfair.oracles import exact_bruteforce_tiny  # noqa: E402
import make_golden as MG  # noqa: E402

OUT = os.path.join(HERE, "golden_acceptance.npz")


def flat(inst):
    f = MG.flat_from_instance(inst)
    return {k: f[k] for k in ("capacity", "demand0", "com_path_ptr0", "path_edge_ptr0", "path_edges0")}


def main():
    out = {}
    for i, inst in enumerate(TA.tiny_multipath_family()):
        for k, v in flat(inst).items():
            out[f"c2/{i}/in/{k}"] = v
        step = 0.01 * float(inst.demand.max())
        out[f"c2/{i}/step"] = np.array([step])
        for alpha in (0, 1, 2):
            out[f"c2/{i}/a{alpha}/ref_sums"] = exact_bruteforce_tiny(inst, alpha, step).sums
    family = [("sym", TA.shared_edge(2, cap=10.0, demand=20.0)), ("sym", TA.shared_edge(3, cap=9.0, demand=20.0)),
              ("sym", TA.diamond(20.0, 5.0, 5.0)), ("asym", TA.two_unequal(10.0, 2.0, 20.0)),
              ("asym", TA.diamond(20.0, 4.0, 8.0))]
    for i, (tag, inst) in enumerate(family):
        for k, v in flat(inst).items():
            out[f"c7/{i}/in/{k}"] = v
        step = 0.01 * float(inst.demand.max())
        out[f"c7/{i}/step"] = np.array([step])
        out[f"c7/{i}/sym"] = np.array([tag == "sym"])
        out[f"c7/{i}/ref_sums"] = exact_bruteforce_tiny(inst, None, step).sums
    np.savez_compressed(OUT, **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
