"""Seeded random solver states shared by the fixture generator and the tests.

`random_state` draws exactly the arrays the reference's tests/helpers.py:65-89
`random_state` draws, in the same rng call order, so a seed reproduces the
fixture inputs without storing them.
"""

import numpy as np

FIELDS = ("x", "y", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg",
          "slack_demand", "slack_capacity")


def random_state(C, P, E, NP, rng, rate_scale=5.0, dual_scale=1.0, nonneg_floor=False):
    x = rng.uniform(0.0, rate_scale, P)
    dn = np.zeros(P)
    if nonneg_floor:
        dn = rng.uniform(0.0, dual_scale, P)
    return dict(
        x=x,
        y=rng.uniform(0.0, rate_scale, NP),
        dual_demand=rng.uniform(0.0, dual_scale, C),
        dual_capacity=rng.uniform(0.0, dual_scale, E),
        dual_consensus=rng.uniform(0.0, dual_scale, NP),
        dual_nonneg=dn,
        slack_demand=rng.uniform(0.0, dual_scale, C),
        slack_capacity=rng.uniform(0.0, dual_scale, E),
    )


def kernel_case_states(C, P, E, NP, seed, n_states=4):
    """The states used by the per-kernel fixtures: list of (arrays, beta, alpha)."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_states):
        alpha = [0, 1, 2, 4][i % 4]
        beta = float(rng.uniform(0.3, 3.0))
        arrs = random_state(C, P, E, NP, rng, nonneg_floor=bool(i % 2))
        if i >= 2:  # signed rates exercise the non-negativity force
            arrs["x"] = rng.uniform(-2.0, 5.0, P)
        out.append((arrs, beta, alpha))
    return out
