"""Evaluation metrics reused from the reference (pathfair/oracles.py:51-53, 244-259).

These are scalar host metrics over per-commodity sums (not part of the
iterate path); they define the time-to-within-1% measurement.
"""

from __future__ import annotations

import numpy as np

from .topology import InputError


def default_theta(instance):
    dmax = float(instance.demand.max()) if instance.num_commodities else 0.0
    return 1e-6 * (dmax if dmax > 0 else 1.0)


def optimality_from_sums(sums, reference_sums, theta):
    if theta <= 0:
        raise InputError("theta must be > 0")
    sums = np.asarray(sums, np.float64)
    reference_sums = np.asarray(reference_sums, np.float64)
    if sums.shape != reference_sums.shape:
        raise InputError("commodity sets differ between allocation and reference")
    if sums.size == 0:
        return 1.0
    ratios = np.minimum(sums / np.maximum(reference_sums, theta), 1.0)
    return float(ratios.mean())
