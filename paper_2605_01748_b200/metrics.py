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


def dao_carry_rates(rates, drifted_instance, tol=1e-9):
    """oracles.py:262-287: a stale allocation applied to drifted conditions, on
    the GPU and bitwise equal to the reference.  Commodity sums above the new
    demand scale down proportionally; then the most overloaded edge, worst
    first, scales all its paths by capacity over load until feasible (at most
    4 E + 4 passes).  With zero drift the rates come back bit-identical."""
    from ._abi import f64p
    from ._lib import check, lib
    import ctypes as C

    inst = drifted_instance
    x = np.ascontiguousarray(rates, np.float64)
    if x.shape != (inst.num_paths,):
        raise InputError(f"rates length {x.shape} does not match {inst.num_paths} paths")
    out = np.empty(inst.num_paths)
    passes = C.c_int64(0)
    if inst.num_paths:
        check(lib().pf_dao_carry_rates(inst.handle, x.ctypes.data_as(f64p), float(tol), out.ctypes.data_as(f64p),
                                       C.byref(passes)))
    return out


def dao_evaluate(allocation, drifted_instance, drifted_reference, theta):
    """oracles.py:290-297: drift-adjusted optimality -- carry the stale
    allocation into the drifted state, then score it against the reference
    solved there."""
    from .model import commodity_sums

    carried = dao_carry_rates(allocation.rates, drifted_instance)
    return optimality_from_sums(commodity_sums(drifted_instance, carried), drifted_reference.sums, theta)
