"""Feasibility projection (pathfair/projection.py API) on the GPU (csrc/projection.cu)."""

from __future__ import annotations

import numpy as np

from . import _abi as A
from ._lib import check, lib
from .model import Instance, InputError, _vec


def _p(a):
    return a.ctypes.data_as(A.f64p)


def score_paths(instance: Instance, rates, alpha):
    """projection.py:22-32: (commodity sum)^alpha x violated-edge count."""
    r = _vec(rates, instance.num_paths, "rates")
    out = np.empty(instance.num_paths)
    check(lib().pf_score_paths(instance.handle, _p(r), int(alpha), _p(out)))
    return out


def project(instance: Instance, rates, alpha):
    """projection.py:51-107: trimmed, exactly feasible rates."""
    x = np.ascontiguousarray(rates, np.float64)
    if x.shape != (instance.num_paths,):
        raise InputError(f"rates length {x.shape} does not match {instance.num_paths} paths")
    if not np.all(np.isfinite(x)):
        raise InputError("projection input contains non-finite rates")
    out = np.empty(instance.num_paths)
    if instance.num_paths:
        check(lib().pf_project(instance.handle, _p(x), int(alpha), _p(out)))
    return out
