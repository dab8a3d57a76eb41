"""Iterate kernels (pathfair/kernels.py API), executed by the exact-order CUDA
kernels in csrc/exact.cu through the C-ABI.

Each function is a pure function of (state, instance) returning fresh numpy
arrays, like the reference.  The state is uploaded, the kernel runs on the
instance's GPU, the result is copied back.  For alpha in {0, 1} the outputs are
bit-identical to the reference; for alpha >= 2 the roots use CUDA `pow`
(<= 2 ulp) where the reference mixes glibc and numpy SIMD `pow`.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi as A
from ._lib import NativeError, check, last_error, lib
from .model import InputError, Instance, _vec, default_device


class KernelError(RuntimeError):
    """Non-finite coefficients or roots during an iterate computation (kernels.py:20-21)."""


@dataclass
class SolverState:
    """Mutable iterate arrays plus the scalar knobs the controller drives (kernels.py:24-44)."""

    x: np.ndarray
    y: np.ndarray
    dual_demand: np.ndarray
    dual_capacity: np.ndarray
    dual_consensus: np.ndarray
    dual_nonneg: np.ndarray
    slack_demand: np.ndarray
    slack_capacity: np.ndarray
    beta: float
    alpha: int
    iteration: int


def utility(sums, alpha):
    """kernels.py:47-66 (host numpy; a metric, not on the iterate path)."""
    arr = np.asarray(sums, dtype=np.float64)
    scalar = arr.ndim == 0
    arr = np.atleast_1d(arr)
    if alpha == 0:
        out = arr - 1.0
    else:
        out = np.full(arr.shape, -np.inf)
        pos = arr > 0
        if alpha == 1:
            out[pos] = np.log(arr[pos])
        else:
            out[pos] = (arr[pos] ** (1.0 - alpha) - 1.0) / (1.0 - alpha)
    return float(out[0]) if scalar else out


def _p(a):
    return a.ctypes.data_as(A.f64p)


class _View:
    """Keeps contiguous float64 copies alive behind a pf_state_view."""

    def __init__(self, state, instance):
        n = {"x": instance.num_paths, "y": instance.num_pairs, "dual_demand": instance.num_commodities,
             "dual_capacity": instance.num_edges, "dual_consensus": instance.num_pairs,
             "dual_nonneg": instance.num_paths}
        self.arrs = [_vec(getattr(state, f), m, f"state.{f}") for f, m in n.items()]
        self.view = A.StateView(*(_p(a) for a in self.arrs), float(state.beta), int(state.alpha))


def update_duals(state, instance: Instance):
    """kernels.py:206-216: returns (demand, capacity, consensus, nonneg) duals."""
    v = _View(state, instance)
    dd, dc = np.empty(instance.num_commodities), np.empty(instance.num_edges)
    dcon, dn = np.empty(instance.num_pairs), np.empty(instance.num_paths)
    check(lib().pf_update_duals(instance.handle, C.byref(v.view), _p(dd), _p(dc), _p(dcon), _p(dn)))
    return dd, dc, dcon, dn


def update_slacks(state, instance: Instance):
    """kernels.py:219-232."""
    v = _View(state, instance)
    sd, sc = np.empty(instance.num_commodities), np.empty(instance.num_edges)
    check(lib().pf_update_slacks(instance.handle, C.byref(v.view), _p(sd), _p(sc)))
    return sd, sc


def update_rate_suggestions(state, instance: Instance):
    """kernels.py:235-252."""
    v = _View(state, instance)
    y = np.empty(instance.num_pairs)
    check(lib().pf_update_rate_suggestions(instance.handle, C.byref(v.view), _p(y)))
    return y


def _raise_kernel(instance, rc, bad):
    if rc in (A.PF_ERR_KERNEL_COEF, A.PF_ERR_KERNEL_ROOT):
        what = "coefficients" if rc == A.PF_ERR_KERNEL_COEF else "root"
        key = instance.commodity_key(bad) if 0 <= bad < instance.num_commodities else str(bad)
        raise KernelError(f"non-finite sum {what} for commodity {key}")
    if rc != A.PF_OK:
        raise NativeError(f"pf status {rc}: {last_error()}")


def solve_commodity_sums(state, instance: Instance, alpha):
    """kernels.py:267-282: per-commodity sums from the summed stationarity equation."""
    v = _View(state, instance)
    out = np.empty(instance.num_commodities)
    bad = C.c_int64(-1)
    rc = lib().pf_solve_commodity_sums(instance.handle, C.byref(v.view), int(alpha), _p(out), C.byref(bad))
    _raise_kernel(instance, rc, bad.value)
    return out


def update_rates(state, instance: Instance, sums, alpha):
    """kernels.py:285-296."""
    v = _View(state, instance)
    s = _vec(sums, instance.num_commodities, "sums")
    x = np.empty(instance.num_paths)
    check(lib().pf_update_rates(instance.handle, C.byref(v.view), _p(s), int(alpha), _p(x)))
    return x


def solve_sum_equation(w_sum, beta, q, alpha):
    """kernels.py:198-203 (one device thread)."""
    out = C.c_double()
    check(lib().pf_solve_sum_equation(float(w_sum), float(beta), float(q), int(alpha), C.byref(out)))
    return float(out.value)


def det_diff_norm(a, b, device=None):
    """_reduce.py:118-128 (device, 4096-block / 32-chunk order)."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    if a.ndim != 1 or a.shape != b.shape:
        raise InputError(f"det_diff_norm: shapes {a.shape} and {b.shape} differ")
    out = C.c_double()
    dev = default_device() if device is None else device
    check(lib().pf_det_diff_norm(dev, _p(a), _p(b), a.shape[0], C.byref(out)))
    return float(out.value)
