"""Outer solve loop (pathfair/controller.py API) running on the GPU.

`solve(instance, config, warm_start)` is a drop-in for controller.py:197-284:
same config knobs and validation, same SolveResult / IterationTrace shapes,
same error types.  The loop itself runs in the native library:

* ``mode="exact"``: the reference's kernels in exact fp64 operation order
  (csrc/exact.cu) with the scalar controller on the host -- bit-identical to
  the reference for alpha <= 1 at equal iteration counts;
* ``mode="fast"`` (default): the fused persistent kernel (csrc/fused.cu) with
  the controller on the device; deterministic, tolerance-matched.

Both return the GPU-projected, feasible allocation (projection.py:51-107).
"""

from __future__ import annotations

import ctypes as C
import dataclasses
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _abi as A
from ._lib import NativeError, check, last_error, lib
from .kernels import KernelError, SolverState, det_diff_norm
from .model import InputError, Instance


class SolverError(RuntimeError):
    """Iterates went non-finite (controller.py:25-26)."""


_MODES = {"exact": A.PF_MODE_EXACT, "fast": A.PF_MODE_FAST}


@dataclass
class SolverConfig:
    """controller.py:29-61, plus `mode` (exact | fast)."""

    alpha_target: int | None = None
    gamma: float = 1e-3
    beta0: float = 1.0
    residual_ratio: float = 10.0
    beta_scale: float = 2.0
    max_iterations: int = 5000
    beta_min: float = 1e-6
    beta_max: float = 1e6
    adapt: bool = True
    trace: bool = False
    reference_sums: np.ndarray | None = None
    mode: str = "fast"

    def __post_init__(self):
        if self.gamma <= 0:
            raise InputError("gamma must be > 0")
        if self.residual_ratio <= 1 or self.beta_scale <= 1:
            raise InputError("residual_ratio and beta_scale must be > 1")
        if not 0 < self.beta_min <= self.beta_max:
            raise InputError("beta bounds must satisfy 0 < beta_min <= beta_max")
        if self.alpha_target is not None and self.alpha_target < 0:
            raise InputError("alpha_target must be >= 0")
        if self.max_iterations < 1:
            raise InputError("max_iterations must be >= 1")
        if self.mode not in _MODES:
            raise InputError(f"mode must be one of {sorted(_MODES)}")

    def to_c(self, project=True, keep=None, with_reference=True) -> A.Config:
        ref = None
        if self.reference_sums is not None and self.trace and with_reference:
            rs = np.ascontiguousarray(self.reference_sums, np.float64)
            if keep is not None:
                keep.append(rs)
            ref = rs.ctypes.data_as(A.f64p)
        return A.Config(-1 if self.alpha_target is None else int(self.alpha_target), float(self.gamma),
                        float(self.beta0), float(self.residual_ratio), float(self.beta_scale),
                        int(self.max_iterations), float(self.beta_min), float(self.beta_max), int(bool(self.adapt)),
                        int(bool(self.trace)), _MODES[self.mode], int(bool(project)), ref)


@dataclass(frozen=True)
class Residuals:
    s: float
    r: float


@dataclass(frozen=True)
class IterationTrace:
    iteration: int
    alpha: int
    beta: float
    s: float
    r: float
    objective: float
    pct_violated: float
    mean_relative_violation: float
    optimality: float | None


@dataclass(frozen=True)
class SolveResult:
    rates: np.ndarray
    sums: np.ndarray
    iterations: int
    alpha: int
    converged: bool
    runtime_s: float
    trace: tuple | None
    loop_ms: float = field(default=0.0, compare=False)
    projection_ms: float = field(default=0.0, compare=False)
    mode: str = field(default="fast", compare=False)  # the arithmetic that ran: "fast" | "exact"


def _p(a):
    return a.ctypes.data_as(A.f64p)


def _check_warm(instance, warm_start):
    if warm_start is None:
        return None
    x = np.ascontiguousarray(warm_start, np.float64)
    if x.shape != (instance.num_paths,):
        raise InputError(f"warm start has {x.shape[0]} rates, expected {instance.num_paths}")
    # finiteness (controller.py:104-111) is checked by the native init on the
    # device copy; the array is only read during the call, so no copy here
    return x


def _raise(instance, rc, res_bad, it):
    if rc == A.PF_OK:
        return
    if rc in (A.PF_ERR_KERNEL_COEF, A.PF_ERR_KERNEL_ROOT):
        what = "coefficients" if rc == A.PF_ERR_KERNEL_COEF else "root"
        key = instance.commodity_key(res_bad) if 0 <= res_bad < instance.num_commodities else str(res_bad)
        raise KernelError(f"non-finite sum {what} for commodity {key}")
    if rc == A.PF_ERR_SOLVER:
        raise SolverError(last_error())
    if rc == A.PF_ERR_INPUT:
        raise InputError(last_error())
    raise NativeError(f"pf status {rc}: {last_error()}")


def _trace_rows(buf, n):
    rows = []
    for r in buf[:n]:
        opt = None if np.isnan(r.optimality) else float(r.optimality)
        rows.append(IterationTrace(int(r.iteration), int(r.alpha), float(r.beta), float(r.s), float(r.r),
                                   float(r.objective), float(r.pct_violated), float(r.mean_relative_violation), opt))
    return tuple(rows)


def _fallback_warning(res):
    if res.exact_fallback:
        warnings.warn("mode='fast' requested outside the fused kernel's layout limits (more than 32 paths or "
                      "16,384 pairs per commodity, or 65,535 edges): the exact-order kernels ran instead "
                      "(SolveResult.mode == 'exact')", RuntimeWarning, stacklevel=3)


def _result(res, rates, sums, trace, config):
    return SolveResult(rates=rates, sums=sums, iterations=int(res.iterations), alpha=int(res.alpha),
                       converged=bool(res.converged), runtime_s=float(res.runtime_s), trace=trace,
                       loop_ms=float(res.loop_ms), projection_ms=float(res.projection_ms),
                       mode="exact" if (config.mode == "exact" or res.exact_fallback) else "fast")


def solve(instance: Instance, config: SolverConfig | None = None, warm_start=None) -> SolveResult:
    """controller.py:197-284: run the loop on the GPU and return a projected, feasible result."""
    config = config if config is not None else SolverConfig()
    warm = _check_warm(instance, warm_start)
    if config.trace:
        return _solve_traced(instance, config, warm)
    keep = []
    cfg = config.to_c(keep=keep, with_reference=False)  # reference_sums only feed the trace
    rates = np.empty(instance.num_paths)
    sums = np.empty(instance.num_commodities)
    res = A.Result()
    tlen = C.c_int64(0)
    rc = lib().pf_solve(instance.handle, C.byref(cfg), _p(warm) if warm is not None else None, _p(rates),
                        _p(sums), C.byref(res), None, 0, C.byref(tlen))
    _raise(instance, rc, res.bad_commodity, res.iterations)
    _fallback_warning(res)
    return _result(res, rates, sums, None, config)


def _solve_traced(instance, config, warm):
    """solve() with trace=True through the device-resident solver, so the rows
    are copied out by the run's actual length (the reference's trace list grows
    lazily; a buffer of max_iterations rows would not)."""
    ref_ok = (config.reference_sums is None
              or np.asarray(config.reference_sums).shape == (instance.num_commodities,))
    s = Solver(instance, config if ref_ok else dataclasses.replace(config, reference_sums=None))
    s.init(warm)
    if not ref_ok and instance.num_paths:
        # the reference fails in its first trace row (optimality_from_sums,
        # controller.py:183), i.e. after iteration 1's kernels: a KernelError there wins
        s.run(1)
        raise InputError("commodity sets differ between allocation and reference")
    s.run(config.max_iterations)
    rates, sums = s.finish()
    res = s.result()
    _fallback_warning(res)
    return _result(res, rates, sums, s.trace(), config)


class Solver:
    """Device-resident solver (pf_solver_*): the loop can be advanced in
    chunks, timed on the device and inspected without leaving the GPU."""

    def __init__(self, instance: Instance, config: SolverConfig | None = None):
        self.instance = instance
        self.config = config if config is not None else SolverConfig()
        rs = self.config.reference_sums
        if self.config.trace and rs is not None and np.asarray(rs).shape != (instance.num_commodities,):
            raise InputError("commodity sets differ between allocation and reference")
        self._keep = []
        self._cfg = self.config.to_c(keep=self._keep)
        h = C.c_void_p()
        check(lib().pf_solver_create(instance.handle, C.byref(self._cfg), C.byref(h)))
        self._h = h.value

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().pf_solver_destroy(self._h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None

    def init(self, warm_start=None):
        warm = _check_warm(self.instance, warm_start)
        _raise(self.instance, lib().pf_solver_init(self._h, _p(warm) if warm is not None else None), -1, 0)
        return self

    def run(self, steps: int) -> int:
        done = C.c_int64(0)
        rc = lib().pf_solver_run(self._h, int(steps), C.byref(done))
        if rc != A.PF_OK:
            r = self.result()
            _raise(self.instance, rc, r.bad_commodity, r.iterations)
        return int(done.value)

    def result(self) -> A.Result:
        res = A.Result()
        check(lib().pf_solver_result(self._h, C.byref(res)))
        return res

    def finish(self):
        rates = np.empty(self.instance.num_paths)
        sums = np.empty(self.instance.num_commodities)
        rc = lib().pf_solver_finish(self._h, _p(rates), _p(sums))
        if rc != A.PF_OK:
            r = self.result()
            _raise(self.instance, rc, r.bad_commodity, r.iterations)
        return rates, sums

    def x(self) -> np.ndarray:
        out = np.empty(self.instance.num_paths)
        check(lib().pf_solver_get_x(self._h, _p(out)))
        return out

    def state(self) -> SolverState:
        I = self.instance
        x, y = np.empty(I.num_paths), np.empty(I.num_pairs)
        dd, dc = np.empty(I.num_commodities), np.empty(I.num_edges)
        dcon, dn = np.empty(I.num_pairs), np.empty(I.num_paths)
        beta, alpha, it = C.c_double(), C.c_int64(), C.c_int64()
        check(lib().pf_solver_get_state(self._h, _p(x), _p(y), _p(dd), _p(dc), _p(dcon), _p(dn), C.byref(beta),
                                        C.byref(alpha), C.byref(it)))
        return SolverState(x, y, dd, dc, dcon, dn, np.zeros(I.num_commodities), np.zeros(I.num_edges),
                           float(beta.value), int(alpha.value), int(it.value))

    def time_loop(self, iterations: int):
        """Runs `iterations` fused iterations in one launch; returns (ms, ms/iteration) by CUDA events."""
        tot, per = C.c_float(), C.c_float()
        check(lib().pf_solver_time_loop(self._h, int(iterations), C.byref(tot), C.byref(per)))
        return float(tot.value), float(per.value)

    def trace(self) -> tuple:
        """The IterationTrace rows recorded so far (pf_solver_trace)."""
        total = C.c_int64(0)
        check(lib().pf_solver_trace(self._h, None, 0, C.byref(total)))
        buf = (A.TraceRow * max(total.value, 1))()
        check(lib().pf_solver_trace(self._h, buf, total.value, C.byref(total)))
        return _trace_rows(buf, total.value)

    def time_to_quality(self, reference_sums, target: float = 0.99, sample_every: int = 125,
                        sample_cap: int = 100000) -> dict:
        """From the current state, run to the first iteration k* whose
        post-projection optimality_from_sums(S_k, reference_sums,
        default_theta) >= target (the trace optimality column of
        controller.py:173-194, oracles.py:244-254), in one pass on the device:
        the quality is sampled every `sample_every` iterations and the crossing
        chunk replayed from a device snapshot (pf_solver_time_to_quality).  The
        solver stands at k* (or where the controller stopped) afterwards."""
        ref = np.ascontiguousarray(reference_sums, dtype=np.float64)
        if ref.shape != (self.instance.num_commodities,):
            raise InputError("commodity sets differ between allocation and reference")
        out = A.TtqResult()
        it = np.zeros(sample_cap, np.int64)
        q = np.zeros(sample_cap, np.float64)
        rc = lib().pf_solver_time_to_quality(self._h, _p(ref), float(target), int(sample_every), C.byref(out),
                                             it.ctypes.data_as(A.i64p), _p(q), int(sample_cap))
        if rc != A.PF_OK:
            r = self.result()
            _raise(self.instance, rc, r.bad_commodity, r.iterations)
        n = min(int(out.samples), sample_cap)
        return {"k_star": int(out.k_star) if out.k_star >= 0 else None, "quality": float(out.quality),
                "iterations": int(out.iterations), "loop_ms": float(out.loop_ms),
                "quality_ms": float(out.quality_ms), "samples": list(zip(it[:n].tolist(), q[:n].tolist()))}

    def kernel_stats(self):
        vals = [C.c_int64() for _ in range(4)]
        check(lib().pf_solver_kernel_stats(self._h, *(C.byref(v) for v in vals)))
        return dict(launches=vals[0].value, tiles=vals[1].value, grid=vals[2].value, bytes_per_iter=vals[3].value)


def initialize_state(instance: Instance, config: SolverConfig, warm_start=None) -> SolverState:
    """controller.py:98-128, materialised on the device and copied back."""
    warm = _check_warm(instance, warm_start)
    s = Solver(instance, SolverConfig(**{**config.__dict__, "mode": "exact", "trace": False,
                                         "reference_sums": None}))
    s.init(warm)
    st = s.state()
    return st


def compute_residuals(prev_state, next_state, device=None) -> Residuals:
    """controller.py:131-139 (device det_diff_norm)."""
    s = det_diff_norm(next_state.x, prev_state.x, device)
    r = float(np.sqrt(
        det_diff_norm(next_state.dual_demand, prev_state.dual_demand, device) ** 2
        + det_diff_norm(next_state.dual_capacity, prev_state.dual_capacity, device) ** 2
        + det_diff_norm(next_state.dual_consensus, prev_state.dual_consensus, device) ** 2
        + det_diff_norm(next_state.dual_nonneg, prev_state.dual_nonneg, device) ** 2
    ))
    return Residuals(s=s, r=r)


def adapt_beta(beta, residuals, config):
    """controller.py:142-150."""
    if residuals.r > config.residual_ratio * residuals.s:
        beta = beta * config.beta_scale
    elif residuals.s > config.residual_ratio * residuals.r:
        beta = beta / config.beta_scale
    return float(min(max(beta, config.beta_min), config.beta_max))


def check_convergence(residuals, gamma):
    """controller.py:153-154."""
    return residuals.r <= gamma and residuals.s <= gamma


def advance_alpha(state, config, converged_now, converged_immediately_after_increment):
    """controller.py:157-170."""
    if not converged_now:
        return "continue"
    if config.alpha_target is not None and state.alpha >= config.alpha_target:
        return "stop"
    if converged_immediately_after_increment:
        return "stop"
    return "increment"
