"""ctypes wrapper for the C oracle -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` leg may import it; the
product package ``paper_2605_01748_b200`` never does.

It exposes the reference's hot path (pathfair ``kernels.py``, ``controller.py``,
``projection.py``, ``model.py``, ``_reduce.py``) as plain numpy-in / numpy-out
functions evaluated in the reference's exact fp64 operation order by
``oracle/pf_oracle.c``.  The oracle itself is pinned against fixtures produced
by running the reference (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libpf_oracle.so")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


class Inst(C.Structure):
    _fields_ = [("C", C.c_int64), ("P", C.c_int64), ("E", C.c_int64), ("NP", C.c_int64),
                ("com_path_ptr", _i64p), ("path_com", _i64p), ("pair_ptr", _i64p),
                ("pair_edge", _i64p), ("pair_path", _i64p), ("edge_pair_ptr", _i64p),
                ("edge_pairs", _i64p), ("hops", _i64p), ("edge_path_count", _i64p),
                ("demand", _f64p), ("capacity", _f64p)]


class State(C.Structure):
    _fields_ = [("x", _f64p), ("y", _f64p), ("dd", _f64p), ("dc", _f64p), ("dcon", _f64p),
                ("dn", _f64p), ("sd", _f64p), ("sc", _f64p), ("beta", C.c_double),
                ("alpha", C.c_int64), ("iteration", C.c_int64)]


class Config(C.Structure):
    _fields_ = [("alpha_target", C.c_int64), ("gamma", C.c_double), ("beta0", C.c_double),
                ("residual_ratio", C.c_double), ("beta_scale", C.c_double),
                ("max_iterations", C.c_int64), ("beta_min", C.c_double), ("beta_max", C.c_double),
                ("adapt", C.c_int32), ("trace", C.c_int32)]


class Ctrl(C.Structure):
    _fields_ = [("ema_s", C.c_double), ("ema_r", C.c_double), ("cooldown", C.c_int64),
                ("just_incremented", C.c_int32), ("stopped", C.c_int32)]


class TraceRow(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("alpha", C.c_int64), ("beta", C.c_double),
                ("s", C.c_double), ("r", C.c_double), ("objective", C.c_double),
                ("pct_violated", C.c_double), ("mean_relative_violation", C.c_double)]


OK, KERNEL_COEF, KERNEL_ROOT, SOLVER, INPUT, NOMEM = range(6)


def build_library(force: bool = False) -> str:
    """Compile the oracle (make -C oracle).  Building the checker is not using it."""
    if force or not os.path.exists(_SO) or (
            os.path.getmtime(_SO) < os.path.getmtime(os.path.join(_HERE, "pf_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_library()
        L = C.CDLL(_SO)
        L.pfo_sum_range.restype = C.c_double
        L.pfo_det_diff_norm.restype = C.c_double
        L.pfo_root_scalar.restype = C.c_double
        L.pfo_root_scalar.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int64]
        L.pfo_solve_sum_equation.restype = C.c_double
        L.pfo_solve_sum_equation.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int64]
        L.pfo_adapt_beta.restype = C.c_double
        L.pfo_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _p(a, t=_f64p):
    return a.ctypes.data_as(t)


def set_threads(n: int) -> None:
    lib().pfo_set_threads(int(n))


def num_threads() -> int:
    return int(lib().pfo_num_threads())


# --------------------------------------------------------------------- instance


@dataclass
class FlatInstance:
    """The reference's Instance index spaces (model.py:135-180) as int64 arrays."""

    kept_rows: np.ndarray
    demand: np.ndarray
    capacity: np.ndarray
    com_path_ptr: np.ndarray
    path_com: np.ndarray
    hops: np.ndarray
    pair_ptr: np.ndarray
    pair_edge: np.ndarray
    pair_path: np.ndarray
    edge_path_count: np.ndarray
    edge_pair_ptr: np.ndarray
    edge_pairs: np.ndarray

    @property
    def num_commodities(self):
        return int(self.demand.shape[0])

    @property
    def num_paths(self):
        return int(self.path_com.shape[0])

    @property
    def num_edges(self):
        return int(self.capacity.shape[0])

    @property
    def num_pairs(self):
        return int(self.pair_edge.shape[0])

    def cstruct(self) -> Inst:
        s = Inst(self.num_commodities, self.num_paths, self.num_edges, self.num_pairs,
                 _p(self.com_path_ptr, _i64p), _p(self.path_com, _i64p), _p(self.pair_ptr, _i64p),
                 _p(self.pair_edge, _i64p), _p(self.pair_path, _i64p), _p(self.edge_pair_ptr, _i64p),
                 _p(self.edge_pairs, _i64p), _p(self.hops, _i64p), _p(self.edge_path_count, _i64p),
                 _p(self.demand), _p(self.capacity))
        s._keep = self  # keep arrays alive
        return s

    def with_conditions(self, capacity=None, demand=None) -> "FlatInstance":
        import dataclasses
        return dataclasses.replace(
            self,
            capacity=self.capacity if capacity is None else np.ascontiguousarray(capacity, np.float64),
            demand=self.demand if demand is None else np.ascontiguousarray(demand, np.float64))


def build_instance(capacity, demand0, com_path_ptr0, path_edge_ptr0, path_edges0) -> FlatInstance:
    """model.py:206-271 (index construction; validation is out of the oracle's scope)."""
    capacity = np.ascontiguousarray(capacity, np.float64)
    demand0 = np.ascontiguousarray(demand0, np.float64)
    cpp = np.ascontiguousarray(com_path_ptr0, np.int64)
    pep = np.ascontiguousarray(path_edge_ptr0, np.int64)
    pe = np.ascontiguousarray(path_edges0, np.int64)
    C0, P0, NP0, E = demand0.shape[0], pep.shape[0] - 1, pe.shape[0], capacity.shape[0]
    kept = np.empty(C0, np.int64)
    dem = np.empty(C0, np.float64)
    o_cpp = np.empty(C0 + 1, np.int64)
    path_com = np.empty(P0, np.int64)
    hops = np.empty(P0, np.int64)
    pair_ptr = np.empty(P0 + 1, np.int64)
    pair_edge = np.empty(NP0, np.int64)
    pair_path = np.empty(NP0, np.int64)
    epc = np.empty(E, np.int64)
    epp = np.empty(E + 1, np.int64)
    edge_pairs = np.empty(NP0, np.int64)
    sizes = np.zeros(3, np.int64)
    st = lib().pfo_build_instance(
        C.c_int64(C0), C.c_int64(E), _p(cpp, _i64p), _p(pep, _i64p), _p(pe, _i64p), _p(demand0),
        _p(kept, _i64p), _p(dem), _p(o_cpp, _i64p), _p(path_com, _i64p), _p(hops, _i64p),
        _p(pair_ptr, _i64p), _p(pair_edge, _i64p), _p(pair_path, _i64p), _p(epc, _i64p),
        _p(epp, _i64p), _p(edge_pairs, _i64p), _p(sizes, _i64p))
    if st != OK:
        raise ValueError("oracle build_instance: bad edge id")
    nc, npth, npr = (int(v) for v in sizes)
    return FlatInstance(kept[:nc].copy(), dem[:nc].copy(), capacity.copy(), o_cpp[:nc + 1].copy(),
                        path_com[:npth].copy(), hops[:npth].copy(), pair_ptr[:npth + 1].copy(),
                        pair_edge[:npr].copy(), pair_path[:npr].copy(), epc, epp, edge_pairs[:npr].copy())


# --------------------------------------------------------------------- state


@dataclass
class OState:
    """Mirror of pathfair.kernels.SolverState (kernels.py:24-44)."""

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

    _FIELDS = ("x", "y", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg",
               "slack_demand", "slack_capacity")

    @classmethod
    def like(cls, st) -> "OState":
        return cls(*(np.ascontiguousarray(getattr(st, f), np.float64).copy() for f in cls._FIELDS),
                   float(st.beta), int(st.alpha), int(st.iteration))

    def cstruct(self) -> State:
        s = State(*(_p(getattr(self, f)) for f in self._FIELDS), self.beta, self.alpha, self.iteration)
        s._keep = self
        return s


def _empty_state(I: FlatInstance) -> OState:
    C_, P_, E_, NP_ = I.num_commodities, I.num_paths, I.num_edges, I.num_pairs
    z = np.zeros
    return OState(z(P_), z(NP_), z(C_), z(E_), z(NP_), z(P_), z(C_), z(E_), 1.0, 0, 0)


# --------------------------------------------------------------------- kernels


def commodity_sums(I: FlatInstance, rates) -> np.ndarray:
    rates = np.ascontiguousarray(rates, np.float64)
    out = np.empty(I.num_commodities)
    lib().pfo_commodity_sums(C.byref(I.cstruct()), _p(rates), _p(out))
    return out


def edge_loads(I: FlatInstance, rates) -> np.ndarray:
    rates = np.ascontiguousarray(rates, np.float64)
    out = np.empty(I.num_edges)
    lib().pfo_edge_loads(C.byref(I.cstruct()), _p(rates), _p(out))
    return out


def edge_loads_from_pairs(I: FlatInstance, vals) -> np.ndarray:
    vals = np.ascontiguousarray(vals, np.float64)
    out = np.empty(I.num_edges)
    lib().pfo_edge_loads_from_pairs(C.byref(I.cstruct()), _p(vals), _p(out))
    return out


def det_diff_norm(a, b) -> float:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return float(lib().pfo_det_diff_norm(_p(a), _p(b), C.c_int64(a.shape[0])))


def update_duals(I: FlatInstance, st):
    s = OState.like(st)
    dd, dc = np.empty(I.num_commodities), np.empty(I.num_edges)
    dcon, dn = np.empty(I.num_pairs), np.empty(I.num_paths)
    lib().pfo_update_duals(C.byref(I.cstruct()), C.byref(s.cstruct()), _p(dd), _p(dc), _p(dcon), _p(dn))
    return dd, dc, dcon, dn


def update_slacks(I: FlatInstance, st):
    s = OState.like(st)
    sd, sc = np.empty(I.num_commodities), np.empty(I.num_edges)
    lib().pfo_update_slacks(C.byref(I.cstruct()), C.byref(s.cstruct()), _p(sd), _p(sc))
    return sd, sc


def update_rate_suggestions(I: FlatInstance, st) -> np.ndarray:
    s = OState.like(st)
    y = np.empty(I.num_pairs)
    lib().pfo_update_suggestions(C.byref(I.cstruct()), C.byref(s.cstruct()), _p(y))
    return y


def coefficients(I: FlatInstance, st):
    s = OState.like(st)
    pk, pw = np.empty(I.num_paths), np.empty(I.num_paths)
    ws, q = np.empty(I.num_commodities), np.empty(I.num_commodities)
    lib().pfo_coefficients(C.byref(I.cstruct()), C.byref(s.cstruct()), _p(pk), _p(pw), _p(ws), _p(q))
    return pk, pw, ws, q


class OracleKernelError(RuntimeError):
    def __init__(self, kind, commodity):
        super().__init__(f"{kind} for commodity index {commodity}")
        self.kind, self.commodity = kind, commodity


class OracleSolverError(RuntimeError):
    pass


def solve_commodity_sums(I: FlatInstance, st, alpha: int) -> np.ndarray:
    s = OState.like(st)
    out = np.empty(I.num_commodities)
    bad = C.c_int64(-1)
    rc = lib().pfo_solve_commodity_sums(C.byref(I.cstruct()), C.byref(s.cstruct()), C.c_int64(alpha),
                                        _p(out), C.byref(bad))
    if rc == KERNEL_COEF:
        raise OracleKernelError("non-finite sum coefficients", bad.value)
    if rc == KERNEL_ROOT:
        raise OracleKernelError("non-finite sum root", bad.value)
    return out


def update_rates(I: FlatInstance, st, sums, alpha: int) -> np.ndarray:
    s = OState.like(st)
    sums = np.ascontiguousarray(sums, np.float64)
    x = np.empty(I.num_paths)
    lib().pfo_update_rates(C.byref(I.cstruct()), C.byref(s.cstruct()), _p(sums), C.c_int64(alpha), _p(x))
    return x


def solve_sum_equation(w_sum, beta, q, alpha) -> float:
    return float(lib().pfo_solve_sum_equation(float(w_sum), float(beta), float(q), int(alpha)))


def root_scalar(lin, c, q, alpha) -> float:
    return float(lib().pfo_root_scalar(float(lin), float(c), float(q), int(alpha)))


def score_paths(I: FlatInstance, rates, alpha: int) -> np.ndarray:
    rates = np.ascontiguousarray(rates, np.float64)
    out = np.empty(I.num_paths)
    lib().pfo_score_paths(C.byref(I.cstruct()), _p(rates), C.c_int64(alpha), _p(out))
    return out


def project(I: FlatInstance, rates, alpha: int) -> np.ndarray:
    rates = np.ascontiguousarray(rates, np.float64)
    out = np.empty(I.num_paths)
    if lib().pfo_project(C.byref(I.cstruct()), _p(rates), C.c_int64(alpha), _p(out)) != OK:
        raise ValueError("projection input contains non-finite rates")
    return out


def violation_stats(I: FlatInstance, rates, tol=1e-9):
    rates = np.ascontiguousarray(rates, np.float64)
    pct, mean_rel, nv = C.c_double(), C.c_double(), C.c_int64()
    lib().pfo_violation_stats(C.byref(I.cstruct()), _p(rates), C.c_double(tol), C.byref(pct),
                              C.byref(mean_rel), C.byref(nv))
    return pct.value, mean_rel.value, nv.value


# --------------------------------------------------------------------- controller


def dao_carry_rates(I: FlatInstance, rates, tol=1e-9) -> np.ndarray:
    """oracles.py:262-287: a stale allocation applied to drifted conditions
    (I carries the drifted capacity / demand).  Commodity sums above the new
    demand scale down by D / S; then the most overloaded edge (first index on
    ties) scales its paths (each once) by cap / (over + cap), at most 4 E + 4
    times.  Sums and loads are the exact-order C kernels."""
    x = np.ascontiguousarray(rates, np.float64).copy()
    sums = commodity_sums(I, x)
    for c in np.flatnonzero(sums > I.demand + tol):
        lo, hi = int(I.com_path_ptr[c]), int(I.com_path_ptr[c + 1])
        x[lo:hi] *= I.demand[c] / sums[c]
    if I.num_edges == 0:
        return x
    for _ in range(4 * I.num_edges + 4):
        over = edge_loads(I, x) - I.capacity
        e = int(np.argmax(over))
        if over[e] <= tol:
            break
        load = over[e] + I.capacity[e]
        factor = I.capacity[e] / load
        lo, hi = int(I.edge_pair_ptr[e]), int(I.edge_pair_ptr[e + 1])
        paths = np.unique(I.pair_path[I.edge_pairs[lo:hi]])
        x[paths] *= factor
    return x


def make_config(alpha_target=None, gamma=1e-3, beta0=1.0, residual_ratio=10.0, beta_scale=2.0,
                max_iterations=5000, beta_min=1e-6, beta_max=1e6, adapt=True, trace=False) -> Config:
    """controller.py:29-61 SolverConfig defaults."""
    return Config(-1 if alpha_target is None else int(alpha_target), gamma, beta0, residual_ratio,
                  beta_scale, int(max_iterations), beta_min, beta_max, int(bool(adapt)), int(bool(trace)))


class Loop:
    """controller.py:197-273 `solve` loop, advanced in chunks so tests can
    snapshot the full state at chosen iteration counts."""

    def __init__(self, I: FlatInstance, config: Config, warm=None, trace_cap=0):
        self.I, self.cfg = I, config
        self.s = _empty_state(I)
        self.w = _empty_state(I)
        self.cs = self.s.cstruct()
        self.cw = self.w.cstruct()
        self.ci = I.cstruct()
        self.sums = np.zeros(max(I.num_commodities, 1))
        warm_p = None
        if warm is not None:
            self._warm = np.ascontiguousarray(warm, np.float64)
            warm_p = _p(self._warm)
        if lib().pfo_initialize_state(C.byref(self.ci), C.byref(config), warm_p, C.byref(self.cs)) != OK:
            raise ValueError("warm start contains non-finite rates")
        self.ctrl = Ctrl()
        lib().pfo_ctrl_init(C.byref(self.ctrl))
        self.trace = (TraceRow * max(trace_cap, 1))()
        self.trace_cap = trace_cap
        self.ntrace = C.c_int64(0)
        # addresses -> arrays (the C loop swaps state/scratch pointers)
        self._by_addr = {}
        for st in (self.s, self.w):
            for f in OState._FIELDS:
                a = getattr(st, f)
                self._by_addr[a.ctypes.data] = a

    def step(self, n: int) -> None:
        bad = C.c_int64(-1)
        rc = lib().pfo_iterate(C.byref(self.ci), C.byref(self.cfg), C.byref(self.cs), C.byref(self.ctrl),
                               C.c_int64(n), C.byref(self.cw), _p(self.sums), self.trace,
                               C.c_int64(self.trace_cap), C.byref(self.ntrace), C.byref(bad))
        if rc == KERNEL_COEF:
            raise OracleKernelError("non-finite sum coefficients", bad.value)
        if rc == KERNEL_ROOT:
            raise OracleKernelError("non-finite sum root", bad.value)
        if rc == SOLVER:
            raise OracleSolverError(f"non-finite iterates at iteration {self.cs.iteration}")

    @property
    def stopped(self) -> bool:
        return bool(self.ctrl.stopped)

    def state(self) -> OState:
        """Copy of the current SolverState."""
        vals = []
        for f in State._fields_[:8]:
            addr = C.cast(getattr(self.cs, f[0]), C.c_void_p).value
            vals.append(self._by_addr[addr].copy())
        return OState(*vals, float(self.cs.beta), int(self.cs.alpha), int(self.cs.iteration))

    def last_sums(self) -> np.ndarray:
        return self.sums[: self.I.num_commodities].copy()

    def trace_rows(self):
        n = self.ntrace.value
        return [(r.iteration, r.alpha, r.beta, r.s, r.r, r.objective, r.pct_violated,
                 r.mean_relative_violation) for r in self.trace[:n]]


@dataclass
class OracleResult:
    rates: np.ndarray
    sums: np.ndarray
    iterations: int
    alpha: int
    converged: bool
    trace: list | None
    raw_x: np.ndarray


def solve(I: FlatInstance, alpha_target=None, warm_start=None, **cfg) -> OracleResult:
    """controller.py:197-284 solve(), including the final projection."""
    config = make_config(alpha_target=alpha_target, **cfg)
    trace = bool(cfg.get("trace", False))
    if I.num_paths == 0:
        return OracleResult(np.zeros(0), np.zeros(I.num_commodities), 0,
                            0 if warm_start is None or alpha_target is None else alpha_target,
                            True, [] if trace else None, np.zeros(0))
    loop = Loop(I, config, warm_start, trace_cap=config.max_iterations if trace else 0)
    loop.step(config.max_iterations)
    st = loop.state()
    rates = project(I, st.x, st.alpha)
    return OracleResult(rates, commodity_sums(I, rates), st.iteration, st.alpha, loop.stopped,
                        loop.trace_rows() if trace else None, st.x)
