"""Problem model: validated inputs -> GPU-resident incidence store.

Mirrors pathfair/model.py (names, fields, validation messages).  The flat index
spaces (model.py:135-180) are built ON THE GPU by `pf_instance_create`
(csrc/incidence.cu) and stay resident there; the numpy views below are exported
from the device lazily (and cached) so callers and tests can read them exactly
as they read the reference's Instance.  Sums, loads and validation run on the
device in the reference's exact reduction order.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from functools import cached_property

import numpy as np

from . import _abi as A
from ._lib import check, lib
from .topology import (FEAS_TOL, Commodity, CommodityTable, FlatPathSet, InputError, PathSet, Topology,
                       as_flat, build_topology)

__all__ = ["FEAS_TOL", "Commodity", "CommodityTable", "FlatPathSet", "InputError", "Instance", "PathSet",
           "Topology", "ViolationReport", "build_instance", "build_instance_flat", "build_topology",
           "build_instance_raw", "commodity_sums", "edge_loads", "edge_loads_from_pairs", "validate_allocation", "with_conditions",
           "default_device"]


def default_device() -> int:
    for k in ("PF_DEVICE", "LOCAL_RANK"):
        if os.environ.get(k):
            return int(os.environ[k])
    return 0


def _p(a, t=A.f64p):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, np.float64)


def _i64(a):
    return np.ascontiguousarray(a, np.int64)


_INDEX_FIELDS = {
    "com_path_ptr": A.PF_COM_PATH_PTR, "path_com": A.PF_PATH_COM, "hops": A.PF_HOPS,
    "pair_ptr": A.PF_PAIR_PTR, "pair_edge": A.PF_PAIR_EDGE, "pair_path": A.PF_PAIR_PATH,
    "edge_path_count": A.PF_EDGE_PATH_COUNT, "edge_pair_ptr": A.PF_EDGE_PAIR_PTR,
    "edge_pairs": A.PF_EDGE_PAIRS, "kept_rows": A.PF_KEPT_ROWS,
}


class _Handle:
    """Owns one pf_instance* (device memory is freed with it)."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            try:
                lib().pf_instance_destroy(self.ptr)
            except Exception:  # noqa: BLE001  (interpreter shutdown)
                pass
            self.ptr = None


class Instance:
    """Flat-indexed problem instance (model.py:135-180), resident on a GPU.

    Index spaces: commodities (retained only), paths (commodity-major, input
    order), edges (topology order), and consensus pairs laid out path-major;
    edge_pairs regroups pair ids per edge.  Arrays are exported from the device
    on first access.
    """

    def __init__(self, handle, topology, table, demand, capacity, sizes, device):
        self._h = handle
        self.topology = topology
        self._table = table
        self.demand = demand
        self.capacity = capacity
        self._sizes = sizes
        self.device = device

    # ---- sizes
    @property
    def num_commodities(self):
        return self._sizes[0]

    @property
    def num_paths(self):
        return self._sizes[1]

    @property
    def num_edges(self):
        return self._sizes[2]

    @property
    def num_pairs(self):
        return self._sizes[3]

    @property
    def handle(self):
        return self._h.ptr

    # ---- exported index arrays (bit-exact with the reference; int64)
    def _export(self, field, n):
        out = np.empty(n, np.int64)
        if n:
            check(lib().pf_instance_export_index(self.handle, field, _p(out, A.i64p)))
        return out

    @cached_property
    def kept_rows(self):
        return self._export(A.PF_KEPT_ROWS, self.num_commodities)

    @cached_property
    def com_path_ptr(self):
        return self._export(A.PF_COM_PATH_PTR, self.num_commodities + 1)

    @cached_property
    def path_com(self):
        return self._export(A.PF_PATH_COM, self.num_paths)

    @cached_property
    def hops(self):
        return self._export(A.PF_HOPS, self.num_paths)

    @cached_property
    def pair_ptr(self):
        return self._export(A.PF_PAIR_PTR, self.num_paths + 1)

    @cached_property
    def pair_edge(self):
        return self._export(A.PF_PAIR_EDGE, self.num_pairs)

    @cached_property
    def pair_path(self):
        return self._export(A.PF_PAIR_PATH, self.num_pairs)

    @cached_property
    def edge_path_count(self):
        return self._export(A.PF_EDGE_PATH_COUNT, self.num_edges)

    @cached_property
    def edge_pair_ptr(self):
        return self._export(A.PF_EDGE_PAIR_PTR, self.num_edges + 1)

    @cached_property
    def edge_pairs(self):
        return self._export(A.PF_EDGE_PAIRS, self.num_pairs)

    @cached_property
    def commodities(self):
        return tuple(self._table[int(k)] for k in self.kept_rows)

    def fast_supported(self):
        """(ok, why): whether mode="fast" runs the fused kernel on this instance
        (else solves fall back to the exact-order kernels, with a warning)."""
        ok = C.c_int()
        why = C.create_string_buffer(256)
        check(lib().pf_instance_fast_supported(self.handle, C.byref(ok), why, 256))
        return bool(ok.value), why.value.decode()

    def commodity_key(self, c):
        """Reference Commodity.key ("src→dst") of retained commodity c."""
        return self._table.key(int(self.kept_rows[c]))

    def path_edges(self, p):
        return self.pair_edge[self.pair_ptr[p]:self.pair_ptr[p + 1]]

    def commodity_paths(self, c):
        return range(int(self.com_path_ptr[c]), int(self.com_path_ptr[c + 1]))


def _validate_paths(topology: Topology, table: CommodityTable, flat: FlatPathSet):
    """model.py:183-203 _check_path, vectorised; raises on the first bad path
    in commodity-major order with the reference's message."""
    cpp, pep, pe = flat.com_path_ptr, flat.path_edge_ptr, flat.path_edges
    P0 = pep.shape[0] - 1
    if P0 == 0:
        return
    # the native check (OpenMP) finds whether any path is bad; the vectorised
    # code below only runs to name the first bad path with the reference's message
    from ._lib import gen_lib
    i64 = lambda a: np.ascontiguousarray(a, np.int64)  # noqa: E731
    arrs = [i64(cpp), i64(pep), i64(pe), i64(topology.edge_src), i64(topology.edge_dst), i64(table.src),
            i64(table.dst)]
    ptr = [a.ctypes.data_as(C.POINTER(C.c_int64)) for a in arrs]
    if gen_lib().pf_validate_paths(len(table), ptr[0], ptr[1], ptr[2], topology.num_edges, ptr[3], ptr[4], ptr[5],
                               ptr[6]) < 0:
        return
    m = topology.num_edges
    hops = np.diff(pep)
    owner = np.repeat(np.arange(len(table), dtype=np.int64), np.diff(cpp))
    bad_e = (pe < 0) | (pe >= m)
    cs = np.concatenate([[0], np.cumsum(bad_e)])
    n_bad = cs[pep[1:]] - cs[pep[:-1]]
    safe = np.where(bad_e, 0, pe)
    nonempty = hops > 0
    first = np.where(nonempty, safe[np.minimum(pep[:-1], max(pe.shape[0] - 1, 0))], 0) if pe.size else np.zeros(P0, np.int64)
    last = np.where(nonempty, safe[np.maximum(pep[1:] - 1, 0)], 0) if pe.size else np.zeros(P0, np.int64)
    es, ed = topology.edge_src, topology.edge_dst
    start_bad = nonempty & (es[first] != table.src[owner])
    end_bad = nonempty & (ed[last] != table.dst[owner])
    # adjacency between consecutive pairs of the same path
    pair_path = np.repeat(np.arange(P0, dtype=np.int64), hops)
    same = np.zeros(pe.shape[0], bool)
    if pe.size > 1:
        same[:-1] = pair_path[:-1] == pair_path[1:]
    adj_bad_pair = np.zeros(pe.shape[0], bool)
    if pe.size > 1:
        adj_bad_pair[:-1] = same[:-1] & (ed[safe[:-1]] != es[safe[1:]])
    ca = np.concatenate([[0], np.cumsum(adj_bad_pair)])
    n_adj = ca[pep[1:]] - ca[pep[:-1]]
    # simple: visited = [src(first)] + dst(each edge) must be unique per path
    nodes = np.concatenate([es[first][nonempty], ed[safe]])
    pid = np.concatenate([np.nonzero(nonempty)[0], pair_path])
    order = np.lexsort((nodes, pid))
    ns, ps = nodes[order], pid[order]
    dup = (ns[1:] == ns[:-1]) & (ps[1:] == ps[:-1])
    not_simple = np.zeros(P0, bool)
    not_simple[ps[1:][dup]] = True
    fail = (~nonempty) | (n_bad > 0) | start_bad | end_bad | (n_adj > 0) | not_simple
    if not fail.any():
        return
    p = int(np.flatnonzero(fail)[0])
    c = int(owner[p])
    i = p - int(cpp[c])
    key = table.key(c)
    pre = f"commodity {key}, path {i}: "
    seg = pe[pep[p]:pep[p + 1]]
    if hops[p] == 0:
        raise InputError(pre + "empty path")
    if n_bad[p]:
        e = int(seg[(seg < 0) | (seg >= m)][0])
        raise InputError(pre + f"edge id {e} out of range")
    if start_bad[p]:
        raise InputError(pre + f"does not start at {table.nodes[int(table.src[c])]!r}")
    if end_bad[p]:
        raise InputError(pre + f"does not end at {table.nodes[int(table.dst[c])]!r}")
    if n_adj[p]:
        for a, b in zip(seg[:-1], seg[1:]):
            if ed[a] != es[b]:
                raise InputError(pre + f"edges {int(a)} and {int(b)} are not adjacent")
    raise InputError(pre + "repeated node, path not simple")


def build_instance_flat(topology: Topology, table: CommodityTable, path_set, device=None) -> Instance:
    """Validate and build the GPU incidence store from columnar inputs."""
    flat = as_flat(path_set)
    if flat.num_commodities != len(table):
        raise InputError(f"path set covers {flat.num_commodities} commodities, expected {len(table)}")
    _validate_paths(topology, table, flat)
    dev = default_device() if device is None else int(device)
    cpp, pep, pe = _i64(flat.com_path_ptr), _i64(flat.path_edge_ptr), _i64(flat.path_edges)
    dem0 = _f64(table.demand)
    cap = _f64(topology.capacity).copy()
    h = C.c_void_p()
    check(lib().pf_instance_create(dev, len(table), topology.num_edges, _p(cpp, A.i64p), _p(pep, A.i64p),
                                   _p(pe, A.i64p), _p(dem0), _p(cap), C.byref(h)))
    handle = _Handle(h.value)
    sz = [C.c_int64() for _ in range(4)]
    check(lib().pf_instance_sizes(handle.ptr, *(C.byref(v) for v in sz)))
    sizes = tuple(int(v.value) for v in sz)
    keep = (dem0 > 0) & (np.diff(cpp) > 0)  # model.py:226-229 (same rule as the device)
    demand = dem0[keep].copy()
    return Instance(handle, topology, table, demand, cap, sizes, dev)


def build_instance_raw(capacity, demand0, com_path_ptr0, path_edge_ptr0, path_edges0, device=None) -> Instance:
    """Build from bare CSR arrays, skipping topology/path validation (trusted
    inputs such as generator output or fixtures).  Edge ids are still range
    checked on the device."""
    cap = _f64(capacity).copy()
    dem0 = _f64(demand0)
    cpp, pep, pe = _i64(com_path_ptr0), _i64(path_edge_ptr0), _i64(path_edges0)
    n = dem0.shape[0]
    names = tuple(f"v{i}" for i in range(2 * n)) if n < 100_000 else ("?",)
    if len(names) > 1:
        table = CommodityTable(names, np.arange(0, 2 * n, 2, dtype=np.int64),
                               np.arange(1, 2 * n, 2, dtype=np.int64), dem0)
    else:
        table = CommodityTable(names, np.zeros(n, np.int64), np.zeros(n, np.int64), dem0)
    dev = default_device() if device is None else int(device)
    h = C.c_void_p()
    check(lib().pf_instance_create(dev, n, cap.shape[0], _p(cpp, A.i64p), _p(pep, A.i64p), _p(pe, A.i64p),
                                   _p(dem0), _p(cap), C.byref(h)))
    handle = _Handle(h.value)
    sz = [C.c_int64() for _ in range(4)]
    check(lib().pf_instance_sizes(handle.ptr, *(C.byref(v) for v in sz)))
    keep = (dem0 > 0) & (np.diff(cpp) > 0)
    return Instance(handle, None, table, dem0[keep].copy(), cap, tuple(int(v.value) for v in sz), dev)


def build_instance(topology, commodities, path_set, device=None) -> Instance:
    """model.py:206-271 build_instance(topology, commodities, path_set)."""
    if not isinstance(commodities, CommodityTable):
        commodities = tuple(commodities)
    flat = as_flat(path_set)
    if flat.num_commodities != len(commodities):
        raise InputError(f"path set covers {flat.num_commodities} commodities, expected {len(commodities)}")
    table = (commodities if isinstance(commodities, CommodityTable)
             else CommodityTable.from_commodities(topology, commodities))
    return build_instance_flat(topology, table, flat, device)


def with_conditions(instance: Instance, capacity=None, demand=None) -> Instance:
    """model.py:274-294: same index spaces (shared on device), new capacity/demand."""
    cap = instance.capacity
    if capacity is not None:
        cap = _f64(capacity)
        if cap.shape != instance.capacity.shape:
            raise InputError("capacity vector length mismatch")
        if not np.all(np.isfinite(cap)) or np.any(cap < 0):
            raise InputError("capacities must be finite and >= 0")
    dem = instance.demand
    if demand is not None:
        dem = _f64(demand)
        if dem.shape != instance.demand.shape:
            raise InputError("demand vector length mismatch")
        if not np.all(np.isfinite(dem)) or np.any(dem < 0):
            raise InputError("demands must be finite and >= 0")
    h = C.c_void_p()
    check(lib().pf_instance_with_conditions(instance.handle, _p(cap), _p(dem), C.byref(h)))
    out = Instance(_Handle(h.value), instance.topology, instance._table, dem.copy(), cap.copy(),
                   instance._sizes, instance.device)
    for k in _INDEX_FIELDS:  # share exported host views too
        if k in instance.__dict__:
            out.__dict__[k] = instance.__dict__[k]
    return out


def _vec(a, n, what) -> np.ndarray:
    """Contiguous float64 copy of a length-n vector; a wrong length is an
    InputError (the native side copies exactly n doubles from the host)."""
    a = _f64(a)
    if a.shape != (n,):
        raise InputError(f"{what} length {a.shape} does not match {n}")
    return a


def commodity_sums(instance: Instance, rates) -> np.ndarray:
    """model.py:297-302 (device, reference reduction order)."""
    rates = _vec(rates, instance.num_paths, "rates")
    out = np.empty(instance.num_commodities)
    check(lib().pf_commodity_sums(instance.handle, _p(rates), _p(out)))
    return out


def edge_loads(instance: Instance, rates) -> np.ndarray:
    """model.py:305-311."""
    rates = _vec(rates, instance.num_paths, "rates")
    out = np.empty(instance.num_edges)
    check(lib().pf_edge_loads(instance.handle, _p(rates), _p(out)))
    return out


def edge_loads_from_pairs(instance: Instance, pair_values) -> np.ndarray:
    """model.py:314-319."""
    pv = _vec(pair_values, instance.num_pairs, "pair values")
    out = np.empty(instance.num_edges)
    check(lib().pf_edge_loads_from_pairs(instance.handle, _p(pv), _p(out)))
    return out


@dataclass(frozen=True)
class ViolationReport:
    """model.py:322-332."""

    feasible: bool
    edge_overload: np.ndarray
    commodity_excess: np.ndarray
    negative_count: int
    worst_negative: float
    pct_violated: float
    mean_relative_violation: float


def validate_allocation(instance: Instance, rates, tol=FEAS_TOL) -> ViolationReport:
    """model.py:335-369 (device)."""
    rates = _f64(rates)
    if rates.shape != (instance.num_paths,):
        raise InputError(f"rates length {rates.shape} does not match {instance.num_paths} paths")
    rep = A.Violation()
    ov = np.empty(instance.num_edges)
    ex = np.empty(instance.num_commodities)
    check(lib().pf_validate_allocation(instance.handle, _p(rates), float(tol), C.byref(rep), _p(ov), _p(ex)))
    return ViolationReport(feasible=rep.n_violated == 0, edge_overload=ov, commodity_excess=ex,
                           negative_count=int(rep.negative_count), worst_negative=float(rep.worst_negative),
                           pct_violated=float(rep.pct_violated),
                           mean_relative_violation=float(rep.mean_relative_violation))
