"""Synthetic input generators (input preparation, not the hot path).

Restatements of the reference's generators so that configs 1-3 can be built
on a box without the reference or networkx:

* `random_topology`  -- pathfair/harness.py:200-239 (same numpy RNG call order);
* `gravity_demands`  -- pathfair/harness.py:179-197 (same float op order), plus a
  columnar `gravity_table` that skips per-commodity Python objects;
* `k_shortest_paths` -- pathfair/harness.py:138-176, computed by the native Yen
  implementation in csrc/ksp.cpp (OpenMP), returning a `FlatPathSet`.

All three are pinned against fixtures produced by the reference
(tests/test_generators.py).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .topology import CommodityTable, FlatPathSet, InputError, build_topology


def random_topology(num_nodes, seed, extra_edge_fraction=0.5, capacity_range=(50.0, 200.0),
                    weight_range=(1.0, 10.0)):
    """Ring plus random chords, undirected, uniform capacity/weight (harness.py:200-239)."""
    if num_nodes < 2:
        raise InputError("need at least 2 nodes")
    rng = np.random.default_rng(seed)
    width = len(str(num_nodes - 1))
    names = [f"n{i:0{width}d}" for i in range(num_nodes)]
    pairs = []
    seen = set()
    for i in range(num_nodes):
        a, b = i, (i + 1) % num_nodes
        key = (min(a, b), max(a, b))
        if key not in seen:
            seen.add(key)
            pairs.append(key)
    want = int(round(extra_edge_fraction * num_nodes))
    attempts = 0
    added = 0
    while added < want and attempts < 50 * max(want, 1):
        attempts += 1
        a, b = rng.integers(0, num_nodes, 2)
        if a == b:
            continue
        key = (min(int(a), int(b)), max(int(a), int(b)))
        if key in seen:
            continue
        seen.add(key)
        pairs.append(key)
        added += 1
    rows = []
    for a, b in pairs:
        cap = float(rng.uniform(*capacity_range))
        wgt = float(rng.uniform(*weight_range))
        rows.append((names[a], names[b], cap, wgt, True))
    return build_topology(rows)


def _gravity_weights(topology, total_volume):
    if topology.num_nodes < 2:
        raise InputError("gravity model needs at least 2 nodes")
    if total_volume <= 0:
        raise InputError("total_volume must be > 0")
    w = np.zeros(topology.num_nodes)
    np.add.at(w, topology.edge_src, topology.capacity)
    np.add.at(w, topology.edge_dst, topology.capacity)
    z = float(w.sum() ** 2 - (w ** 2).sum())
    if z <= 0:
        raise InputError("gravity model undefined: no positive capacity")
    return w, z


def gravity_table(topology, total_volume) -> CommodityTable:
    """All ordered pairs s != t in node order with D = V*w_s*w_t/z (harness.py:179-197)."""
    w, z = _gravity_weights(topology, total_volume)
    n = topology.num_nodes
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    mask = ii != jj
    src, dst = ii[mask].astype(np.int64), jj[mask].astype(np.int64)
    demand = float(total_volume) * w[src] * w[dst] / z
    if not np.all(np.isfinite(demand)) or np.any(demand < 0):
        raise InputError("gravity model produced a bad demand")
    return CommodityTable(topology.nodes, src, dst, demand)


def gravity_demands(topology, total_volume):
    """List of Commodity objects, as the reference returns (harness.py:179-197)."""
    return list(gravity_table(topology, total_volume))


def k_shortest_paths(topology, commodities, k=4, threads=None) -> FlatPathSet:
    """Up to k loopless shortest paths per commodity ordered by (weight, edge tuple);
    unreachable pairs get zero paths (harness.py:138-176).  Native host code
    (csrc/ksp.cpp in libpf_gen.so, include/pf_gen.h)."""
    if k < 1:
        raise InputError("k must be >= 1")
    from ._lib import gen_lib

    if not isinstance(commodities, CommodityTable):
        commodities = CommodityTable.from_commodities(topology, commodities)
    L = gen_lib()
    es = np.ascontiguousarray(topology.edge_src, np.int64)
    ed = np.ascontiguousarray(topology.edge_dst, np.int64)
    wt = np.ascontiguousarray(topology.weight, np.float64)
    cap = np.ascontiguousarray(topology.capacity, np.float64)
    cs = np.ascontiguousarray(commodities.src, np.int64)
    cd = np.ascontiguousarray(commodities.dst, np.int64)
    i64 = C.POINTER(C.c_int64)
    f64 = C.POINTER(C.c_double)
    nthr = int(threads if threads is not None else os.cpu_count() or 1)
    h = L.pf_ksp_run(topology.num_nodes, es.shape[0], es.ctypes.data_as(i64), ed.ctypes.data_as(i64),
                     wt.ctypes.data_as(f64), cap.ctypes.data_as(f64), cs.shape[0], cs.ctypes.data_as(i64),
                     cd.ctypes.data_as(i64), int(k), nthr)
    if not h:
        raise InputError("k_shortest_paths: bad arguments")
    try:
        P, NP = C.c_int64(), C.c_int64()
        L.pf_ksp_sizes(h, C.byref(P), C.byref(NP))
        cpp = np.empty(cs.shape[0] + 1, np.int64)
        pep = np.empty(P.value + 1, np.int64)
        pe = np.empty(NP.value, np.int64)
        L.pf_ksp_export(h, cpp.ctypes.data_as(i64), pep.ctypes.data_as(i64), pe.ctypes.data_as(i64))
    finally:
        L.pf_ksp_free(h)
    return FlatPathSet(cpp, pep, pe)
