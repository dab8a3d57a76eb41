"""Host-side problem inputs: topology, commodities, path sets.

Mirrors the reference's input types (pathfair/model.py:20-132) with the same
names, fields, validation and error messages, plus a flat CSR path set
(`FlatPathSet`) so WAN-scale instances (millions of paths) never go through
nested Python tuples.  These are plain host data; the GPU incidence store is
built from them by `model.build_instance`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

FEAS_TOL = 1e-9  # model.py:17


class InputError(ValueError):
    """Invalid topology, demand, or path input (model.py:20-21)."""


@dataclass(frozen=True, eq=False)
class Topology:
    """Directed capacitated graph (model.py:24-60).  Edge order is load order
    with undirected rows expanded (reverse edge right after the forward one)."""

    nodes: tuple
    edge_src: np.ndarray
    edge_dst: np.ndarray
    capacity: np.ndarray
    weight: np.ndarray

    @property
    def num_nodes(self):
        return len(self.nodes)

    @property
    def num_edges(self):
        return int(self.edge_src.shape[0])

    def node_index(self):
        return {name: i for i, name in enumerate(self.nodes)}

    def edge_index(self):
        return {(self.nodes[self.edge_src[e]], self.nodes[self.edge_dst[e]]): e
                for e in range(self.num_edges)}

    def edge_names(self, e):
        return self.nodes[self.edge_src[e]], self.nodes[self.edge_dst[e]]


def build_topology(rows):
    """model.py:62-102: (src, dst, capacity, weight[, undirected]) rows -> Topology."""
    expanded = []
    for n, row in enumerate(rows):
        if len(row) == 4:
            src, dst, cap, w = row
            undirected = False
        elif len(row) == 5:
            src, dst, cap, w, undirected = row
        else:
            raise InputError(f"edge row {n}: expected 4 or 5 fields, got {len(row)}")
        src, dst = str(src), str(dst)
        cap, w = float(cap), float(w)
        if src == dst:
            raise InputError(f"edge row {n}: self-loop {src!r}")
        if not np.isfinite(cap) or cap < 0:
            raise InputError(f"edge row {n}: capacity must be finite and >= 0, got {cap}")
        if not np.isfinite(w) or w <= 0:
            raise InputError(f"edge row {n}: weight must be finite and > 0, got {w}")
        expanded.append((src, dst, cap, w))
        if undirected:
            expanded.append((dst, src, cap, w))
    seen = set()
    for src, dst, _, _ in expanded:
        if (src, dst) in seen:
            raise InputError(f"duplicate edge {src!r} -> {dst!r}")
        seen.add((src, dst))
    names = sorted({n for e in expanded for n in e[:2]})
    index = {name: i for i, name in enumerate(names)}
    m = len(expanded)
    return Topology(
        tuple(names),
        np.fromiter((index[e[0]] for e in expanded), np.int64, m),
        np.fromiter((index[e[1]] for e in expanded), np.int64, m),
        np.fromiter((e[2] for e in expanded), np.float64, m),
        np.fromiter((e[3] for e in expanded), np.float64, m),
    )


@dataclass(frozen=True)
class Commodity:
    """model.py:105-121."""

    src: str
    dst: str
    demand: float

    def __post_init__(self):
        if self.src == self.dst:
            raise InputError(f"commodity {self.src!r} -> {self.dst!r}: src == dst")
        d = float(self.demand)
        if not np.isfinite(d) or d < 0:
            raise InputError(f"commodity {self.src!r} -> {self.dst!r}: bad demand {self.demand}")
        object.__setattr__(self, "demand", d)

    @property
    def key(self):
        return f"{self.src}→{self.dst}"


@dataclass(frozen=True)
class PathSet:
    """paths[c][i] is the i-th path of commodity c as a tuple of edge ids (model.py:124-132)."""

    paths: tuple

    @classmethod
    def from_lists(cls, lists):
        return cls(tuple(tuple(tuple(int(e) for e in p) for p in per_com) for per_com in lists))

    def to_flat(self) -> "FlatPathSet":
        counts = np.fromiter((len(pc) for pc in self.paths), np.int64, len(self.paths))
        cpp = np.zeros(len(self.paths) + 1, np.int64)
        np.cumsum(counts, out=cpp[1:])
        flat = [p for pc in self.paths for p in pc]
        hops = np.fromiter((len(p) for p in flat), np.int64, len(flat))
        pep = np.zeros(len(flat) + 1, np.int64)
        np.cumsum(hops, out=pep[1:])
        pe = (np.fromiter((e for p in flat for e in p), np.int64, int(pep[-1]))
              if len(flat) else np.zeros(0, np.int64))
        return FlatPathSet(cpp, pep, pe)


@dataclass(frozen=True, eq=False)
class FlatPathSet:
    """CSR path set: commodity c owns paths [com_path_ptr[c], com_path_ptr[c+1]);
    path p is edges path_edges[path_edge_ptr[p]:path_edge_ptr[p+1]]."""

    com_path_ptr: np.ndarray
    path_edge_ptr: np.ndarray
    path_edges: np.ndarray

    @property
    def num_commodities(self):
        return int(self.com_path_ptr.shape[0] - 1)

    @property
    def paths(self):
        """Nested-tuple view (PathSet.paths layout); O(P) Python objects."""
        cpp, pep, pe = self.com_path_ptr, self.path_edge_ptr, self.path_edges
        return tuple(
            tuple(tuple(int(e) for e in pe[pep[p]:pep[p + 1]]) for p in range(cpp[c], cpp[c + 1]))
            for c in range(self.num_commodities))


def as_flat(path_set) -> FlatPathSet:
    if isinstance(path_set, FlatPathSet):
        return path_set
    if isinstance(path_set, PathSet):
        return path_set.to_flat()
    return PathSet.from_lists(path_set).to_flat()


@dataclass(frozen=True, eq=False)
class CommodityTable:
    """Columnar commodity list: src/dst node ids and demands (O(1) Python objects)."""

    nodes: tuple
    src: np.ndarray
    dst: np.ndarray
    demand: np.ndarray

    def __len__(self):
        return int(self.demand.shape[0])

    def __getitem__(self, i):
        return Commodity(self.nodes[int(self.src[i])], self.nodes[int(self.dst[i])], float(self.demand[i]))

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]

    def key(self, i):
        return f"{self.nodes[int(self.src[i])]}→{self.nodes[int(self.dst[i])]}"

    @classmethod
    def from_commodities(cls, topology, commodities):
        coms = tuple(commodities)
        index = topology.node_index()
        for com in coms:
            if com.src not in index or com.dst not in index:
                raise InputError(f"commodity {com.key}: unknown node")
        n = len(coms)
        return cls(topology.nodes,
                   np.fromiter((index[c.src] for c in coms), np.int64, n),
                   np.fromiter((index[c.dst] for c in coms), np.int64, n),
                   np.fromiter((c.demand for c in coms), np.float64, n))
