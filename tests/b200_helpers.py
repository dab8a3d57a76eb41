"""Instance builders for the GPU tests, mirroring the reference's
tests/helpers.py:16-62 builders through this package's public API, plus
loaders for the golden fixtures."""

import numpy as np

import golden_io as G
import paper_2605_01748_b200 as pf


def make_instance(edges, commodities):
    topo = pf.build_topology(edges)
    coms = [pf.Commodity(s, d, dem) for s, d, dem, _ in commodities]
    ps = pf.PathSet.from_lists([paths for _, _, _, paths in commodities])
    return pf.build_instance(topo, coms, ps)


def single_bottleneck(cap=10.0, demand=20.0):
    return make_instance([("A", "B", cap, 1)], [("A", "B", demand, [(0,)])])


def shared_edge(n=2, cap=10.0, demand=20.0):
    edges = [(f"s{i}", "M", 10 * n * max(cap, demand), 1) for i in range(n)]
    edges.append(("M", "T", cap, 1))
    coms = [(f"s{i}", "T", demand, [(i, n)]) for i in range(n)]
    return make_instance(edges, coms)


def chain(demand=100.0):
    return make_instance(
        [("A", "B", 10, 1), ("B", "C", 5, 1)],
        [("A", "B", demand, [(0,)]), ("A", "C", demand, [(0, 1)]), ("B", "C", demand, [(1,)])],
    )


def diamond(demand=20.0, cap_top=4.0, cap_bottom=8.0):
    return make_instance(
        [("A", "T", cap_top, 1), ("T", "B", cap_top, 1), ("A", "U", cap_bottom, 1), ("U", "B", cap_bottom, 1)],
        [("A", "B", demand, [(0, 1), (2, 3)])],
    )


SMALL_BUILDERS = {
    "single_bottleneck": lambda: single_bottleneck(),
    "shared_edge2": lambda: shared_edge(n=2),
    "shared_edge3": lambda: shared_edge(n=3),
    "chain": lambda: chain(),
    "diamond": lambda: diamond(),
}


def golden_instance(prefix):
    f = G.flat_inputs(prefix)
    return pf.build_instance_raw(f["capacity"], f["demand0"], f["com_path_ptr0"], f["path_edge_ptr0"],
                                 f["path_edges0"])


def oracle_instance(prefix):
    from oracle import oracle as O
    f = G.flat_inputs(prefix)
    return O.build_instance(f["capacity"], f["demand0"], f["com_path_ptr0"], f["path_edge_ptr0"],
                            f["path_edges0"])


def generated(n, k, vol_frac, seed=None):
    """A config built with this package's generators (pinned to the reference's)."""
    topo = pf.random_topology(n, seed=n if seed is None else seed)
    tab = pf.gravity_table(topo, vol_frac * float(topo.capacity.sum()))
    ps = pf.k_shortest_paths(topo, tab, k)
    return topo, tab, ps
