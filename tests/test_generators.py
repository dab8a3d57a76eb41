"""Input generators vs the reference's own (fixtures from make_golden.py). CPU only.

random_topology / gravity_demands: bitwise (harness.py:179-239).
k_shortest_paths (native Yen, csrc/ksp.cpp): identical path sets and order to
networkx-based harness.py:138-176 on all cfg1 commodities (k=4), a 300-commodity
sample of the 500-node WAN (k=1 and k=8), and a topology with failed links.
"""

import numpy as np
import pytest

import golden_io as G
from paper_2605_01748_b200 import harness as H
from paper_2605_01748_b200.topology import CommodityTable, InputError, build_topology


@pytest.mark.parametrize("n", [40, 500])
def test_random_topology_and_gravity_bitwise(n):
    A, D = G.arrays(), G.digests()
    topo = H.random_topology(n, seed=n)
    for f in ("edge_src", "edge_dst", "capacity", "weight"):
        assert np.array_equal(getattr(topo, f), A[f"gen/n{n}/{f}"]), f
    assert list(topo.nodes) == list(A[f"gen/n{n}/nodes"])
    tab = H.gravity_table(topo, 1.5 * float(topo.capacity.sum()))
    assert G.digest(tab.demand) == D[f"gen/n{n}/gravity"]
    coms = H.gravity_demands(topo, 1.5 * float(topo.capacity.sum()))
    assert np.array_equal([c.demand for c in coms[:64]], A[f"gen/n{n}/gravity_head"])


def _eq(ps, prefix):
    A = G.arrays()
    assert np.array_equal(ps.com_path_ptr, A[f"{prefix}/com_path_ptr"])
    assert np.array_equal(ps.path_edge_ptr, A[f"{prefix}/path_edge_ptr"])
    assert np.array_equal(ps.path_edges, A[f"{prefix}/path_edges"])


def test_ksp_cfg1_all_commodities():
    f = G.flat_inputs("cfg1_v0.3")
    topo = H.random_topology(40, seed=40)
    ps = H.k_shortest_paths(topo, H.gravity_table(topo, 0.3 * float(topo.capacity.sum())), 4)
    assert np.array_equal(ps.com_path_ptr, f["com_path_ptr0"])
    assert np.array_equal(ps.path_edge_ptr, f["path_edge_ptr0"])
    assert np.array_equal(ps.path_edges, f["path_edges0"])


@pytest.mark.parametrize("k", [1, 8])
def test_ksp_500_node_sample(k):
    A = G.arrays()
    topo = H.random_topology(500, seed=500)
    tab = H.gravity_table(topo, 1.5 * float(topo.capacity.sum()))
    pick = A[f"gen/n500/ksp{k}/pick"]
    sub = CommodityTable(tab.nodes, tab.src[pick], tab.dst[pick], tab.demand[pick])
    _eq(H.k_shortest_paths(topo, sub, k), f"gen/n500/ksp{k}")


def test_ksp_skips_failed_links_and_k1():
    A = G.arrays()
    topo = H.random_topology(40, seed=40)
    rows = []
    for e in range(topo.num_edges):
        s, t = topo.edge_names(e)
        rows.append((s, t, 0.0 if e in (3, 17, 40) else float(topo.capacity[e]), float(topo.weight[e])))
    cut = build_topology(rows)
    assert np.array_equal(cut.capacity, A["gen/n40cut/capacity"])
    coms = H.gravity_demands(topo, 1.0)
    _eq(H.k_shortest_paths(cut, coms, 4), "gen/n40cut/ksp4")
    ps1 = H.k_shortest_paths(topo, coms, 1)
    assert np.array_equal(ps1.path_edges, A["gen/n40/ksp1/path_edges"])
    assert np.array_equal(ps1.path_edge_ptr, A["gen/n40/ksp1/path_edge_ptr"])


def test_generator_input_errors():
    with pytest.raises(InputError):
        H.random_topology(1, seed=0)
    topo = H.random_topology(5, seed=5)
    with pytest.raises(InputError):
        H.gravity_table(topo, 0.0)
    with pytest.raises(InputError):
        H.k_shortest_paths(topo, H.gravity_demands(topo, 1.0), 0)


def _golden_ksp():
    import json
    import os
    p = os.path.join(G.GOLDEN, "golden_ksp.json")
    if not os.path.exists(p):
        pytest.skip("golden_ksp.json not generated")
    with open(p) as fh:
        return json.load(fh)


def _chunk_digests(topo, tab, idx_chunks, k):
    import hashlib
    out = []
    for idx in idx_chunks:
        sub = CommodityTable(tab.nodes, tab.src[idx], tab.dst[idx], tab.demand[idx])
        ps = H.k_shortest_paths(topo, sub, k)
        h = hashlib.sha256()
        for a in (ps.com_path_ptr, ps.path_edge_ptr, ps.path_edges):
            h.update(np.ascontiguousarray(a, np.int64).tobytes())
        out.append(h.hexdigest()[:32])
    return out


def test_ksp_config2_all_commodities_vs_networkx():
    """SURVEY 8(f)#2 gate: all 249,500 commodities of config 2 (k = 8) give
    path sets identical to the reference's networkx k_shortest_paths
    (harness.py:138-176), chunk by chunk (tests/golden/make_golden_ksp.py)."""
    g = _golden_ksp()
    topo = H.random_topology(500, seed=500)
    tab = H.gravity_table(topo, 1.0)
    C = len(tab)
    assert C == g["cfg2"]["commodities"]
    ch = g["chunk"]
    chunks = [np.arange(s, min(C, s + ch)) for s in range(0, C, ch)]
    got = _chunk_digests(topo, tab, chunks, g["k"])
    bad = [i for i, (a, b) in enumerate(zip(got, g["cfg2"]["digests"])) if a != b]
    assert not bad, f"chunks differing from networkx: {bad[:10]}"
    full = H.k_shortest_paths(topo, tab, g["k"])
    assert full.path_edge_ptr.shape[0] - 1 == g["cfg2"]["paths"] and full.path_edges.shape[0] == g["cfg2"]["pairs"]


def test_ksp_config3_sample_vs_networkx():
    """10,000 commodities of config 3 (2000 nodes, 6,000 edges, k = 8)."""
    g = _golden_ksp()["cfg3_sample"]
    topo = H.random_topology(2000, seed=2000)
    tab = H.gravity_table(topo, 1.0)
    assert len(tab) == g["commodities_total"]
    pick = np.sort(np.random.default_rng(g["seed"]).choice(len(tab), g["size"], replace=False))
    chunks = [pick[s:s + g["chunk"]] for s in range(0, pick.size, g["chunk"])]
    assert _chunk_digests(topo, tab, chunks, 8) == g["digests"]
