"""Parity at the benchmarked scales (SURVEY 8(d) gates), on the GPU through
the C-ABI, against the C oracle (the reference's exact operation order,
pinned to the reference by tests/golden/).

* config 2 (the bench workload, 18.3M pairs): exact mode bitwise equal to
  the oracle in every state array after iterations 1, 2, 3 and 10;
* the reference algorithm's fixed points (tests/golden/golden_fixed_points.*,
  made by the oracle with make_golden_fixed_points.py) on config 1, the
  north-star 500-node k=4 instance and config 2 at V = 0.3 x capacity, run
  to the stagnation stop or the 5,000-iteration cap:
  - exact mode: the same stop, the raw iterate and the projected rates
    bitwise (alpha <= 1 there; cfg1 ends at alpha 2 and is checked to 1e-9);
  - fast mode (the timed path): the same stop (iteration count, alpha),
    a feasible allocation and the sorted post-projection commodity sums
    within 1e-4 relative of the oracle's at equal iteration count;
* config 3 (2000 nodes, E = 6,000, the large-E layout): a 10,000-commodity
  sample -- incidence bit-exact vs the oracle, fused iterations 1-3 within
  1e-9 of the exact-order path.
"""

import json
import os

import numpy as np
import pytest

import golden_io as G

pytestmark = pytest.mark.gpu

pf = pytest.importorskip("paper_2605_01748_b200")

FP_JSON = os.path.join(G.GOLDEN, "golden_fixed_points.json")
FP_NPZ = os.path.join(G.GOLDEN, "golden_fixed_points.npz")
INSTANCES = {"cfg1_v0.3": (40, 4, 0.3), "target_k4_v0.3": (500, 4, 0.3), "cfg2_v0.3": (500, 8, 0.3)}
STATE = (("x", "x"), ("y", "y"), ("dual_demand", "dual_demand"), ("dual_capacity", "dual_capacity"),
         ("dual_consensus", "dual_consensus"), ("dual_nonneg", "dual_nonneg"))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _fixed_points():
    if not os.path.exists(FP_JSON):
        pytest.skip("golden_fixed_points not generated")
    with open(FP_JSON) as fh:
        meta = json.load(fh)
    return meta, dict(np.load(FP_NPZ))


def _build(n, k, vol, oracle=False):
    from b200_helpers import generated
    topo, tab, ps = generated(n, k, vol)
    inst = pf.build_instance_flat(topo, tab, ps, device=0)
    if not oracle:
        return inst, None
    from oracle import oracle as O
    return inst, O.build_instance(topo.capacity, tab.demand, ps.com_path_ptr, ps.path_edge_ptr, ps.path_edges)


def test_exact_cfg2_bitwise_vs_oracle():
    """18,282,422 pairs, 53k-term sequential per-edge chains, int32 device
    indexing: every state array bitwise after iterations 1, 2, 3 and 10."""
    from oracle import oracle as O
    inst, I = _build(500, 8, 1.5, oracle=True)
    assert inst.num_pairs == I.num_pairs == 18282422
    ex = pf.Solver(inst, pf.SolverConfig(mode="exact")).init()
    loop = O.Loop(I, O.make_config())
    done = 0
    for it in (1, 2, 3, 10):
        ex.run(it - done)
        loop.step(it - done)
        done = it
        a, b = ex.state(), loop.state()
        assert a.iteration == b.iteration == it
        assert a.beta == b.beta and a.alpha == b.alpha, it
        for fa, fb in STATE:
            assert np.array_equal(getattr(a, fa), getattr(b, fb)), (it, fa)


@pytest.mark.parametrize("name", list(INSTANCES))
def test_exact_reaches_the_oracle_fixed_point(name):
    meta, arrs = _fixed_points()
    if name not in meta:
        pytest.skip(f"{name} not in golden_fixed_points")
    m = meta[name]
    inst, _ = _build(*INSTANCES[name])
    assert (inst.num_commodities, inst.num_paths, inst.num_pairs) == (m["commodities"], m["paths"], m["pairs"])
    s = pf.Solver(inst, pf.SolverConfig(mode="exact")).init()
    s.run(m["iterations"] + 1)
    r = s.result()
    assert (int(r.iterations), int(r.alpha), bool(r.converged)) == (m["iterations"], m["alpha"], m["converged"])
    x = s.x()
    rates, sums = s.finish()
    want = arrs[f"{name}/opt_sums"]
    if m["alpha"] <= 1:
        assert G.digest(x) == m["raw_x_digest"]
        assert G.digest(rates) == m["rates_digest"]
        assert np.array_equal(sums, want)
    else:  # alpha >= 2: CUDA pow vs glibc pow in the Newton roots
        np.testing.assert_allclose(sums, want, rtol=1e-9, atol=1e-9 * float(want.max()))


@pytest.mark.parametrize("name", list(INSTANCES))
def test_fast_matches_the_oracle_at_equal_iterations(name):
    """The timed path against the reference algorithm: same stop, feasible,
    sorted post-projection sums within 1e-4 relative (north_star tolerance)."""
    meta, arrs = _fixed_points()
    if name not in meta:
        pytest.skip(f"{name} not in golden_fixed_points")
    m = meta[name]
    inst, _ = _build(*INSTANCES[name])
    res = pf.solve(inst, pf.SolverConfig(mode="fast"))
    assert res.mode == "fast"
    assert pf.validate_allocation(inst, res.rates).feasible
    want = np.sort(arrs[f"{name}/opt_sums"])
    got = np.sort(res.sums)
    if m["converged"]:
        # stagnation stops are a residual threshold: the iteration may differ by a few
        assert res.converged and res.alpha == m["alpha"]
        assert abs(res.iterations - m["iterations"]) <= 0.05 * m["iterations"]
    else:
        assert (res.iterations, res.alpha, res.converged) == (m["iterations"], m["alpha"], False)
    scale = float(want.max())
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-4 * scale)
    # and the objective the trace reports (the utility of the sorted vector)
    theta = m["theta"]
    assert pf.optimality_from_sums(res.sums, arrs[f"{name}/opt_sums"], theta) >= 0.999


def test_cfg3_sample_incidence_and_fused_iterations():
    """Config 3's topology (2000 nodes, 6,000 edges: the large-E layout) with a
    10,000-commodity sample of its all-pairs gravity demands, k = 8."""
    from oracle import oracle as O
    topo = pf.random_topology(2000, seed=2000)
    tab = pf.gravity_table(topo, 1.5 * float(topo.capacity.sum()))
    pick = np.sort(np.random.default_rng(11).choice(len(tab), 10000, replace=False))
    sub = pf.CommodityTable(tab.nodes, tab.src[pick], tab.dst[pick], tab.demand[pick])
    ps = pf.k_shortest_paths(topo, sub, 8)
    inst = pf.build_instance_flat(topo, sub, ps, device=0)
    I = O.build_instance(topo.capacity, sub.demand, ps.com_path_ptr, ps.path_edge_ptr, ps.path_edges)
    for f in G.INCIDENCE:
        got = inst.demand if f == "demand" else getattr(inst, f)
        assert np.array_equal(np.asarray(got), getattr(I, f)), f
    assert inst.num_edges == 6000
    ex = pf.Solver(inst, pf.SolverConfig(mode="exact")).init()
    fa = pf.Solver(inst, pf.SolverConfig(mode="fast")).init()
    loop = O.Loop(I, O.make_config())
    for it in (1, 2, 3):
        ex.run(1)
        fa.run(1)
        loop.step(1)
        a, b, o = ex.state(), fa.state(), loop.state()
        assert a.iteration == b.iteration == o.iteration == it
        assert a.beta == b.beta == o.beta and a.alpha == b.alpha == o.alpha
        xs = float(np.max(np.abs(a.x)))
        for fa_, fb in STATE:
            want, got = getattr(a, fa_), getattr(b, fa_)
            assert np.array_equal(want, getattr(o, fb)), (it, fa_)  # exact == oracle, bitwise
            scale = max(float(np.max(np.abs(want))), xs)
            assert float(np.max(np.abs(got - want))) <= 1e-9 * scale, (it, fa_)


@pytest.mark.parametrize("name", ["cfg1_v0.3", "target_k4_v0.3"])
def test_time_to_quality_one_device_pass(name):
    """f3: k* found in one device pass (sampled post-projection optimality,
    crossing chunk replayed from a snapshot) equals the first traced row whose
    optimality column (controller.py:176-183, one projection per row) reaches
    0.99; every sample is bitwise that row's optimality; the solver stands
    bitwise where a fresh solver run to k* stands."""
    meta, arrs = _fixed_points()
    if name not in meta:
        pytest.skip(f"{name} not in golden_fixed_points")
    m = meta[name]
    inst, _ = _build(*INSTANCES[name])
    opt = arrs[f"{name}/opt_sums"]
    dev = pf.Solver(inst, pf.SolverConfig(mode="fast", max_iterations=5000)).init()
    found = dev.time_to_quality(opt, 0.99, sample_every=64)
    k = found["k_star"]
    assert k is not None and abs(k - m["k_star"]) <= 0.02 * m["k_star"], (k, m["k_star"])
    assert dev.result().iterations == k
    # the per-row instrument (a projection and the metric per traced row)
    tr2 = pf.Solver(inst, pf.SolverConfig(mode="fast", max_iterations=5000, trace=True, reference_sums=opt)).init()
    tr2.run(k)
    rows = {r.iteration: r.optimality for r in tr2.trace()}
    first = min(i for i, q in rows.items() if q >= 0.99)
    assert first == k
    for it, q in found["samples"]:
        if it in rows:
            assert q == rows[it], (it, q, rows[it])
    ref = pf.Solver(inst, pf.SolverConfig(mode="fast", max_iterations=5000)).init()
    ref.run(k)
    assert np.array_equal(ref.x(), dev.x())


def test_time_to_quality_edges():
    """pf_solver_time_to_quality's edge behaviour: an unreachable target runs
    to the controller's stop and reports no k*; an exact-mode solver is refused
    (the search replays fused-kernel snapshots); a reference vector of the
    wrong length is an InputError."""
    from b200_helpers import generated
    topo, tab, ps = generated(24, 4, 0.3)
    inst = pf.build_instance(topo, tab, ps, device=0)
    ref = pf.solve(inst, pf.SolverConfig(mode="exact")).sums
    s = pf.Solver(inst, pf.SolverConfig(mode="fast", max_iterations=300)).init()
    out = s.time_to_quality(ref, 1.5, sample_every=16)
    assert out["k_star"] is None
    assert out["iterations"] == int(s.result().iterations) <= 300
    assert len(out["samples"]) >= 1 and all(q <= 1.0 for _, q in out["samples"])
    ex = pf.Solver(inst, pf.SolverConfig(mode="exact")).init()
    with pytest.raises(pf.InputError):
        ex.time_to_quality(ref, 0.99)
    with pytest.raises(pf.InputError):
        pf.Solver(inst, pf.SolverConfig(mode="fast")).init().time_to_quality(ref[:-1], 0.99)
