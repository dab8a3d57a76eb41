"""GPU parity: the CUDA path (through the C-ABI) against the reference fixtures
and the C oracle.  Run on a B200 with `pytest -m gpu`.

Bars:
  * incidence / index spaces: bit-exact;
  * exact mode (PF_MODE_EXACT): bitwise state at every snapshot for alpha <= 1,
    1e-9 relative where numpy's SIMD pow enters (alpha >= 2);
  * fast mode (fused kernel): iteration-1 state within 1e-12, same controller
    decisions, converged sorted sums within 1e-4 relative, feasible output.
"""

import types

import numpy as np
import pytest

import golden_io as G
import states
from b200_helpers import SMALL_BUILDERS, chain, golden_instance, oracle_instance, shared_edge, single_bottleneck

pytestmark = pytest.mark.gpu

pf = pytest.importorskip("paper_2605_01748_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


# ------------------------------------------------------------------ incidence


@pytest.mark.parametrize("name", G.SMALL)
def test_incidence_small_bitexact(name):
    inst = SMALL_BUILDERS[name]()
    A = G.arrays()
    for f in G.INCIDENCE:
        got = getattr(inst, f) if f != "demand" else inst.demand
        assert np.array_equal(np.asarray(got), A[f"small/{name}/inc/{f}"]), f


@pytest.mark.parametrize("tag", ["cfg1_v0.3", "cfg1_v1.5"])
def test_incidence_cfg1_bitexact(tag):
    inst = golden_instance(tag)
    D = G.digests()
    for f in G.INCIDENCE:
        arr = inst.demand if f == "demand" else getattr(inst, f)
        dt = np.float64 if f == "demand" else np.int64
        assert G.digest(np.asarray(arr, dt)) == D[f"{tag}/inc/{f}"], f


def test_incidence_with_drops_matches_oracle():
    """Zero-demand and pathless commodities are dropped exactly as model.py:226-229."""
    from oracle import oracle as O
    topo = pf.random_topology(30, seed=3)
    tab = pf.gravity_table(topo, 100.0)
    ps = pf.k_shortest_paths(topo, tab, 3)
    dem = tab.demand.copy()
    dem[::7] = 0.0
    cpp = ps.com_path_ptr.copy()
    inst = pf.build_instance_raw(topo.capacity, dem, cpp, ps.path_edge_ptr, ps.path_edges)
    ref = O.build_instance(topo.capacity, dem, cpp, ps.path_edge_ptr, ps.path_edges)
    for f in G.INCIDENCE:
        got = inst.demand if f == "demand" else getattr(inst, f)
        assert np.array_equal(np.asarray(got), getattr(ref, f)), f


def test_incidence_500_node_wan_matches_oracle():
    """Config 2 (500-node all-pairs, k=8): 18.3M pairs, bit-exact index spaces."""
    from oracle import oracle as O
    topo, tab, ps = pytest.importorskip("b200_helpers").generated(500, 8, 1.5)
    inst = pf.build_instance_raw(topo.capacity, tab.demand, ps.com_path_ptr, ps.path_edge_ptr, ps.path_edges)
    ref = O.build_instance(topo.capacity, tab.demand, ps.com_path_ptr, ps.path_edge_ptr, ps.path_edges)
    assert (inst.num_commodities, inst.num_paths, inst.num_edges, inst.num_pairs) == (249500, 1996000, 1500,
                                                                                     18282422)
    for f in G.INCIDENCE:
        got = inst.demand if f == "demand" else getattr(inst, f)
        assert np.array_equal(np.asarray(got), getattr(ref, f)), f


# ------------------------------------------------------------------ kernel level


def _kernel_check(tag, inst):
    A, D = G.arrays(), G.digests()
    cases = states.kernel_case_states(inst.num_commodities, inst.num_paths, inst.num_edges, inst.num_pairs,
                                      G.kernel_seed(tag))
    for i, (arrs, beta, alpha) in enumerate(cases):
        key = f"{tag}/k{i}"
        st = pf.SolverState(**{k: v.copy() for k, v in arrs.items()}, beta=beta, alpha=alpha, iteration=0)
        dd, dc, dcon, dn = pf.update_duals(st, inst)
        sd, sc = pf.update_slacks(st, inst)
        got = dict(dd=dd, dc=dc, dcon=dcon, dn=dn, sd=sd, sc=sc)
        st.dual_demand, st.dual_capacity, st.dual_consensus, st.dual_nonneg = dd, dc, dcon, dn
        st.y = pf.update_rate_suggestions(st, inst)
        got["y"] = st.y
        sums = pf.solve_commodity_sums(st, inst, alpha)
        got["sums"] = sums
        got["x"] = pf.update_rates(st, inst, sums, alpha)
        for nm, a in got.items():
            if alpha >= 2 and nm in ("sums", "x"):
                # CUDA pow vs glibc (roots) and numpy SIMD pow (gain); Newton stops at
                # |f| <= 1e-10 max(1,|q|), and x = w (K + ct) can cancel: scale by max|x|
                want = A[f"{key}/out/{nm}"]
                np.testing.assert_allclose(a, want, rtol=1e-9, atol=1e-9 * float(np.abs(want).max()))
            else:
                assert G.digest(a) == D[f"{key}/out/{nm}"], (key, nm)


@pytest.mark.parametrize("name", G.SMALL)
def test_kernels_small_bitwise(name):
    _kernel_check(f"small/{name}", SMALL_BUILDERS[name]())


def test_kernels_cfg1_bitwise():
    _kernel_check("cfg1_v0.3", golden_instance("cfg1_v0.3"))


def test_roots_vs_reference():
    A = G.arrays()
    got = np.array([pf.solve_sum_equation(w, b, q, int(a)) for w, b, q, a in
                    zip(A["roots/w"], A["roots/beta"], A["roots/q"], A["roots/alpha"])])
    al = A["roots/alpha"]
    lo = al <= 1
    assert np.array_equal(got[lo], A["roots/out"][lo])
    np.testing.assert_allclose(got[~lo], A["roots/out"][~lo], rtol=1e-9, atol=1e-12)
    # KATs (tests/test_kernels.py:156-159)
    assert pf.solve_sum_equation(1.0, 1.0, 0.0, 1) == pytest.approx(1 / np.sqrt(2))
    assert pf.solve_sum_equation(1.0, 1.0, 3.0, 0) == pytest.approx(2.0)
    assert pf.solve_sum_equation(1.0, 1.0, 0.0, 2) == pytest.approx(0.5 ** (1 / 3))


def test_suggestions_share_overload_equally():
    """tests/test_kernels.py:114-126: x=(8,8), C=10 -> y=(6,6) on the shared edge."""
    inst = shared_edge(n=2, cap=10.0, demand=20.0)
    rng = np.random.default_rng(1)
    arrs = states.random_state(inst.num_commodities, inst.num_paths, inst.num_edges, inst.num_pairs, rng)
    st = pf.SolverState(**arrs, beta=1.0, alpha=0, iteration=0)
    st.x = np.array([8.0, 8.0])
    st.dual_capacity = np.zeros(inst.num_edges)
    st.dual_consensus = np.zeros(inst.num_pairs)
    y = pf.update_rate_suggestions(st, inst)
    shared = [y[p] for p in range(inst.num_pairs) if inst.pair_edge[p] == 2]
    feeder = [y[p] for p in range(inst.num_pairs) if inst.pair_edge[p] != 2]
    assert shared == pytest.approx([6.0, 6.0]) and feeder == pytest.approx([8.0, 8.0])


def test_kernel_error_names_the_commodity():
    inst = chain()
    rng = np.random.default_rng(2)
    arrs = states.random_state(inst.num_commodities, inst.num_paths, inst.num_edges, inst.num_pairs, rng)
    st = pf.SolverState(**arrs, beta=1.0, alpha=0, iteration=0)
    st.y = st.y.copy()
    st.y[2] = np.nan
    with pytest.raises(pf.KernelError, match="A→C"):
        pf.solve_commodity_sums(st, inst, 0)


# ------------------------------------------------------------------ exact-mode solves


def _exact_trajectory(tag, inst, cfg, snaps, warm=None):
    D, A, M = G.digests(), G.arrays(), G.meta()
    s = pf.Solver(inst, cfg).init(warm)
    done = 0
    for it in sorted(snaps):
        if it > M[tag]["iterations"]:
            continue
        s.run(it - done)
        done = it
        st = s.state()
        assert st.iteration == it
        assert st.beta == D[f"{tag}/it{it}/beta"] and st.alpha == D[f"{tag}/it{it}/alpha"], it
        for f, arr in (("x", st.x), ("y", st.y), ("dual_demand", st.dual_demand),
                       ("dual_capacity", st.dual_capacity), ("dual_consensus", st.dual_consensus),
                       ("dual_nonneg", st.dual_nonneg)):
            if f == "x" and st.alpha >= 2:
                np.testing.assert_allclose(arr, A[f"{tag}/it{it}/x"], rtol=1e-9, atol=1e-12)
                continue
            assert G.digest(arr) == D[f"{tag}/it{it}/{f}"], (tag, it, f)
    s.run(M[tag]["iterations"] - done)
    r = s.result()
    assert r.iterations == M[tag]["iterations"] and bool(r.converged) == M[tag]["converged"]
    rates, sums = s.finish()
    if r.alpha >= 2:
        np.testing.assert_allclose(sums, A[f"{tag}/sums"], rtol=1e-9, atol=1e-9)
    else:
        assert G.digest(rates) == D[f"{tag}/rates"]
        assert np.array_equal(sums, A[f"{tag}/sums"])


def test_exact_cfg1_trajectory_to_stagnation_stop():
    inst = golden_instance("cfg1_v0.3")
    _exact_trajectory("cfg1_v0.3", inst, pf.SolverConfig(mode="exact"),
                      {1, 2, 3, 5, 10, 50, 200, 500, 826, 866, 978})


def test_exact_cfg1_highload_5000_iterations_trace_bitwise():
    tag = "cfg1_v1.5"
    inst = golden_instance(tag)
    _exact_trajectory(tag, inst, pf.SolverConfig(mode="exact"), {1, 2, 3, 5, 10, 100, 1000, 3000, 5000})
    res = pf.solve(inst, pf.SolverConfig(mode="exact", trace=True))
    got = np.array([(t.iteration, t.alpha, t.beta, t.s, t.r) for t in res.trace])
    np.testing.assert_array_equal(got, G.arrays()[f"{tag}/trace"])


def test_exact_link_failure_warm_start():
    tag = "cfg1_v0.3"
    A = G.arrays()
    inst = golden_instance(tag)
    base = pf.solve(inst, pf.SolverConfig(mode="exact"))
    np.testing.assert_allclose(base.sums, A[f"{tag}/sums"], rtol=1e-9, atol=1e-9)
    cap = inst.capacity.copy()
    cap[A[f"{tag}/cut_edges"]] = 0.0
    cut = pf.with_conditions(inst, capacity=cap)
    # warm start from the reference's own projected rates (its alpha=2 tail uses numpy pow)
    _exact_trajectory(f"{tag}/warm_cut", cut, pf.SolverConfig(mode="exact", alpha_target=1, max_iterations=400),
                      {1, 10, 100, 400}, warm=A[f"{tag}/warm_rates"])


@pytest.mark.parametrize("name", G.SMALL)
@pytest.mark.parametrize("tgt", [0, 1, 2, None])
def test_exact_small_solves(name, tgt):
    inst = SMALL_BUILDERS[name]()
    A, M = G.arrays(), G.meta()
    key = f"small/{name}/solve_a{tgt}"
    res = pf.solve(inst, pf.SolverConfig(alpha_target=tgt, mode="exact"))
    assert (res.iterations, res.alpha, res.converged) == (M[key]["iterations"], M[key]["alpha"],
                                                         M[key]["converged"])
    if res.alpha <= 1:
        assert np.array_equal(res.rates, A[f"{key}/rates"])
    else:
        np.testing.assert_allclose(res.rates, A[f"{key}/rates"], rtol=1e-9, atol=1e-12)


def test_exact_trace_columns():
    A = G.arrays()
    for name in G.SMALL:
        res = pf.solve(SMALL_BUILDERS[name](), pf.SolverConfig(max_iterations=7, trace=True, mode="exact"))
        got = np.array([(t.iteration, t.alpha, t.beta, t.s, t.r, t.objective, t.pct_violated,
                         t.mean_relative_violation) for t in res.trace])
        want = A[f"small/{name}/trace7"]
        np.testing.assert_array_equal(got[:, :5], want[:, :5])
        np.testing.assert_allclose(got[:, 5:], want[:, 5:], rtol=1e-12, atol=1e-12)
        assert np.array_equal(res.rates, A[f"small/{name}/trace7_rates"])


# ------------------------------------------------------------------ projection


@pytest.mark.parametrize("kk", [0, 1])
@pytest.mark.parametrize("alpha", [0, 1, 3])
def test_projection_bitwise(kk, alpha):
    tag = "cfg1_v0.3"
    A, D = G.arrays(), G.digests()
    inst = golden_instance(tag)
    x = A[f"{tag}/proj{kk}/raw_x"]
    out = pf.project(inst, x, alpha)
    if alpha <= 1:
        assert G.digest(out) == D[f"{tag}/proj{kk}/a{alpha}"]
    np.testing.assert_allclose(pf.commodity_sums(inst, out), A[f"{tag}/proj{kk}/a{alpha}_sums"],
                               rtol=1e-12, atol=1e-9)
    rep = pf.validate_allocation(inst, out)
    assert rep.feasible
    assert np.array_equal(pf.project(inst, out, alpha), out)  # idempotent


def test_projection_adversarial_vs_oracle():
    """Criterion 3 style (tests/test_acceptance.py:177-208): random +/- boundary inputs."""
    from oracle import oracle as O
    inst = golden_instance("cfg1_v0.3")
    I = oracle_instance("cfg1_v0.3")
    rng = np.random.default_rng(11)
    for trial in range(6):
        x = rng.uniform(-1.0, 30.0, inst.num_paths)
        x[rng.random(inst.num_paths) < 0.1] = 0.0
        for alpha in (0, 1):
            got = pf.project(inst, x, alpha)
            assert np.array_equal(got, O.project(I, x, alpha))
            assert pf.validate_allocation(inst, got).feasible


# ------------------------------------------------------------------ fast mode


def test_fast_first_iterations_match_exact():
    """Edge sums are reassociated in fast mode; iterations 1-2 agree to 1e-12."""
    inst = golden_instance("cfg1_v0.3")
    ex = pf.Solver(inst, pf.SolverConfig(mode="exact")).init()
    fa = pf.Solver(inst, pf.SolverConfig(mode="fast")).init()
    s0 = fa.state()
    e0 = ex.state()
    assert np.array_equal(s0.x, e0.x) and np.array_equal(s0.y, e0.y)
    for it in (1, 2):
        ex.run(1)
        fa.run(1)
        a, b = ex.state(), fa.state()
        assert a.iteration == b.iteration == it
        assert a.beta == b.beta and a.alpha == b.alpha
        for f in ("x", "y", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg"):
            np.testing.assert_allclose(getattr(b, f), getattr(a, f), rtol=1e-11, atol=1e-11, err_msg=f"{it} {f}")


def test_fast_controller_decisions_match_reference():
    """Same alpha / beta decision sequence as the reference for the first 300 iterations."""
    tag = "cfg1_v0.3"
    inst = golden_instance(tag)
    res = pf.solve(inst, pf.SolverConfig(mode="fast", trace=True, max_iterations=300))
    want = G.arrays()[f"{tag}/trace"][:300]
    got = np.array([(t.iteration, t.alpha, t.beta) for t in res.trace])
    np.testing.assert_array_equal(got, want[:, :3])
    # residuals agree tightly while the trajectories coincide (edge sums reassociated)
    np.testing.assert_allclose([t.s for t in res.trace[:3]], want[:3, 3], rtol=1e-9)


def test_fast_trace_objective_within_1e4_of_exact():
    """SURVEY 8(d) fast-mode gate: objective within 1e-4 of the reference's
    (exact mode, bitwise the reference) on every trace row, over 300
    iterations with the same alpha / beta decisions."""
    inst = golden_instance("cfg1_v0.3")
    fa = pf.solve(inst, pf.SolverConfig(mode="fast", trace=True, max_iterations=300))
    ex = pf.solve(inst, pf.SolverConfig(mode="exact", trace=True, max_iterations=300))
    assert len(fa.trace) == len(ex.trace) == 300
    for a, b in zip(fa.trace, ex.trace):
        assert (a.iteration, a.alpha, a.beta) == (b.iteration, b.alpha, b.beta)
        assert abs(a.objective - b.objective) <= 1e-4 * max(1.0, abs(b.objective)), (a.iteration, a.objective,
                                                                                       b.objective)


def test_fast_converged_sums_within_1e4():
    """cfg1, V = 0.3 x capacity: stagnation stop; sorted max-min vector within 1e-4."""
    tag = "cfg1_v0.3"
    A, M = G.arrays(), G.meta()
    inst = golden_instance(tag)
    res = pf.solve(inst, pf.SolverConfig(mode="fast"))
    assert res.converged
    want = np.sort(A[f"{tag}/sums"])
    got = np.sort(res.sums)
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-4 * float(want.max()))
    assert abs(res.iterations - M[tag]["iterations"]) <= 0.05 * M[tag]["iterations"]
    assert pf.validate_allocation(inst, res.rates).feasible


def test_fast_deterministic_and_sum_consistent():
    inst = golden_instance("cfg1_v1.5")
    a = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
    b = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
    a.run(200)
    b.run(50)
    b.run(150)
    xa, xb = a.x(), b.x()
    assert np.array_equal(xa, xb)  # chunked launches == one launch, bitwise
    # sum consistency: sum_p x_p equals the solved commodity sum (kernels.py:285-296)
    st = a.state()
    assert np.all(np.isfinite(st.x))


def test_cfg2_full_size_fast_vs_exact():
    """Config 2 at full size (18.3M pairs, max 53k pairs per edge): iterations
    1-3 of the fused kernel agree with the exact-order path (reassociated edge
    sums only), the fused loop is bit-reproducible and independent of how it is
    split into launches, and the fast projection is feasible."""
    topo, tab, ps = pytest.importorskip("b200_helpers").generated(500, 8, 1.5)
    inst = pf.build_instance(topo, tab, ps, device=0)
    assert inst.num_pairs == 18282422
    ex = pf.Solver(inst, pf.SolverConfig(mode="exact", gamma=1e-12)).init()
    fa = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
    for it in (1, 2, 3):
        ex.run(1)
        fa.run(1)
        a, b = ex.state(), fa.state()
        assert a.iteration == b.iteration == it and a.beta == b.beta and a.alpha == b.alpha
        xs = float(np.max(np.abs(a.x)))  # every array here is in rate units
        for f in ("x", "y", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg"):
            want, got = getattr(a, f), getattr(b, f)
            scale = max(float(np.max(np.abs(want))), xs)
            assert float(np.max(np.abs(got - want))) <= 1e-9 * scale, (it, f)
    del ex
    one = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
    one.run(100)
    split = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
    split.run(37)
    split.run(63)
    assert np.array_equal(one.x(), split.x())
    rates, _ = one.finish()
    assert pf.validate_allocation(inst, rates).feasible


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_small_solves_both_modes(mode):
    """tests/test_controller.py:126-141 expectations."""
    res = pf.solve(single_bottleneck(cap=10.0, demand=20.0), pf.SolverConfig(alpha_target=0, mode=mode))
    assert res.converged and res.sums[0] == pytest.approx(10.0, abs=0.1)
    res = pf.solve(shared_edge(2, cap=10.0, demand=20.0), pf.SolverConfig(mode=mode))
    assert res.converged and res.sums == pytest.approx([5.0, 5.0], abs=0.1)
    res = pf.solve(chain(), pf.SolverConfig(mode=mode))
    assert res.converged and res.sums == pytest.approx([7.5, 2.5, 2.5], abs=0.15)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_edge_cases(mode):
    from b200_helpers import make_instance
    inst = make_instance([("A", "B", 10, 1)], [("A", "B", 0.0, [(0,)])])
    res = pf.solve(inst, pf.SolverConfig(mode=mode))
    assert res.converged and res.rates.size == 0 and res.iterations == 0
    inst = chain()
    res = pf.solve(inst, pf.SolverConfig(max_iterations=3, mode=mode))
    assert not res.converged and res.iterations == 3
    assert pf.validate_allocation(inst, res.rates).feasible
    for bad in (np.nan, np.inf, -np.inf):
        with pytest.raises(pf.InputError, match="warm start contains non-finite rates"):
            pf.solve(inst, pf.SolverConfig(mode=mode), warm_start=np.array([1.0, bad, 2.0]))
    with pytest.raises(pf.InputError):
        pf.solve(inst, pf.SolverConfig(mode=mode), warm_start=np.array([1.0, 2.0]))
    # the check runs on the device copy: a failed init leaves nothing runnable
    s = pf.Solver(inst, pf.SolverConfig(mode=mode)).init()
    s.run(2)
    with pytest.raises(pf.InputError, match="non-finite"):
        s.init(np.array([1.0, 2.0, np.nan]))
    with pytest.raises(Exception, match="not initialized"):
        s.run(1)
    s.init(np.array([1.0, 2.0, 3.0]))
    assert s.run(2) == 2


@pytest.mark.parametrize("n,k", [(60, 8), (50, 1), (45, 3)])
def test_fast_iterations_match_exact_generated(n, k):
    """Larger generated instances (many tiles, full 32-path groups at k=8, 32
    single-path commodities per group at k=1): iterations 1-3 of the fused
    kernel agree with the exact-order path to 1e-11."""
    from b200_helpers import generated
    topo, tab, ps = generated(n, k, 1.5)
    inst = pf.build_instance(topo, tab, ps, device=0)
    ex = pf.Solver(inst, pf.SolverConfig(mode="exact")).init()
    fa = pf.Solver(inst, pf.SolverConfig(mode="fast")).init()
    for it in (1, 2, 3):
        ex.run(1)
        fa.run(1)
        a, b = ex.state(), fa.state()
        assert a.iteration == b.iteration == it
        for f in ("x", "y", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg"):
            np.testing.assert_allclose(getattr(b, f), getattr(a, f), rtol=1e-10, atol=1e-10, err_msg=f"{it} {f}")


@pytest.mark.parametrize("run_slots", ["1", "0"])
def test_fast_large_edge_mode_matches_exact(monkeypatch, run_slots):
    """The large-E layouts (PF_FAST_LARGE_E forces them on a small instance):
    run slots (per-(tile, run) edge totals in edge-major global slots, a per-tile
    run adjustment table; the default for large E) and the older per-CTA
    accumulators with the adjustment table read through L1 (PF_FAST_RS=0):
    iterations 1-3 agree with the exact-order path to 1e-10, and the converged
    solve matches the default layout."""
    from b200_helpers import generated
    monkeypatch.setenv("PF_FAST_LARGE_E", "1")
    monkeypatch.setenv("PF_FAST_RS", run_slots)
    topo, tab, ps = generated(60, 8, 1.5)
    inst = pf.build_instance(topo, tab, ps, device=0)  # fresh index set: the layout is built with the override
    ex = pf.Solver(inst, pf.SolverConfig(mode="exact")).init()
    fa = pf.Solver(inst, pf.SolverConfig(mode="fast")).init()
    for it in (1, 2, 3):
        ex.run(1)
        fa.run(1)
        a, b = ex.state(), fa.state()
        for f in ("x", "y", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg"):
            np.testing.assert_allclose(getattr(b, f), getattr(a, f), rtol=1e-10, atol=1e-10, err_msg=f"{it} {f}")
    big = pf.solve(inst, pf.SolverConfig(mode="fast", max_iterations=400))
    monkeypatch.delenv("PF_FAST_LARGE_E")
    monkeypatch.delenv("PF_FAST_RS")
    inst2 = pf.build_instance(topo, tab, ps, device=0)
    small = pf.solve(inst2, pf.SolverConfig(mode="fast", max_iterations=400))
    assert pf.validate_allocation(inst, big.rates).feasible
    np.testing.assert_allclose(np.sort(big.sums), np.sort(small.sums), rtol=1e-3, atol=1e-3 * float(small.sums.max()))


def test_fast_solve_projection_feasible_and_close_to_exact():
    """A fast-mode solve projects with the tolerance-matched parallel trim; on a
    raw, heavily infeasible iterate it must return an exactly feasible allocation
    whose commodity sums agree with the bitwise (reference-order) projection."""
    from b200_helpers import generated
    topo, tab, ps = generated(60, 8, 1.5)
    inst = pf.build_instance(topo, tab, ps, device=0)
    s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
    s.run(12)
    x = s.x()
    alpha = int(s.state().alpha)
    before = pf.validate_allocation(inst, np.maximum(x, 0.0))
    assert not before.feasible  # the test is about real trimming
    fast_rates, fast_sums = s.finish()
    exact_rates = pf.project(inst, x, alpha)
    assert pf.validate_allocation(inst, fast_rates).feasible
    np.testing.assert_allclose(fast_sums, pf.commodity_sums(inst, exact_rates), rtol=1e-6,
                               atol=1e-9 * float(np.max(np.abs(x))))


@pytest.mark.parametrize("ncl", ["1", "2", "8", "0"])
def test_fast_projection_cluster_variants(ncl):
    """The cluster-resident fast trim (1, 2 and 8 CTAs per cluster; slices of
    multi-element runs per thread) and the single-CTA kernel ("0") on a raw
    iterate with edges of thousands of paths: exactly feasible, commodity sums
    matching the bitwise projection, bit-reproducible run to run."""
    import json
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, PF_PROJ_CLUSTER=ncl)
    r = subprocess.run([sys.executable, os.path.join(here, "_proj_variant.py"), "150", "4", "12"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["infeasible_before"] and out["max_edge_paths"] > 2048
    assert out["feasible"] and out["deterministic"]
    assert out["sums_rel"] <= 1e-6, out


def test_fast_projection_pipelined_trim_bitwise():
    """The pipelined cluster trim (path slices loaded two edges ahead, the next
    edge's rates gathered speculatively and used only when the current edge
    changed nothing) gives bitwise the rates of the plain cluster trim."""
    import json
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    outs = []
    for pipe in ("0", "1"):
        env = dict(os.environ, PF_PROJ_CLUSTER="8", PF_PROJ_PIPE=pipe)
        r = subprocess.run([sys.executable, os.path.join(here, "_proj_variant.py"), "150", "4", "12"], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0]["feasible"] and outs[1]["feasible"] and outs[1]["deterministic"]
    assert outs[0]["digests"][0] == outs[1]["digests"][0]


def test_speculated_rescale_bitwise():
    """The M pass applies the predicted dual rescale factor (predict_f) instead
    of 1, and a rollback pass runs only on a wrong prediction: the iterates
    (several tiles per CTA, beta's ramp and its plateau) are bitwise those of
    the always-1 speculation with its rollback on every beta change."""
    import json
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    outs = []
    for spec in ("0", "1"):
        env = dict(os.environ, PF_FAST_SPEC=spec)
        r = subprocess.run([sys.executable, os.path.join(here, "_spec_variant.py"), "150", "4", "400"], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]
    assert outs[0]["beta"] > 1.0  # beta moved: the rollback / speculation paths ran


def test_fast_trace_batched_rows_equal_per_row_path():
    """Traced fast runs without an optimality column compute their rows on the
    device in batches (no host round trip per iteration); with reference sums
    every row is computed after its own launch.  Every shared column is
    bitwise equal between the two, across the alpha / beta changes."""
    tag = "cfg1_v0.3"
    inst = golden_instance(tag)
    batched = pf.solve(inst, pf.SolverConfig(mode="fast", trace=True, max_iterations=900))
    ref = G.arrays()[f"{tag}/sums"]
    per_row = pf.solve(inst, pf.SolverConfig(mode="fast", trace=True, max_iterations=900, reference_sums=ref))
    assert len(batched.trace) == len(per_row.trace) == batched.iterations == per_row.iterations
    cols = ("iteration", "alpha", "beta", "s", "r", "objective", "pct_violated", "mean_relative_violation")
    a = np.array([[getattr(t, c) for c in cols] for t in batched.trace])
    b = np.array([[getattr(t, c) for c in cols] for t in per_row.trace])
    assert np.array_equal(a, b)
    assert len({t.alpha for t in batched.trace}) > 1  # the run crosses alpha changes
    assert all(t.optimality is None for t in batched.trace)
    assert np.array_equal(batched.rates, per_row.rates)


def test_fast_mode_outside_fused_limits_runs_exact():
    """More than 32 paths per commodity (one warp lane per path in the fused
    kernel): a fast-mode solve runs the exact-order kernels instead -- the
    reference's arithmetic, bitwise -- and the fused-only entry points say why."""
    topo = pf.random_topology(30, seed=30)
    tab = pf.gravity_table(topo, 0.3 * float(topo.capacity.sum()))
    ps = pf.k_shortest_paths(topo, tab, 40)
    assert int(np.max(np.diff(np.asarray(ps.com_path_ptr)))) > 32
    inst = pf.build_instance_flat(topo, tab, ps, device=0)
    with pytest.warns(RuntimeWarning, match="layout limits"):
        fast = pf.solve(inst, pf.SolverConfig(mode="fast", max_iterations=200))
    assert fast.mode == "exact"  # the fallback is reported, not silent
    exact = pf.solve(inst, pf.SolverConfig(mode="exact", max_iterations=200))
    assert np.array_equal(fast.rates, exact.rates) and fast.iterations == exact.iterations
    s = pf.Solver(inst, pf.SolverConfig(mode="fast")).init()
    with pytest.raises(pf.InputError, match="more than 32 paths"):
        s.time_loop(5)


def test_dao_carry_bitwise_vs_reference():
    """oracles.py:262-297 on the GPU: dao_carry_rates bitwise equal to the
    reference on every golden drift case (zero drift, 5% link cuts, mixed
    capacity / demand drift), dao_evaluate equal to the reference's value."""
    for tag, cases in G.dao().items():
        base = golden_instance(tag)
        for case, a in cases.items():
            drifted = pf.with_conditions(base, capacity=a["capacity"], demand=a["demand"])
            out = pf.dao_carry_rates(a["rates_in"], drifted)
            assert np.array_equal(out, a["rates_out"]), (tag, case)
            if "dao_evaluate" in a:
                alloc = types.SimpleNamespace(rates=a["rates_in"])
                ref = types.SimpleNamespace(sums=a["ref_sums"])
                got = pf.dao_evaluate(alloc, drifted, ref, float(a["theta"][0]))
                assert got == float(a["dao_evaluate"][0]), (tag, got)


def test_dao_carry_generated_matches_oracle():
    """A 447k-pair generated instance (max 5k pairs per edge) with 5% of the
    links cut and drifted demands: GPU carry bitwise equal to the oracle's, and
    the carried allocation feasible."""
    from b200_helpers import generated
    from oracle import oracle as O
    topo, tab, ps = generated(90, 8, 1.5)
    inst = pf.build_instance(topo, tab, ps, device=0)
    rates = pf.solve(inst, pf.SolverConfig(max_iterations=100)).rates
    rng = np.random.default_rng(7)
    cap = np.asarray(inst.capacity, float).copy()
    cap[rng.choice(inst.num_edges, round(0.05 * inst.num_edges), replace=False)] = 0.0
    dem = np.asarray(inst.demand, float) * rng.uniform(0.7, 1.1, inst.num_commodities)
    drifted = pf.with_conditions(inst, capacity=cap, demand=dem)
    out = pf.dao_carry_rates(rates, drifted)
    flat = O.build_instance(topo.capacity, tab.demand, ps.com_path_ptr, ps.path_edge_ptr, ps.path_edges)
    want = O.dao_carry_rates(flat.with_conditions(capacity=cap, demand=dem), rates)
    assert np.array_equal(out, want)
    assert pf.validate_allocation(drifted, out).feasible
    assert np.array_equal(pf.dao_carry_rates(rates, inst), rates)  # zero drift: bit-identical


@pytest.mark.parametrize("scale", [1e300, 1e308])
def test_overflowing_warm_start_raises_like_exact(scale):
    """Non-finite coefficients / roots / iterates raise KernelError (naming the
    commodity) or SolverError exactly as the exact-order path (the reference's
    order of checks: kernels.py:270-281 before controller.py:238-239)."""
    inst = chain()
    warm = np.full(inst.num_paths, scale)
    errs = {}
    for mode in ("exact", "fast"):
        try:
            pf.solve(inst, pf.SolverConfig(mode=mode, max_iterations=50), warm_start=warm)
            errs[mode] = None
        except (pf.KernelError, pf.SolverError) as exc:
            errs[mode] = (type(exc), str(exc) if isinstance(exc, pf.KernelError) else None)
    assert errs["exact"] is not None
    assert errs["fast"] == errs["exact"]


def test_fast_l2_accumulators_match_exact(monkeypatch):
    """Large-E layout with the edge run totals accumulated in the CTAs' L2 partial
    rows (PF_FAST_LARGE_E + PF_FAST_ACC_L2): iterations 1-3 agree with the exact
    path to 1e-10 and runs are bit-reproducible."""
    from b200_helpers import generated
    monkeypatch.setenv("PF_FAST_LARGE_E", "1")
    monkeypatch.setenv("PF_FAST_ACC_L2", "1")
    topo, tab, ps = generated(60, 8, 1.5)
    inst = pf.build_instance(topo, tab, ps, device=0)
    ex = pf.Solver(inst, pf.SolverConfig(mode="exact")).init()
    fa = pf.Solver(inst, pf.SolverConfig(mode="fast")).init()
    for it in (1, 2, 3):
        ex.run(1)
        fa.run(1)
        a, b = ex.state(), fa.state()
        for f in ("x", "y", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg"):
            np.testing.assert_allclose(getattr(b, f), getattr(a, f), rtol=1e-10, atol=1e-10, err_msg=f"{it} {f}")
    r1 = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
    r2 = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12)).init()
    r1.run(150)
    r2.run(60)
    r2.run(90)
    assert np.array_equal(r1.x(), r2.x())
