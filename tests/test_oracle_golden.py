"""Pin the C oracle to the reference (CPU only).

Every expectation comes from tests/golden/, produced by running the unmodified
reference (make_golden.py).  Bitwise for alpha in {0,1}; alpha >= 2 kernel
outputs that pass through numpy's SIMD `power` are pinned at 1e-12 relative.
"""

import numpy as np
import pytest

import golden_io as G
import states
from oracle import oracle as O


def _inst(prefix):
    f = G.flat_inputs(prefix)
    return O.build_instance(f["capacity"], f["demand0"], f["com_path_ptr0"], f["path_edge_ptr0"],
                            f["path_edges0"])


@pytest.mark.parametrize("name", G.SMALL)
def test_incidence_small_exact(name):
    I = _inst(f"small/{name}")
    A = G.arrays()
    for f in G.INCIDENCE:
        assert np.array_equal(getattr(I, f), A[f"small/{name}/inc/{f}"]), f


@pytest.mark.parametrize("tag", ["cfg1_v0.3", "cfg1_v1.5"])
def test_incidence_cfg1_exact(tag):
    I = _inst(tag)
    D = G.digests()
    for f in G.INCIDENCE:
        dt = np.float64 if f == "demand" else np.int64
        assert G.digest(np.asarray(getattr(I, f), dt)) == D[f"{tag}/inc/{f}"], f


def _kernel_check(tag, I):
    A, D = G.arrays(), G.digests()
    cases = states.kernel_case_states(I.num_commodities, I.num_paths, I.num_edges, I.num_pairs,
                                      G.kernel_seed(tag))
    for i, (arrs, beta, alpha) in enumerate(cases):
        key = f"{tag}/k{i}"
        st = O.OState(*(arrs[f].copy() for f in G.STATE), beta, alpha, 0)
        dd, dc, dcon, dn = O.update_duals(I, st)
        sd, sc = O.update_slacks(I, st)
        got = dict(dd=dd, dc=dc, dcon=dcon, dn=dn, sd=sd, sc=sc)
        st.dual_demand, st.dual_capacity, st.dual_consensus, st.dual_nonneg = dd, dc, dcon, dn
        st.y = O.update_rate_suggestions(I, st)
        got["y"] = st.y
        sums = O.solve_commodity_sums(I, st, alpha)
        got["sums"] = sums
        got["x"] = O.update_rates(I, st, sums, alpha)
        for nm, a in got.items():
            if alpha >= 2 and nm == "x":
                # numpy SIMD power vs glibc pow in the gain term (kernels.py:289)
                np.testing.assert_allclose(a, A[f"{key}/out/x"], rtol=1e-12, atol=1e-12)
            else:
                assert G.digest(a) == D[f"{key}/out/{nm}"], (key, nm)


@pytest.mark.parametrize("name", G.SMALL)
def test_kernels_small(name):
    _kernel_check(f"small/{name}", _inst(f"small/{name}"))


def test_kernels_cfg1():
    _kernel_check("cfg1_v0.3", _inst("cfg1_v0.3"))


def test_roots_match_reference_bitwise():
    A = G.arrays()
    got = np.array([O.solve_sum_equation(w, b, q, int(a)) for w, b, q, a in
                    zip(A["roots/w"], A["roots/beta"], A["roots/q"], A["roots/alpha"])])
    assert np.array_equal(got, A["roots/out"])


def test_root_kats():
    # tests/test_kernels.py:156-159
    assert O.solve_sum_equation(1.0, 1.0, 0.0, 1) == pytest.approx(1 / np.sqrt(2))
    assert O.solve_sum_equation(1.0, 1.0, 3.0, 0) == pytest.approx(2.0)
    assert O.solve_sum_equation(1.0, 1.0, 0.0, 2) == pytest.approx(0.5 ** (1 / 3))


@pytest.mark.parametrize("name", G.SMALL)
@pytest.mark.parametrize("tgt", [0, 1, 2, None])
def test_small_solves_bitwise(name, tgt):
    I = _inst(f"small/{name}")
    A, M = G.arrays(), G.meta()
    key = f"small/{name}/solve_a{tgt}"
    res = O.solve(I, alpha_target=tgt)
    assert res.iterations == M[key]["iterations"]
    assert res.alpha == M[key]["alpha"]
    assert res.converged == M[key]["converged"]
    if res.alpha <= 1:
        assert np.array_equal(res.rates, A[f"{key}/rates"])
        assert np.array_equal(res.sums, A[f"{key}/sums"])
    else:  # numpy SIMD power in update_rates (kernels.py:289) vs glibc pow
        np.testing.assert_allclose(res.rates, A[f"{key}/rates"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(res.sums, A[f"{key}/sums"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("name", G.SMALL)
def test_small_trace(name):
    I = _inst(f"small/{name}")
    A = G.arrays()
    res = O.solve(I, max_iterations=7, trace=True)
    want = A[f"small/{name}/trace7"]
    got = np.array(res.trace, dtype=np.float64)
    assert got.shape == want.shape
    np.testing.assert_array_equal(got[:, :5], want[:, :5])  # iteration, alpha, beta, s, r
    np.testing.assert_allclose(got[:, 5:], want[:, 5:], rtol=1e-12, atol=1e-12)
    assert np.array_equal(res.rates, A[f"small/{name}/trace7_rates"])


def test_warm_start_chain():
    I = _inst("small/chain")
    A, M = G.arrays(), G.meta()
    res = O.solve(I, alpha_target=1, warm_start=A["small/chain/warm/start"])
    assert res.iterations == M["small/chain/warm"]["iterations"]
    assert np.array_equal(res.rates, A["small/chain/warm/rates"])


def _trajectory(tag, I, loop, snaps_meta_iters):
    D, A, M = G.digests(), G.arrays(), G.meta()
    want_trace = A[f"{tag}/trace"]
    done = 0
    for it in sorted(snaps_meta_iters):
        if it > M[tag]["iterations"]:
            continue
        loop.step(it - done)
        done = it
        st = loop.state()
        assert st.iteration == it
        assert st.beta == D[f"{tag}/it{it}/beta"] and st.alpha == D[f"{tag}/it{it}/alpha"]
        for f in G.STATE:
            if f == "x" and st.alpha >= 2:  # numpy SIMD power (kernels.py:289)
                np.testing.assert_allclose(st.x, A[f"{tag}/it{it}/x"], rtol=1e-9, atol=1e-12)
                continue
            assert G.digest(getattr(st, f)) == D[f"{tag}/it{it}/{f}"], (tag, it, f)
        assert G.digest(loop.last_sums()) == D[f"{tag}/it{it}/sums"], (tag, it)
    loop.step(M[tag]["iterations"] - done)
    st = loop.state()
    assert st.iteration == M[tag]["iterations"]
    assert loop.stopped == M[tag]["converged"]
    got_trace = np.array([r[:5] for r in loop.trace_rows()])
    np.testing.assert_array_equal(got_trace, want_trace)
    rates = O.project(I, st.x, st.alpha)
    if st.alpha >= 2:
        np.testing.assert_allclose(st.x, A[f"{tag}/raw_x"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(O.commodity_sums(I, rates), A[f"{tag}/sums"], rtol=1e-9, atol=1e-9)
    else:
        assert G.digest(st.x) == D[f"{tag}/raw_x"]
        assert G.digest(rates) == D[f"{tag}/rates"]
        assert np.array_equal(O.commodity_sums(I, rates), A[f"{tag}/sums"])


def test_cfg1_trajectory_to_stop_bitwise():
    """978 iterations, alpha 0 -> 2 with the stagnation stop."""
    tag = "cfg1_v0.3"
    I = _inst(tag)
    loop = O.Loop(I, O.make_config(trace=True), trace_cap=5000)
    _trajectory(tag, I, loop, {1, 2, 3, 5, 10, 50, 200, 500, 826, 866, 978})


def test_cfg1_highload_trajectory_bitwise():
    """V = 1.5 x total capacity: 5,000-iteration cap, never converges."""
    tag = "cfg1_v1.5"
    I = _inst(tag)
    loop = O.Loop(I, O.make_config(trace=True), trace_cap=5000)
    _trajectory(tag, I, loop, {1, 2, 3, 5, 10, 100, 1000, 3000, 5000})


def test_cfg1_link_failure_warm_start():
    tag = "cfg1_v0.3"
    I = _inst(tag)
    A, D, M = G.arrays(), G.digests(), G.meta()
    base = O.solve(I)
    np.testing.assert_allclose(base.sums, A[f"{tag}/sums"], rtol=1e-9, atol=1e-9)
    cap = I.capacity.copy()
    cap[A[f"{tag}/cut_edges"]] = 0.0
    Ic = I.with_conditions(capacity=cap)
    wtag = f"{tag}/warm_cut"
    loop = O.Loop(Ic, O.make_config(alpha_target=1, max_iterations=400, trace=True),
                  warm=base.rates, trace_cap=400)
    _trajectory(wtag, Ic, loop, {1, 10, 100, 400})


@pytest.mark.parametrize("kk", [0, 1])
@pytest.mark.parametrize("alpha", [0, 1, 3])
def test_projection_of_raw_iterates(kk, alpha):
    tag = "cfg1_v0.3"
    I = _inst(tag)
    A, D = G.arrays(), G.digests()
    x = A[f"{tag}/proj{kk}/raw_x"]
    out = O.project(I, x, alpha)
    sums = O.commodity_sums(I, out)
    if alpha <= 1:
        assert G.digest(out) == D[f"{tag}/proj{kk}/a{alpha}"]
    np.testing.assert_allclose(sums, A[f"{tag}/proj{kk}/a{alpha}_sums"], rtol=1e-12, atol=1e-9)
    # feasibility + idempotence (tests/test_projection.py:81-102)
    pct, _, nv = O.violation_stats(I, out)
    assert nv == 0
    assert np.array_equal(O.project(I, out, alpha), out)


def test_dao_carry_oracle_matches_reference():
    """oracles.py:262-287 restated in oracle/ (exact-order sums): bitwise equal
    to the reference's dao_carry_rates on every golden drift case."""
    from b200_helpers import oracle_instance
    for tag, cases in G.dao().items():
        base = oracle_instance(tag)
        for case, a in cases.items():
            inst = base.with_conditions(capacity=a["capacity"], demand=a["demand"])
            out = O.dao_carry_rates(inst, a["rates_in"])
            assert np.array_equal(out, a["rates_out"]), (tag, case)
            if case == "zero_drift":
                assert np.array_equal(out, a["rates_in"])
