"""SPEC acceptance criteria 1-9 (reference tests/test_acceptance.py:77-401) with
the GPU solvers swapped in for pathfair.solve: same instance families, seeds and
thresholds.  Criteria 2 and 7 compare against the reference grid oracle's
values recorded by tests/golden/make_golden_acceptance.py.  The single-path max-min reference is
a progressive-filling oracle restated here (pathfair/oracles.py:56-93:
raise every unfrozen commodity equally, freeze it at its demand or when its
path meets a saturated edge) -- test infrastructure, not product code."""

import numpy as np
import pytest

import paper_2605_01748_b200 as pf
from b200_helpers import shared_edge

pytestmark = pytest.mark.gpu

_SAT = 1e-12


def maxmin_singlepath(inst):
    """Progressive filling on a one-path-per-commodity instance (oracles.py:56-93)."""
    cpp = np.asarray(inst.com_path_ptr)
    assert np.all(np.diff(cpp) == 1), "one path per commodity"
    pptr, pedge = np.asarray(inst.pair_ptr), np.asarray(inst.pair_edge)
    cap, dem = np.asarray(inst.capacity, float), np.asarray(inst.demand, float)
    n, E = len(dem), len(cap)
    edges = [pedge[pptr[c]:pptr[c + 1]] for c in range(n)]
    x = np.zeros(n)
    frozen = np.zeros(n, bool)
    for _ in range(2 * (n + E) + 4):
        loads = np.zeros(E)
        for c in range(n):
            loads[edges[c]] += x[c]
        headroom = cap - loads
        saturated = headroom <= _SAT * np.maximum(cap, 1.0)
        frozen |= x >= dem - _SAT * np.maximum(dem, 1.0)
        for c in np.flatnonzero(~frozen):
            if saturated[edges[c]].any():
                frozen[c] = True
        live = np.flatnonzero(~frozen)
        if live.size == 0:
            break
        on_edge = np.zeros(E)
        for c in live:
            on_edge[edges[c]] += 1.0
        step = float(np.min(dem[live] - x[live]))
        used = on_edge > 0
        if used.any():
            step = min(step, float(np.min(headroom[used] / on_edge[used])))
        if step <= 0:
            continue
        x[live] += step
    return x


def _singlepath(topo_seed, n, volume_factor=1.5, **topo_kw):
    topo = pf.random_topology(n, seed=topo_seed, **topo_kw)
    tab = pf.gravity_table(topo, volume_factor * float(topo.capacity.sum()))
    return pf.build_instance(topo, tab, pf.k_shortest_paths(topo, tab, k=1), device=0)


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_criterion_01_singlepath_optimality(mode):
    opts, runtimes = [], []
    for seed in range(50):
        rng = np.random.default_rng(3000 + seed)
        inst = _singlepath(3000 + seed, int(rng.integers(5, 21)))
        res = pf.solve(inst, pf.SolverConfig(mode=mode))
        ref = maxmin_singlepath(inst)
        opts.append(pf.optimality_from_sums(res.sums, ref, pf.default_theta(inst)))
        runtimes.append(res.runtime_s)
    assert min(opts) >= 0.97, f"optimality min {min(opts):.4f} (need >= 0.97 each)"
    assert max(runtimes) <= 5.0


def test_criterion_05_residual_balancing():
    ratios = []
    for seed in range(20):
        rng = np.random.default_rng(1000 + seed)
        inst = _singlepath(2000 + seed, int(rng.integers(6, 14)), capacity_range=(1000.0, 4000.0))
        adaptive = pf.solve(inst, pf.SolverConfig(alpha_target=0, adapt=True, max_iterations=30000))
        fixed = pf.solve(inst, pf.SolverConfig(alpha_target=0, adapt=False, max_iterations=30000))
        ratios.append(adaptive.iterations / fixed.iterations)
    assert np.median(ratios) <= 1.0
    assert float(np.mean(np.asarray(ratios) <= 0.75)) >= 0.5


def test_criterion_06_warm_start():
    cold_its, warm_its = [], []
    for seed in range(20):
        rng = np.random.default_rng(500 + seed)
        inst = _singlepath(700 + seed, int(rng.integers(6, 14)))
        base = pf.solve(inst, pf.SolverConfig())
        factor = 1.0 + rng.uniform(-0.05, 0.05, inst.num_commodities)
        drifted = pf.with_conditions(inst, demand=np.asarray(inst.demand) * factor)
        cfg = pf.SolverConfig(alpha_target=base.alpha)
        cold_its.append(pf.solve(drifted, cfg).iterations)
        warm_its.append(pf.solve(drifted, cfg, warm_start=base.rates).iterations)
    assert np.median(warm_its) <= 0.5 * np.median(cold_its), (np.median(warm_its), np.median(cold_its))


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_criterion_08_stagnation_stop(mode):
    inst = shared_edge(2, cap=10.0, demand=20.0)
    res = pf.solve(inst, pf.SolverConfig(mode=mode))  # no target: the stop must come from stagnation
    ref = maxmin_singlepath(inst)
    rel = float(np.max(np.abs(res.sums - ref) / ref))
    assert res.converged and rel <= 0.01, (res.converged, rel, res.alpha)


def test_criterion_09_dao_identities():
    """Criterion 9 (tests/test_acceptance.py:379-401): with zero drift the
    drift-adjusted optimality equals the plain optimality; after a 50% cut on
    the most loaded link the stale allocation carried into the new state scores
    below a re-solve."""
    import types
    rng = np.random.default_rng(777)
    inst = _singlepath(777, int(rng.integers(5, 21)))
    theta = pf.default_theta(inst)
    base = pf.solve(inst, pf.SolverConfig())
    alloc = types.SimpleNamespace(rates=base.rates, sums=pf.commodity_sums(inst, base.rates))
    ref = types.SimpleNamespace(sums=maxmin_singlepath(inst))
    zero_drift_equal = (pf.dao_evaluate(alloc, inst, ref, theta)
                        == pf.optimality_from_sums(alloc.sums, ref.sums, theta))
    loaded = int(np.argmax(pf.edge_loads(inst, base.rates)))
    cut = np.asarray(inst.capacity, float).copy()
    cut[loaded] *= 0.5
    drifted = pf.with_conditions(inst, capacity=cut)
    dref = types.SimpleNamespace(sums=maxmin_singlepath(drifted))
    stale = pf.dao_evaluate(alloc, drifted, dref, theta)
    fresh = pf.solve(drifted, pf.SolverConfig())
    resolved = pf.optimality_from_sums(pf.commodity_sums(drifted, fresh.rates), dref.sums, theta)
    assert zero_drift_equal and stale < resolved, (zero_drift_equal, stale, resolved)


def _two_unequal(cap, d0, d1):
    from b200_helpers import make_instance
    big = 100 * max(cap, d0, d1)
    return make_instance([("s0", "M", big, 1), ("s1", "M", big, 1), ("M", "T", cap, 1)],
                         [("s0", "T", d0, [(0, 2)]), ("s1", "T", d1, [(1, 2)])])


def test_criterion_03_projection_feasible_idempotent():
    """Criterion 3 (tests/test_acceptance.py:169-208): 10,000 randomised and
    boundary inputs over the same five instances -- the GPU projection is
    feasible at 1e-9 and idempotent on every one."""
    from b200_helpers import chain, diamond, shared_edge
    topo = pf.random_topology(12, seed=99)
    tab = pf.gravity_table(topo, 1.5 * float(topo.capacity.sum()))
    medium = pf.build_instance(topo, tab, pf.k_shortest_paths(topo, tab, k=2), device=0)
    insts = [chain(), diamond(), shared_edge(3, cap=7.0, demand=4.0), _two_unequal(10.0, 2.0, 20.0), medium]
    rng = np.random.default_rng(404)
    checked = infeasible = non_idempotent = 0
    for inst in insts:
        n = inst.num_paths
        cap_floor = float(np.min(inst.capacity))
        dem = np.asarray(inst.demand, float)
        d_max = float(dem.max())
        path_com = np.asarray(inst.path_com)
        for _ in range(2000):
            kind = rng.integers(5)
            if kind == 0:
                raw = rng.uniform(-d_max, 2 * d_max, n)
            elif kind == 1:
                raw = np.full(n, cap_floor / max(n, 1)) + rng.uniform(-1e-9, 1e-9, n)
            elif kind == 2:
                raw = dem[path_com] + rng.uniform(-1e-9, 1e-9, n)
            elif kind == 3:
                raw = rng.uniform(0.0, 1.0, n) * 1e3 * d_max
            else:
                raw = np.where(rng.random(n) < 0.3, 0.0, rng.uniform(0, d_max, n))
            alpha = int(rng.choice([0, 1, 2]))
            out = pf.project(inst, raw, alpha)
            checked += 1
            infeasible += not pf.validate_allocation(inst, out).feasible
            non_idempotent += not np.array_equal(pf.project(inst, out, alpha), out)
    assert checked == 10_000 and infeasible == 0 and non_idempotent == 0, (checked, infeasible, non_idempotent)


def _bisect_linear(w, beta, q):
    """Sign-agnostic bisection for alpha = 0 (tests/test_acceptance.py:211-224)."""
    lin, c = 1.0 + w, w / beta
    span = 1.0 + abs(q) + c
    lo, hi = -span, span
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if lin * mid - c - q >= 0.0:
            hi = mid
        else:
            lo = mid
    return 0.5 * (lo + hi)


def _bisect_root(w_sum, beta, q, alpha, tol=1e-12):
    """Pure-bisection root of (1+W)S - (W/beta)S^(-alpha) - Q on (0, inf)
    (tests/helpers.py:92-112), independent of the Newton path."""
    lin, c = 1.0 + w_sum, w_sum / beta

    def f(s):
        return lin * s - c * s ** (-float(alpha)) - q if alpha else lin * s - c - q
    lo, hi = 1e-300, max(1.0, q / lin)
    while f(hi) < 0.0:
        hi *= 2.0
    for _ in range(20000):
        mid = 0.5 * (lo + hi)
        if f(mid) >= 0.0:
            hi = mid
        else:
            lo = mid
        if hi - lo <= tol * max(1.0, hi):
            break
    return 0.5 * (lo + hi)


def _rate_block_objective(inst, st, x, alpha):
    """The x-block objective the rate update minimises (tests/helpers.py:119-131)."""
    x = np.asarray(x, np.float64)
    sums = pf.commodity_sums(inst, x)
    val = -np.sum(pf.utility(sums, alpha)) / st.beta
    val += 0.5 * np.sum(np.maximum(sums - (np.asarray(inst.demand) - st.dual_demand), 0.0) ** 2)
    diff = x[np.asarray(inst.pair_path)] - st.y + st.dual_consensus
    val += 0.5 * np.sum(diff ** 2)
    val += 0.5 * np.sum(np.maximum(st.dual_nonneg - x, 0.0) ** 2)
    return float(val)


def _random_state(inst, rng, beta, alpha, nonneg_floor=False):
    import states
    a = states.random_state(inst.num_commodities, inst.num_paths, inst.num_edges, inst.num_pairs, rng,
                            nonneg_floor=nonneg_floor)
    return pf.SolverState(**a, beta=beta, alpha=alpha, iteration=0)


def test_criterion_04_kernel_exactness():
    """Criterion 4 (tests/test_acceptance.py:227-284) on the GPU kernels: 1,000
    roots (residual and bisection gap <= 1e-8), sum consistency of the rate
    update (<= 1e-8) and stationarity of the rate block by finite differences
    (<= 1e-4)."""
    from b200_helpers import chain, diamond, shared_edge
    rng = np.random.default_rng(88)
    worst_f = worst_agree = 0.0
    for _ in range(1000):
        w = float(rng.uniform(1e-6, 10.0))
        beta = float(10 ** rng.uniform(-3, 3))
        q = float(rng.uniform(-1e3, 1e3))
        alpha = int(rng.choice([0, 1, 2, 3, 8]))
        s = pf.solve_sum_equation(w, beta, q, alpha)
        f = (1 + w) * s - (w / beta) * (s ** (-alpha) if alpha else 1.0) - q
        worst_f = max(worst_f, abs(f) / max(1.0, abs(q)))
        ref = _bisect_linear(w, beta, q) if alpha == 0 else _bisect_root(w, beta, q, alpha)
        worst_agree = max(worst_agree, abs(s - ref) / max(1.0, abs(ref)))
    assert worst_f <= 1e-8 and worst_agree <= 1e-8, (worst_f, worst_agree)

    worst_sum = 0.0
    for alpha in (0, 1, 2, 4):
        for inst in (chain(), diamond(), shared_edge(3)):
            for _ in range(5):
                st = _random_state(inst, rng, float(rng.uniform(0.2, 4)), alpha, nonneg_floor=True)
                sums = pf.solve_commodity_sums(st, inst, alpha)
                st.x = pf.update_rates(st, inst, sums, alpha)
                got = pf.commodity_sums(inst, st.x)
                worst_sum = max(worst_sum, float((np.abs(got - sums) / np.maximum(1.0, np.abs(sums))).max()))
    assert worst_sum <= 1e-8, worst_sum

    h = 1e-5
    worst_grad = 0.0
    insts = (chain(), diamond(), shared_edge(2))
    for i in range(20):
        alpha = i % 2
        inst = insts[i % 3]
        st = _random_state(inst, rng, float(rng.uniform(0.3, 3)), alpha)
        dd, dc, dcon, dn = pf.update_duals(st, inst)
        sd, sc = pf.update_slacks(st, inst)
        st.dual_demand, st.dual_capacity, st.dual_consensus, st.dual_nonneg = dd, dc, dcon, dn
        st.slack_demand, st.slack_capacity = sd, sc
        st.y = pf.update_rate_suggestions(st, inst)
        sums = pf.solve_commodity_sums(st, inst, alpha)
        st.x = pf.update_rates(st, inst, sums, alpha)
        for p in range(inst.num_paths):
            up, down = st.x.copy(), st.x.copy()
            up[p] += h
            down[p] -= h
            grad = (_rate_block_objective(inst, st, up, alpha) - _rate_block_objective(inst, st, down, alpha)) / (2 * h)
            worst_grad = max(worst_grad, abs(grad))
    assert worst_grad <= 1e-4, worst_grad


# ---------------------------------------------------------------- criteria 2 and 7
# The reference's grid oracle (oracles.py:158 exact_bruteforce_tiny) on its own
# instance families, recorded by tests/golden/make_golden_acceptance.py.


def _acc_golden():
    import os
    import golden_io as G
    p = os.path.join(G.GOLDEN, "golden_acceptance.npz")
    if not os.path.exists(p):
        pytest.skip("golden_acceptance.npz not generated")
    return dict(np.load(p))


def _acc_instance(A, key):
    f = {k: A[f"{key}/in/{k}"] for k in ("capacity", "demand0", "com_path_ptr0", "path_edge_ptr0", "path_edges0")}
    return pf.build_instance_raw(f["capacity"], f["demand0"], f["com_path_ptr0"], f["path_edge_ptr0"],
                                 f["path_edges0"], device=0)


def _objective(sums, alpha):
    return float(np.sum(pf.utility(np.maximum(sums, 1e-12), alpha)))


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_criterion_02_tiny_multipath_objective(mode):
    """tests/test_acceptance.py:142-166: 20 instances x alpha in (0, 1, 2), the
    objective gap to the grid oracle within max(2% of the optimum, one grid
    step's first-order cost on every commodity)."""
    A = _acc_golden()
    n = len({k.split("/")[1] for k in A if k.startswith("c2/")})
    assert n == 20
    worst = -np.inf
    for i in range(n):
        inst = _acc_instance(A, f"c2/{i}")
        step = float(A[f"c2/{i}/step"][0])
        theta = pf.default_theta(inst)
        for alpha in (0, 1, 2):
            ref = A[f"c2/{i}/a{alpha}/ref_sums"]
            res = pf.solve(inst, pf.SolverConfig(alpha_target=alpha, mode=mode))
            gap = _objective(ref, alpha) - _objective(res.sums, alpha)
            one_step = step * float(np.sum(np.maximum(ref, theta) ** (-float(alpha))))
            allowed = max(0.02 * abs(_objective(ref, alpha)), one_step)
            worst = max(worst, gap / allowed)
            assert gap <= allowed, (i, alpha, gap, allowed)
    assert worst <= 1.0


@pytest.mark.parametrize("mode", ["fast", "exact"])
def test_criterion_07_alpha_continuation_trend(mode):
    """tests/test_acceptance.py:331-365: max-min optimality non-decreasing over
    alpha_target 0..3 (within one grid step), and >= 0.85 at alpha 0 on the
    symmetric instances."""
    A = _acc_golden()
    for i in range(5):
        inst = _acc_instance(A, f"c7/{i}")
        step = float(A[f"c7/{i}/step"][0])
        ref = A[f"c7/{i}/ref_sums"]
        theta = pf.default_theta(inst)
        dip = step * float(np.mean(1.0 / np.maximum(ref, theta)))
        opts = [pf.optimality_from_sums(pf.solve(inst, pf.SolverConfig(alpha_target=a, mode=mode)).sums, ref, theta)
                for a in (0, 1, 2, 3)]
        for lo, hi in zip(opts, opts[1:]):
            assert hi >= lo - dip - 1e-12, (i, opts)
        if bool(A[f"c7/{i}/sym"][0]):
            assert opts[0] >= 0.85, (i, opts)
