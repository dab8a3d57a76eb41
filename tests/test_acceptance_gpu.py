"""SPEC acceptance criteria 1, 3, 5, 6, 8 and 9 (reference tests/test_acceptance.py:77-89,
169-208, 287-328, 368-401) with the GPU solvers swapped in for pathfair.solve: same
instance families, seeds and thresholds.  The single-path max-min reference is
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
