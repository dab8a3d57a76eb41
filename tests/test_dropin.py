"""The reference-side drop-in (paper_2605_01748_b200/dropin.py)
exercised at the reference's own entry points.

When the unmodified reference package is importable (baseline/_ref, installed
with pip --no-deps from /root/reference/pkg; skipped otherwise), `install()`
rebinds the `solve` that `pathfair.harness` (harness.py:23, used at :464) and
`pathfair.cli` (cli.py:20, used at :147) imported, and the reference's
test_controller.py:126-141 solves run through it on the GPU, returning the
reference's own result types.  Exact mode through the shim equals the
reference's own solve bitwise (alpha <= 1).
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _pathfair():
    try:
        import pathfair  # noqa: F401
    except ImportError:
        ref = os.path.join(ROOT, "baseline", "_ref")
        if not os.path.isdir(os.path.join(ref, "pathfair")):
            pytest.skip("reference package not installed (baseline/_ref)")
        sys.path.insert(0, ref)
    try:
        import pathfair
        import pathfair.cli  # noqa: F401
        import pathfair.harness  # noqa: F401
    except ImportError as exc:  # numba / networkx missing on this box
        pytest.skip(f"reference package not importable: {exc}")
    return pathfair


@pytest.fixture(scope="module")
def ref():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return _pathfair()


def _make(ref, edges, commodities):
    from pathfair.model import Commodity, PathSet, build_instance, build_topology
    topo = build_topology(edges)
    coms = [Commodity(s, d, dem) for s, d, dem, _ in commodities]
    return build_instance(topo, coms, PathSet.from_lists([p for _, _, _, p in commodities]))


# the reference's tests/helpers.py:25-62 builders (same rows)
def single_bottleneck(ref, cap=10.0, demand=20.0):
    return _make(ref, [("A", "B", cap, 1)], [("A", "B", demand, [(0,)])])


def shared_edge(ref, n=2, cap=10.0, demand=20.0):
    edges = [(f"s{i}", "M", 10 * n * max(cap, demand), 1) for i in range(n)] + [("M", "T", cap, 1)]
    return _make(ref, edges, [(f"s{i}", "T", demand, [(i, n)]) for i in range(n)])


def chain(ref, demand=100.0):
    return _make(ref, [("A", "B", 10, 1), ("B", "C", 5, 1)],
                 [("A", "B", demand, [(0,)]), ("A", "C", demand, [(0, 1)]), ("B", "C", demand, [(1,)])])


def test_reference_entry_points_run_on_gpu(ref):
    from paper_2605_01748_b200 import dropin
    from pathfair import cli, controller, harness
    original = harness.solve
    restore = dropin.install(ref)
    try:
        assert harness.solve is dropin.solve and cli.solve is dropin.solve
        # test_controller.py:126-141 through the rebound name
        res = harness.solve(single_bottleneck(ref), controller.SolverConfig(alpha_target=0))
        assert isinstance(res, controller.SolveResult)
        assert res.converged and res.sums[0] == pytest.approx(10.0, abs=0.1)
        res = harness.solve(shared_edge(ref), controller.SolverConfig())
        assert res.converged and res.sums == pytest.approx([5.0, 5.0], abs=0.1)
        res = harness.solve(chain(ref), controller.SolverConfig())
        assert res.converged and res.sums == pytest.approx([7.5, 2.5, 2.5], abs=0.15)
        # the harness's own call site (harness.py:454-466)
        cfg = {"alpha_target": None, "gamma": 1e-3, "beta0": 1.0, "max_iterations": 5000, "adapt_beta": True,
               "trace": True}
        alloc, iters, runtime, trace = harness._run_named_solver("pathfair", chain(ref), cfg, None)
        assert iters > 0 and runtime > 0 and len(trace) == iters
        assert isinstance(trace[0], controller.IterationTrace)
        assert np.allclose(sorted(alloc.rates), sorted(res.rates))
    finally:
        restore()
    assert harness.solve is original


def test_shim_exact_mode_equals_reference_bitwise(ref):
    from paper_2605_01748_b200 import dropin
    from pathfair import controller, harness
    orig = controller.solve
    inst = chain(ref)
    cfg = controller.SolverConfig(alpha_target=1)
    want = orig(inst, cfg)
    restore = dropin.install(ref, mode="exact")
    try:
        got = harness.solve(inst, cfg)
    finally:
        restore()
    assert (got.iterations, got.alpha, got.converged) == (want.iterations, want.alpha, want.converged)
    assert np.array_equal(got.rates, want.rates) and np.array_equal(got.sums, want.sums)


def test_shim_generated_instance_with_conditions(ref):
    """A generated WAN instance with drifted capacity (model.py:274-294) through
    the shim: same stop as the reference's own solve in exact mode, bitwise."""
    from paper_2605_01748_b200 import dropin
    from pathfair import controller, harness, model
    topo = harness.random_topology(24, seed=24)
    coms = harness.gravity_demands(topo, 0.3 * float(topo.capacity.sum()))
    inst = model.build_instance(topo, coms, harness.k_shortest_paths(topo, coms, 3))
    cap = inst.capacity.copy()
    cap[::9] = 0.0
    cut = model.with_conditions(inst, capacity=cap)
    cfg = controller.SolverConfig(alpha_target=1, max_iterations=400)
    want = controller.solve(cut, cfg)
    restore = dropin.install(ref, mode="exact")
    try:
        got = harness.solve(cut, cfg)
    finally:
        restore()
    assert got.iterations == want.iterations
    assert np.array_equal(got.rates, want.rates)


def test_shim_maps_errors_to_reference_types(ref):
    from paper_2605_01748_b200 import dropin
    from pathfair import controller, kernels, model
    inst = chain(ref)
    with pytest.raises(model.InputError):
        dropin.solve(inst, controller.SolverConfig(), warm_start=np.array([1.0, np.nan, 2.0]))
    try:
        controller.solve(inst, controller.SolverConfig(max_iterations=50), warm_start=np.full(3, 1e308))
        want = None
    except (kernels.KernelError, controller.SolverError) as exc:
        want = type(exc)
    try:
        dropin.solve(inst, controller.SolverConfig(max_iterations=50), warm_start=np.full(3, 1e308))
        got = None
    except (kernels.KernelError, controller.SolverError) as exc:
        got = type(exc)
    assert got is want
