"""Reference-side drop-in: the reference package's own `solve()` call sites
run on the B200.

The reference binds `solve` by name in its two callers
(`pathfair/harness.py:23` -> `_run_named_solver`, `harness.py:464`;
`pathfair/cli.py:20` -> `_cmd_solve`, `cli.py:147`).  `install(pathfair)`
rebinds those names to `solve` below, which takes the reference's own
`Instance` and `SolverConfig`, runs this package's GPU solver, and returns the
reference's own `SolveResult` / `IterationTrace` types, raising the
reference's own `InputError` / `KernelError` / `SolverError`.

Nothing here imports the reference: its modules are reached through the
objects the caller passes in (or the package handed to `install`).
"""

from __future__ import annotations

import importlib
import sys

import numpy as np

from .controller import SolverConfig, SolverError, solve as _solve
from .kernels import KernelError
from .model import FlatPathSet, InputError, build_instance_flat, with_conditions
from .topology import CommodityTable, Topology

_CONFIG_FIELDS = ("alpha_target", "gamma", "beta0", "residual_ratio", "beta_scale", "max_iterations",
                  "beta_min", "beta_max", "adapt", "trace", "reference_sums")


def _ref_modules(ref_instance):
    pkg = type(ref_instance).__module__.rsplit(".", 1)[0]
    return (importlib.import_module(f"{pkg}.model"), importlib.import_module(f"{pkg}.kernels"),
            importlib.import_module(f"{pkg}.controller"))


def from_reference_instance(ref_instance, device=None):
    """A GPU Instance with the same index spaces as the reference's
    `Instance` (model.py:135-180): the retained commodities, their paths in
    order (`pair_ptr` / `pair_edge` are exactly the flat path set), and the
    instance's current capacity / demand (with_conditions may have replaced them,
    model.py:274-294)."""
    t = ref_instance.topology
    topo = Topology(tuple(t.nodes), np.asarray(t.edge_src, np.int64), np.asarray(t.edge_dst, np.int64),
                    np.asarray(t.capacity, np.float64), np.asarray(t.weight, np.float64))
    table = CommodityTable.from_commodities(topo, ref_instance.commodities)
    flat = FlatPathSet(np.asarray(ref_instance.com_path_ptr, np.int64), np.asarray(ref_instance.pair_ptr, np.int64),
                       np.asarray(ref_instance.pair_edge, np.int64))
    g = build_instance_flat(topo, table, flat, device)
    cap = np.asarray(ref_instance.capacity, np.float64)
    dem = np.asarray(ref_instance.demand, np.float64)
    if not (np.array_equal(cap, g.capacity) and np.array_equal(dem, g.demand)):
        g = with_conditions(g, capacity=cap, demand=dem)
    return g


def solve(instance, config=None, warm_start=None):
    """controller.py:197 `solve(instance, config, warm_start) -> SolveResult`,
    with the reference's types in and out, computed on the GPU."""
    rmodel, rkernels, rcontroller = _ref_modules(instance)
    cfg = config if config is not None else rcontroller.SolverConfig()
    gcfg = SolverConfig(**{f: getattr(cfg, f) for f in _CONFIG_FIELDS}, mode=_MODE)
    try:
        g = _cached(instance)
        r = _solve(g, gcfg, warm_start)
    except InputError as exc:
        raise rmodel.InputError(str(exc)) from exc
    except KernelError as exc:
        raise rkernels.KernelError(str(exc)) from exc
    except SolverError as exc:
        raise rcontroller.SolverError(str(exc)) from exc
    trace = None
    if r.trace is not None:
        trace = tuple(rcontroller.IterationTrace(t.iteration, t.alpha, t.beta, t.s, t.r, t.objective,
                                                 t.pct_violated, t.mean_relative_violation, t.optimality)
                      for t in r.trace)
    return rcontroller.SolveResult(r.rates, r.sums, r.iterations, r.alpha, r.converged, r.runtime_s, trace)


_MODE = "fast"
_CACHE: dict = {}


def _cached(ref_instance):
    """Reference instances are frozen and immutable (model.py:135): the GPU copy
    is built once per instance object."""
    key = id(ref_instance)
    hit = _CACHE.get(key)
    if hit is not None and hit[0] is ref_instance:
        return hit[1]
    g = from_reference_instance(ref_instance)
    while len(_CACHE) >= 4:  # a harness run walks many drifted snapshots
        _CACHE.pop(next(iter(_CACHE)))
    _CACHE[key] = (ref_instance, g)
    return g


def install(pathfair_pkg, mode: str = "fast"):
    """Rebind `solve` where the reference's harness and CLI imported it
    (harness.py:23, cli.py:20).  Returns a callable that restores them."""
    global _MODE
    _MODE = mode
    mods = []
    for name in ("harness", "cli"):
        m = sys.modules.get(f"{pathfair_pkg.__name__}.{name}") or importlib.import_module(
            f"{pathfair_pkg.__name__}.{name}")
        mods.append((m, m.solve))
        m.solve = solve

    def restore():
        for m, fn in mods:
            m.solve = fn
        _CACHE.clear()
    return restore
