"""Benchmark: GATE max-min-fair TE solver iterations/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl b200|reference]

A STEP is one solver iteration (kernels.py's five updates + residuals +
controller, controller.py:225-273) over the whole synthetic instance.  The
workload at N=1 is BASELINE config 2: a synthetic 500-node WAN (reference
random_topology(500, seed=500)), all-pairs gravity demands (V = 1.5 x total
capacity, the reference test-suite convention), k = 8 shortest paths:
249,500 demands / 1,996,000 paths / 18,282,422 demand-path pairs.

value : iterations/s of the fused device loop (inputs resident in HBM), timed
        with CUDA events around exactly K iterations after W warm-up iterations.
e2e   : the same metric through the reference-facing C-ABI call `pf_solve`
        with HOST buffers: warm-start rates H2D, K iterations, GPU projection,
        rates + sums D2H, all inside the timed region.
Working set (~0.5 GB) exceeds the 126 MB L2, so no L2 flush is needed.

Extra keys (rank 0, N=1): time_to_1pct on cfg1 / cfg2 / the north-star-scale
instance at V = 0.3 x capacity; config4_link_failure_resolve (5% of the links
cut, warm re-solve) and config5_alpha_sweep (alpha_target 0..4 and max-min) on
the 500-node WAN (--no-ttq / --no-extras skip them).

--impl reference times the reference algorithm's CPU implementation (the
exact-order C oracle, oracle/pf_oracle.c, OpenMP over all host cores) on the
same config; each step is one iteration.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TE solve time to within 1% of optimal max-min (ms); iterations/s at 1/2/4/8 B200"
CONFIGS = {
    # name: (nodes, k, volume fraction of total capacity, description)
    "cfg1": (40, 4, 1.5, "GEANT-sized: random_topology(40), all-pairs gravity, k=4"),
    "cfg1_v0.3": (40, 4, 0.3, "GEANT-sized, V=0.3*cap (reference stop rule fires)"),
    "cfg2": (500, 8, 1.5, "synthetic 500-node WAN, all-pairs gravity, k=8 (~18.3M demand-path pairs)"),
    "cfg2_v0.3": (500, 8, 0.3, "500-node WAN, V=0.3*cap, k=8"),
    "mid150_v0.3": (150, 4, 0.3, "150-node all-pairs gravity, k=4, V=0.3*cap (tuning: mid-size instances)"),
    "target_k4_v0.3": (500, 4, 0.3, "north-star target scale: 500-node all-pairs, k=4 (~1M paths), V=0.3*cap"),
    "cfg3": (2000, 8, 1.5, "synthetic 2000-node WAN-A-scale, all-pairs gravity, k=8 (~355M demand-path pairs)"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PF_BENCH_SHARE_GPU") == "1":
        # test hook: time-slice several ranks on the GPUs present (the line then
        # says so in config.shared_gpus); never set by the driver
        import torch
        local %= max(1, torch.cuda.device_count())
    return rank, world, local


def cache_path(name):
    return os.path.join(ROOT, "data", f"{name}.npz")


def build_inputs(name):
    """(topology, commodity table, flat path set) for a config, from this
    package's generators (pinned to the reference's: tests/test_generators.py,
    tests/golden/golden_ksp.json); paths cached under data/."""
    import paper_2605_01748_b200 as pf
    from paper_2605_01748_b200 import gen
    n, k, vol, _ = CONFIGS[name]
    cache = cache_path(name)
    topo = pf.random_topology(n, seed=n)
    tab = pf.gravity_table(topo, vol * float(topo.capacity.sum()))
    if os.path.exists(cache):
        z = np.load(cache)
        flat = pf.FlatPathSet(z["cpp"], z["pep"], z["pe"])
    else:
        t = time.perf_counter()
        flat = pf.k_shortest_paths(topo, tab, k)
        log(f"[bench] k_shortest_paths({name}) {time.perf_counter() - t:.1f}s (native, {os.cpu_count()} threads)")
        try:
            gen.write(cache, n, k, vol, topo, tab, flat)
        except OSError:
            pass
    return topo, tab, flat


def reference_inputs(name):
    """The same inputs for the reference arm WITHOUT loading this package's
    solver: a cached file, else the generator step (paper_2605_01748_b200.gen,
    host-only libpf_gen.so) run as a separate process."""
    n, k, vol, _ = CONFIGS[name]
    cache = cache_path(name)
    z = np.load(cache) if os.path.exists(cache) else None
    if z is None or "capacity" not in z:
        subprocess.run([sys.executable, "-m", "paper_2605_01748_b200.gen", "--nodes", str(n), "--k", str(k),
                        "--volume", str(vol), "--out", cache], check=True, cwd=ROOT)
        z = np.load(cache)
    return z["capacity"], z["demand"], z["cpp"], z["pep"], z["pe"]


def algorithmic_bytes(C, P, NP, E):
    """SURVEY 8(d) B_iter: bytes one iteration must move with y stored (fp64
    state, int32 indices): 36/pair + 40/path + 32/commodity + 32/edge."""
    return 36 * NP + 40 * P + 32 * C + 32 * E


B200_L2_BYTES = 132644864  # queried on the pool's B200s (cudaDevAttrL2CacheSize)


def workload_config(name, C, P, NP, E, world):
    """The `config` object -- identical in both arms (same workload, same keys)."""
    try:
        import torch
        l2 = int(torch.cuda.get_device_properties(0).L2_cache_size) if torch.cuda.is_available() else B200_L2_BYTES
    except Exception:  # noqa: BLE001
        l2 = B200_L2_BYTES
    ws = algorithmic_bytes(C, P, NP, E) // max(world, 1)
    if ws > l2:
        how = "inputs larger than L2 (no flush)"
    else:
        how = ("per-GPU working set fits in L2: iterations after the first are L2-resident "
               "(one persistent launch, no flush between iterations)")
    return {"workload": name, "description": CONFIGS[name][3], "commodities": int(C), "paths": int(P),
            "pairs": int(NP), "edges": int(E), "parallelism": f"dp{world}" if world > 1 else "single",
            "l2": how, "l2_bytes": l2, "working_set_bytes_per_gpu": int(ws)}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML every 2 ms from a thread (the timed loop is one blocking
    native call that releases the GIL); nvidia-smi as a fallback."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index=0, period_s=0.002):
        self.index = index
        self.period = period_s
        self.samples = []  # (sm_mhz, reasons_mask)
        self.max_mhz = None
        self._stop = threading.Event()
        self.th = None
        self.nvml = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            # the first NVML queries are slow: issue them here, outside the timed
            # region, and return only once the thread is sampling
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            first = threading.Event()

            def run():
                while not self._stop.is_set():
                    try:
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((mhz, rs))
                    except Exception:  # noqa: BLE001
                        pass
                    first.set()
                    time.sleep(self.period)
            self.th = threading.Thread(target=run, daemon=True)
            self.th.start()
            first.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.nvml = None
        return self

    def stop(self):
        self._stop.set()
        if self.th:
            self.th.join(timeout=2)
        if self.nvml is None or not self.samples:
            return self._smi_once()
        sm = [m for m, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml (2 ms)"}

    def _smi_once(self):
        try:
            out = subprocess.run(["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=10).stdout.strip().split(",")
            return {"sm_mhz": float(out[0]), "sm_max_mhz": float(out[1]), "reasons": [], "samples": 1,
                    "source": "nvidia-smi after the timed region"}
        except Exception:  # noqa: BLE001
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def profile_traffic(name):
    """dram bytes per launch from the committed ncu summary (profiles/), if present."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(name, {}).get("dram_bytes_per_iteration")
    except (OSError, ValueError):
        return None


def cpu_baseline(flat, tab, topo, budget_s=15.0):
    """The reference algorithm on the host cores (C oracle, OpenMP): iterations/s
    on a bounded sample (a few iterations of the same instance)."""
    from oracle import oracle as O
    I = O.build_instance(topo.capacity, tab.demand, flat.com_path_ptr, flat.path_edge_ptr, flat.path_edges)
    threads = O.num_threads()
    loop = O.Loop(I, O.make_config(gamma=1e-12, max_iterations=10 ** 6))
    loop.step(1)  # warm
    t = time.perf_counter()
    n = 0
    while True:
        loop.step(1)
        n += 1
        dt = time.perf_counter() - t
        if dt > budget_s or n >= 200:
            break
    return {"value": n / dt, "unit": "iterations/s", "cores": threads, "kind": "port",
            "sample": f"{n} iterations of the full instance (C oracle, exact reference op order)"}


def oracle_fixed_point(name):
    """The reference algorithm's own fixed point for a ttq instance, computed
    once by the oracle (tests/golden/make_golden_fixed_points.py, committed):
    (meta, post-projection commodity sums) or None."""
    pj = os.path.join(ROOT, "tests", "golden", "golden_fixed_points.json")
    pz = os.path.join(ROOT, "tests", "golden", "golden_fixed_points.npz")
    if not (os.path.exists(pj) and os.path.exists(pz)):
        return None
    with open(pj) as fh:
        meta = json.load(fh)
    if name not in meta:
        return None
    return meta[name], np.load(pz)[f"{name}/opt_sums"]


def time_to_quality(name, device=0, cpu=True, chunk=None):
    """Time to within 1% of the reference algorithm's fixed point.

    OPT_ref = the post-projection commodity sums of the reference algorithm's
    own solve (the exact-order oracle run to its stagnation stop or the
    5,000-iteration cap; committed fixture), or -- when no fixture exists for the
    instance -- the fast solver's own end point (flagged).  k* = first iteration
    whose post-projection optimality_from_sums(S_k, OPT_ref, default_theta) >=
    0.99 (oracles.py:51-53, 244-254).  The timed figure is the device time of k*
    fused iterations (one launch) plus one GPU projection.  The reference
    trajectory's own k* comes with the fixture; the CPU column times the C oracle
    for that many iterations plus one projection (measured when cheap, else
    extrapolated from a bounded sample and marked so)."""
    import paper_2605_01748_b200 as pf
    topo, tab, flat = build_inputs(name)
    inst = pf.build_instance_flat(topo, tab, flat, device=device)
    fp = oracle_fixed_point(name)
    theta = pf.default_theta(inst)
    if fp is not None:
        meta, opt = fp
        opt_kind = "reference algorithm's fixed point (exact-order oracle, tests/golden/golden_fixed_points.npz)"
        own = None
    else:
        s = pf.Solver(inst, pf.SolverConfig(mode="fast", max_iterations=5000)).init()
        s.run(5000)
        _, own = s.finish()
        meta, opt = None, own
        opt_kind = "fast solver's own end point (no oracle fixture for this instance)"
    # k*: one pass on the device (sampled post-projection optimality, the crossing
    # chunk replayed from a device snapshot; pf_solver_time_to_quality)
    srch = pf.Solver(inst, pf.SolverConfig(mode="fast", max_iterations=5000)).init()
    found = srch.time_to_quality(opt, 0.99, sample_every=chunk or 125)
    kstar = found["k_star"]
    srch.run(5000)  # on to the algorithm's own stop: its end point vs OPT_ref
    r = srch.result()
    _, end = srch.finish()
    hi = kstar if kstar is not None else int(r.iterations)
    t = pf.Solver(inst, pf.SolverConfig(mode="fast", max_iterations=5000)).init()
    ms_loop, _ = t.time_loop(hi)
    t.finish()
    ms_proj = t.result().projection_ms
    out = {"config": name, "k_star": kstar, "opt_ref": opt_kind,
           "end_optimality_vs_opt_ref": pf.optimality_from_sums(end, opt, theta),
           "fast_stop": {"iterations": int(r.iterations), "alpha": int(r.alpha), "converged": bool(r.converged)},
           "k_star_search": {"how": "one device pass: optimality sampled every "
                                    f"{chunk or 125} iterations, crossing chunk replayed from a device snapshot",
                             "samples": len(found["samples"]), "loop_ms": found["loop_ms"],
                             "quality_ms": found["quality_ms"]},
           "gpu_ms": ms_loop + ms_proj, "gpu_loop_ms": ms_loop, "gpu_projection_ms": ms_proj,
           "pairs": inst.num_pairs, "mode": "fast"}
    if meta is not None:
        out["reference"] = {"k_star": meta["k_star"], "iterations": meta["iterations"], "alpha": meta["alpha"],
                            "converged": meta["converged"]}
    k_cpu = meta["k_star"] if meta is not None and meta["k_star"] else kstar
    if cpu and k_cpu:
        from oracle import oracle as O
        I = O.build_instance(topo.capacity, tab.demand, flat.com_path_ptr, flat.path_edge_ptr, flat.path_edges)
        loop = O.Loop(I, O.make_config(max_iterations=5000))
        t0 = time.perf_counter()
        loop.step(1)
        t1 = time.perf_counter() - t0
        if t1 * k_cpu < 60.0:
            t0 = time.perf_counter()
            loop2 = O.Loop(I, O.make_config(max_iterations=5000))
            loop2.step(k_cpu)
            st = loop2.state()
            O.project(I, st.x, st.alpha)
            out["cpu_ms"] = 1e3 * (time.perf_counter() - t0)
            out["cpu_kind"] = "measured"
        else:
            loop.step(3)
            per = (time.perf_counter() - t0 - t1) / 3
            st = loop.state()
            t0 = time.perf_counter()
            O.project(I, st.x, st.alpha)
            pj = time.perf_counter() - t0
            out["cpu_ms"] = 1e3 * (per * k_cpu + pj)
            out["cpu_kind"] = "extrapolated from 3 iterations + 1 projection"
        out["cpu_iterations"] = int(k_cpu)
        out["cpu_cores"] = O.num_threads()
    return out


def config45(name, device=0):
    """BASELINE configs 4 and 5 at config-2 scale, fast mode:
    4: after a cold solve, cut 5% of the links (rng = default_rng(1), capacity 0
       via with_conditions, paths kept as in run_experiment) and re-solve warm
       from the previous rates with alpha_target = the previous alpha;
    5: the alpha_target sweep {0, 1, 2, 3, 4, None} (max-min) from cold starts.
    Times are the solver's runtime_s (init through projection, controller.py:276)."""
    import paper_2605_01748_b200 as pf
    topo, tab, flat = build_inputs(name)
    inst = pf.build_instance_flat(topo, tab, flat, device=device)
    cold = pf.solve(inst, pf.SolverConfig(mode="fast"))
    rng = np.random.default_rng(1)
    E = inst.num_edges
    cut = rng.choice(E, int(round(0.05 * E)), replace=False)
    cap = np.array(topo.capacity, np.float64)
    cap[cut] = 0.0
    failed = pf.with_conditions(inst, capacity=cap)
    warm = pf.solve(failed, pf.SolverConfig(mode="fast", alpha_target=int(cold.alpha)), warm_start=cold.rates)
    fresh = pf.solve(failed, pf.SolverConfig(mode="fast", alpha_target=int(cold.alpha)))
    theta = pf.default_theta(failed)
    out4 = {"config": name, "links_cut": int(cut.size),
            "cold_solve": {"iterations": int(cold.iterations), "alpha": int(cold.alpha),
                           "converged": bool(cold.converged), "ms": 1e3 * cold.runtime_s},
            "warm_resolve": {"iterations": int(warm.iterations), "converged": bool(warm.converged),
                             "ms": 1e3 * warm.runtime_s,
                             "feasible": bool(pf.validate_allocation(failed, warm.rates).feasible),
                             "optimality_vs_cold_resolve": pf.optimality_from_sums(warm.sums, fresh.sums, theta)},
            "cold_resolve": {"iterations": int(fresh.iterations), "converged": bool(fresh.converged),
                             "ms": 1e3 * fresh.runtime_s}}
    # the stale allocation carried into the failed state (oracles.py:262-297,
    # bitwise the reference's): wall time of the GPU carry, host buffers
    pf.dao_carry_rates(cold.rates, failed)  # warm (workspace)
    t0 = time.perf_counter()
    carried = pf.dao_carry_rates(cold.rates, failed)
    dao_ms = 1e3 * (time.perf_counter() - t0)
    out4["dao_carry"] = {"ms": dao_ms, "feasible": bool(pf.validate_allocation(failed, carried).feasible),
                         "dao_evaluate_vs_cold_resolve": pf.dao_evaluate(cold, failed, fresh, theta)}
    out5 = []
    for at in (0, 1, 2, 3, 4, None):
        r = pf.solve(inst, pf.SolverConfig(mode="fast", alpha_target=at))
        out5.append({"alpha_target": at, "iterations": int(r.iterations), "alpha": int(r.alpha),
                     "converged": bool(r.converged), "ms": 1e3 * r.runtime_s,
                     "min_sum": float(np.min(r.sums)) if r.sums.size else None,
                     "feasible": bool(pf.validate_allocation(inst, r.rates).feasible)})
    return out4, out5


REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # the unmodified reference, pip-installed (git-ignored)


def reference_numba(name, cpp, pep, pe, iterations=2):
    """The reference's OWN implementation (pathfair, Python + numba, installed
    unmodified into baseline/_ref) timed on this host for `iterations` loop
    bodies (controller.py:226-236: update_duals, update_slacks,
    update_rate_suggestions, solve_commodity_sums, update_rates,
    compute_residuals, called through the reference's public kernel API) at
    set_threads(cpu_count) and set_threads(1).  The
    instance is the reference's build_instance of its own random_topology /
    gravity_demands with the k-shortest paths of this workload (the native
    KSP, pinned equal to the reference's networkx one).  Runs in a child
    process (numba's thread pool is sized at import).  Reported next to the
    C port; the arm's value stays the port's."""
    if not os.path.isdir(os.path.join(REF_DIR, "pathfair")):
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref the reference)"}
    if int(pe.size) > 50_000_000:
        # the reference's build_instance takes a nested-tuple PathSet: at config 3
        # (355M pairs) that is tens of GB of Python objects and hours of work
        return {"unavailable": f"{int(pe.size):,} pairs: the reference's PathSet (nested Python tuples) does not "
                               f"fit a bounded run; timed at config 2 instead"}
    import tempfile
    n, k, vol, _ = CONFIGS[name]
    with tempfile.TemporaryDirectory() as td:
        np.savez(os.path.join(td, "paths.npz"), cpp=cpp, pep=pep, pe=pe)
        env = dict(os.environ, NUMBA_CACHE_DIR=os.path.join(td, "nb"), NUMBA_NUM_THREADS=str(os.cpu_count()),
                   PYTHONPATH=REF_DIR)
        code = f"""
import copy, json, os, time
import numpy as np
import pathfair as R
from pathfair import kernels as K, controller as Ctl, _reduce as RD
z = np.load({os.path.join(td, "paths.npz")!r})
cpp, pep, pe = z["cpp"], z["pep"], z["pe"]
topo = R.harness.random_topology({n}, seed={n})
coms = R.harness.gravity_demands(topo, {vol} * float(topo.capacity.sum()))
lists = [[tuple(int(e) for e in pe[pep[p]:pep[p + 1]]) for p in range(cpp[c], cpp[c + 1])] for c in range(len(coms))]
t0 = time.perf_counter()
inst = R.build_instance(topo, coms, R.PathSet.from_lists(lists))
t_build = time.perf_counter() - t0
cfg = Ctl.SolverConfig(gamma=1e-12)
out = {{"build_instance_s": t_build, "pairs": int(inst.num_pairs)}}
def body(state):
    prev = copy.copy(state)
    dd, dc, dcon, dn = K.update_duals(state, inst)
    sd, sc = K.update_slacks(state, inst)
    state.dual_demand, state.dual_capacity, state.dual_consensus, state.dual_nonneg = dd, dc, dcon, dn
    state.slack_demand, state.slack_capacity = sd, sc
    state.y = K.update_rate_suggestions(state, inst)
    sums = K.solve_commodity_sums(state, inst, state.alpha)
    state.x = K.update_rates(state, inst, sums, state.alpha)
    Ctl.compute_residuals(prev, state)
for threads in (os.cpu_count(), 1):
    eff = RD.set_threads(threads)
    state = Ctl.initialize_state(inst, cfg)
    body(state)  # JIT + warm-up
    t = time.perf_counter()
    for _ in range({iterations}):
        body(state)
    dt = (time.perf_counter() - t) / {iterations}
    out[f"threads_{{eff}}"] = {{"iterations_per_s": 1.0 / dt, "ms_per_iteration": 1e3 * dt}}
print(json.dumps(out))
"""
        try:
            r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        except subprocess.TimeoutExpired:
            return {"unavailable": "timed out"}
        if r.returncode != 0:
            return {"unavailable": (r.stderr.strip().splitlines() or ["failed"])[-1][:300]}
        out = json.loads(r.stdout.strip().splitlines()[-1])
    out.update(kind="reference (pathfair, numba, unmodified, baseline/_ref)", workload=name,
               sample=f"{iterations} loop bodies per thread count after one warm-up body")
    return out


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (the
    exact-order C oracle, all host threads) on the same workload; rank 0 only.
    This process never loads the B200 solver library: inputs come from the
    generator step (a separate process) or its cached file."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    name = resolve_config(args, world)
    cap, dem, cpp, pep, pe = reference_inputs(name)
    I = O.build_instance(cap, dem, cpp, pep, pe)
    loop = O.Loop(I, O.make_config(gamma=1e-12, max_iterations=10 ** 7))
    # each step = one iteration; bound the run to a few minutes
    t0 = time.perf_counter()
    loop.step(1)
    t_it = time.perf_counter() - t0
    budget = 120.0
    warm = min(args.warmup, max(1, int(10.0 / max(t_it, 1e-6))))
    steps = min(args.steps, max(3, int(budget / max(t_it, 1e-6))))
    loop.step(warm)
    t = time.perf_counter()
    loop.step(steps)
    dt = time.perf_counter() - t
    assert loop.state().iteration == 1 + warm + steps
    v = steps / dt
    line = {"metric": METRIC, "value": v, "unit": "iterations/s", "n_gpus": world, "steps": steps,
            "warmup": warm, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(name, I.num_commodities, I.num_paths, I.num_pairs, I.num_edges, world),
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "iterations/s", "cores": O.num_threads(), "kind": "port",
                             "sample": f"{steps} iterations of the full instance (C oracle, exact reference "
                                       f"op order, OpenMP)"},
            "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not getattr(args, "no_reference_numba", False):
        line["reference_numba"] = reference_numba(name, cpp, pep, pe)
    print(json.dumps(line), flush=True)
    return 0


def resolve_config(args, world):
    """Default workload: config 2 on one GPU (BASELINE's single-B200 config),
    config 3 when sharded over N > 1 GPUs (BASELINE's multi-GPU config)."""
    return args.config or ("cfg2" if world == 1 else "cfg3")


def single_gpu_rate(name, device, steps=20, warmup=3):
    """Fused-loop iterations/s of one workload on one GPU (the N=1 point of a
    sharded config's scaling curve): `steps` iterations in one launch after
    `warmup`, so the window holds the beta ramp's rollback passes in the same
    proportion as the main line's 1,000 iterations do (rollbacks: a second pass
    on the iterations where beta changes, every 10 iterations while it ramps)."""
    import torch

    import paper_2605_01748_b200 as pf
    t0 = time.perf_counter()
    topo, tab, flat = build_inputs(name)
    t_gen = time.perf_counter() - t0
    inst = pf.build_instance_flat(topo, tab, flat, device=device)
    t_build = time.perf_counter() - t0 - t_gen
    s = pf.Solver(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)).init()
    s.time_loop(warmup)
    it0 = int(s.result().iterations)
    ms, _ = s.time_loop(steps)
    torch.cuda.synchronize()
    assert int(s.result().iterations) - it0 == steps, "the controller stopped inside the timed region"
    C, P, E, NP = inst.num_commodities, inst.num_paths, inst.num_edges, inst.num_pairs
    b = algorithmic_bytes(C, P, NP, E)
    peak, _ = measured_peaks()
    out = {"workload": name, "n_gpus": 1, "value": steps / (ms / 1e3), "unit": "iterations/s",
           "ms_per_step": ms / steps, "steps": steps, "pairs": NP, "edges": E,
           "roofline_frac": b * steps / (ms / 1e3) / 1e9 / peak, "inputs_s": t_gen, "instance_build_s": t_build}
    del s, inst
    return out


def run_b200(args):
    import torch

    import paper_2605_01748_b200 as pf
    rank, world, local = dist_env()
    args.config = resolve_config(args, world)
    if world > 1:
        from paper_2605_01748_b200 import distributed as D
        return D.bench_main(args, sys.modules[__name__])
    torch.cuda.set_device(local)
    topo, tab, flat = build_inputs(args.config)
    inst = pf.build_instance_flat(topo, tab, flat, device=local)
    C, P, E, NP = inst.num_commodities, inst.num_paths, inst.num_edges, inst.num_pairs
    cfg = pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)
    solver = pf.Solver(inst, cfg).init()
    # warm-up (W iterations, untimed)
    solver.time_loop(max(args.warmup, 3))
    torch.cuda.synchronize()
    it0 = int(solver.result().iterations)
    clocks = ClockSampler(local).start()
    t_wall = time.perf_counter()
    ms, ms_it = solver.time_loop(args.steps)  # CUDA events around exactly K iterations (one launch)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    clk = clocks.stop()
    done = int(solver.result().iterations) - it0
    if done != args.steps:
        raise RuntimeError(f"timed region ran {done} iterations, expected {args.steps}")
    value = args.steps / (ms / 1e3)

    # roofline: algorithmic bytes per launch / launch duration
    b_iter = algorithmic_bytes(C, P, NP, E)
    peak, peak_kind = measured_peaks()
    achieved = b_iter * args.steps / (ms / 1e3) / 1e9
    stats = solver.kernel_stats()

    # e2e through the C-ABI with host buffers (pf_solve: H2D warm start, K its, projection, D2H)
    # the step's input (warm-start rates) in pinned host memory
    warm = torch.empty(P, dtype=torch.float64).pin_memory().numpy()
    warm[:] = solver.x()
    e2e_cfg = pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=args.steps)
    pf.solve(inst, pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=3), warm_start=warm)  # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = pf.solve(inst, e2e_cfg, warm_start=warm)
    e2e_s = time.perf_counter() - t
    if res.iterations != args.steps:
        raise RuntimeError(f"e2e solve ran {res.iterations} iterations, expected {args.steps}")
    e2e = {"value": args.steps / e2e_s, "unit": "iterations/s", "h2d_bytes_per_step": 8 * P / args.steps,
           "d2h_bytes_per_step": 8 * (P + C) / args.steps, "projection_ms": res.projection_ms,
           "loop_ms": res.loop_ms, "wall_ms": 1e3 * e2e_s,
           "call": "pf_solve (pinned host warm start -> K iterations -> GPU projection -> host rates/sums)"}

    cpu = cpu_baseline(flat, tab, topo) if (rank == 0 and not args.no_cpu_baseline) else None
    ttq = None
    if rank == 0 and not args.no_ttq:
        ttq = [time_to_quality(n, device=local, cpu=not args.no_cpu_baseline) for n in args.ttq.split(",") if n]
    cfg4 = cfg5 = None
    if rank == 0 and not args.no_extras:
        cfg4, cfg5 = config45(args.extras_config, device=local)
    del solver
    sharded_n1 = None
    if rank == 0 and args.sharded_config and args.sharded_config != args.config:
        sharded_n1 = single_gpu_rate(args.sharded_config, local, steps=1000, warmup=10)
    line = {
        "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.config, C, P, NP, E, world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": profile_traffic(args.config), "peak_kind": peak_kind,
                     "bytes_per_iteration_algorithmic": b_iter,
                     "bytes_per_iteration_compulsory_this_layout": stats["bytes_per_iter"]},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "time_to_1pct": ttq,
        "config4_link_failure_resolve": cfg4,
        "config5_alpha_sweep": cfg5,
        "sharded_config_n1": sharded_n1,
        "clocks": clk,
        "gpu_launches": 1,
        "wall_s_timed_region": t_wall,
        "kernel": {"name": "pf::k_fused (cooperative persistent kernel)", "grid": stats["grid"],
                   "tiles": stats["tiles"], "launches_total": stats["launches"]},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(argv, n):
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) the
    way the driver does and return their exit status."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]
    return subprocess.run(cmd).returncode


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="workload (default: cfg2 on one GPU, cfg3 sharded over N > 1)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttq", action="store_true", help="skip the time-to-within-1%% measurement")
    ap.add_argument("--ttq", default="cfg1_v0.3,cfg2_v0.3,target_k4_v0.3", help="configs for time-to-within-1%%")
    ap.add_argument("--no-extras", action="store_true", help="skip the config 4 / config 5 measurements")
    ap.add_argument("--extras-config", default="cfg2_v0.3", help="instance for the config 4 / 5 measurements")
    ap.add_argument("--no-reference-numba", action="store_true",
                    help="reference arm: skip timing the reference's own numba implementation (baseline/_ref)")
    ap.add_argument("--sharded-config", default="cfg3",
                    help="at N=1 also time this workload on one GPU (the N=1 point of the sharded curve; '' skips)")
    args = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        return spawn_ranks(argv, args.gpus)
    if world and world != args.gpus and os.environ.get("PF_BENCH_SHARE_GPU") != "1":
        log(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}")
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
