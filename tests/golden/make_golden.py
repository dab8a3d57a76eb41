"""Generate the golden fixtures that pin the oracle to the reference.

Run HERE (the build container) where the reference can be imported:

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

It imports the UNMODIFIED reference package (``/root/reference/pkg/src/pathfair``)
and records, for seeded inputs built with the reference's own generators:

* incidence index arrays (model.py:206-271),
* per-kernel outputs on random states (kernels.py:206-296; tests/helpers.py:65-89),
* full solve trajectories (controller.py:197-284): per-iteration (alpha, beta, s, r)
  and state digests at chosen iterations,
* projection outputs (projection.py:51-107),
* sum-equation roots (kernels.py:134-173, 198-203),
* generator outputs (harness.py:138-239).

Arrays are stored verbatim when small, else as SHA-256 digests of their bytes
(after ``+ 0.0`` so that -0.0 and +0.0 hash alike).  Nothing here is read by the
product; tests compare the oracle (and, on the GPU, the CUDA path) against it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

from pathfair import controller, harness, kernels, model, projection  # noqa: E402
from pathfair.kernels import SolverState  # noqa: E402
import helpers  # noqa: E402  (reference tests/helpers.py)

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import states  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        a = a + 0.0
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]


def flat_inputs(inst0_topology, commodities, path_set):
    """Flatten a (topology, commodities, PathSet) triple to CSR arrays."""
    cpp = np.zeros(len(commodities) + 1, np.int64)
    pep = [0]
    pe = []
    for c, paths in enumerate(path_set.paths):
        cpp[c + 1] = cpp[c] + len(paths)
        for p in paths:
            pe.extend(p)
            pep.append(len(pe))
    return dict(capacity=inst0_topology.capacity.copy(),
                demand0=np.array([c.demand for c in commodities], np.float64),
                com_path_ptr0=cpp, path_edge_ptr0=np.array(pep, np.int64),
                path_edges0=np.array(pe, np.int64))


INCIDENCE = ("kept_rows", "demand", "com_path_ptr", "path_com", "hops", "pair_ptr", "pair_edge",
             "pair_path", "edge_path_count", "edge_pair_ptr", "edge_pairs")
STATE = ("x", "y", "dual_demand", "dual_capacity", "dual_consensus", "dual_nonneg",
         "slack_demand", "slack_capacity")


def small_instances():
    """The reference test-suite builders (tests/helpers.py:25-62, test_controller.py:19-27)."""
    out = {
        "single_bottleneck": (helpers.single_bottleneck, {}),
        "shared_edge2": (helpers.shared_edge, dict(n=2)),
        "shared_edge3": (helpers.shared_edge, dict(n=3)),
        "chain": (helpers.chain, {}),
        "diamond": (helpers.diamond, {}),
    }
    return out


def instance_from_builder(fn, kw):
    inst = fn(**kw)
    return inst


def flat_from_instance(inst):
    """Recover flat pre-drop inputs from a built Instance (small builders keep every commodity)."""
    paths = [[tuple(int(e) for e in inst.path_edges(p)) for p in inst.commodity_paths(c)]
             for c in range(inst.num_commodities)]
    return flat_inputs(inst.topology, inst.commodities, model.PathSet.from_lists(paths))


def gen_instance(n, k, vol_frac, seed=None):
    topo = harness.random_topology(n, seed=n if seed is None else seed)
    V = vol_frac * float(topo.capacity.sum())
    coms = harness.gravity_demands(topo, V)
    ps = harness.k_shortest_paths(topo, coms, k)
    return topo, coms, ps, model.build_instance(topo, coms, ps)


def kernel_cases(tag, inst, seed, arrays, digests, verbatim):
    """Per-kernel outputs on seeded random states (tests/golden/states.py, mirroring
    tests/helpers.py:65-89).  Outputs are stored verbatim for small instances and
    for alpha >= 2 (tolerance-pinned), else as digests."""
    cases = states.kernel_case_states(inst.num_commodities, inst.num_paths, inst.num_edges,
                                      inst.num_pairs, seed)
    for i, (arrs, beta, alpha) in enumerate(cases):
        st = SolverState(**{k: v.copy() for k, v in arrs.items()}, beta=beta, alpha=alpha, iteration=0)
        key = f"{tag}/k{i}"
        outs = {}
        dd, dc, dcon, dn = kernels.update_duals(st, inst)
        sd, sc = kernels.update_slacks(st, inst)
        outs.update(dd=dd, dc=dc, dcon=dcon, dn=dn, sd=sd, sc=sc)
        st.dual_demand, st.dual_capacity, st.dual_consensus, st.dual_nonneg = dd, dc, dcon, dn
        y = kernels.update_rate_suggestions(st, inst)
        outs["y"] = y
        st.y = y
        sums = kernels.solve_commodity_sums(st, inst, alpha)
        outs["sums"] = sums
        outs["x"] = kernels.update_rates(st, inst, sums, alpha)
        for nm, a in outs.items():
            if verbatim or (alpha >= 2 and nm in ("sums", "x")):
                arrays[f"{key}/out/{nm}"] = a
            digests[f"{key}/out/{nm}"] = digest(a)


def trajectory(tag, inst, cfg, snaps, store, arrays, meta, warm=None):
    """Replay controller.solve's loop (controller.py:216-273) and snapshot the state."""
    t0 = time.perf_counter()
    state = controller.initialize_state(inst, cfg, warm)
    just_incremented = False
    stopped = False
    ema_s = ema_r = -1.0
    cooldown = 0
    rows = []
    for it in range(1, cfg.max_iterations + 1):
        prev = __import__("copy").copy(state)
        dd, dc, dcon, dn = kernels.update_duals(state, inst)
        sd, sc = kernels.update_slacks(state, inst)
        state.dual_demand, state.dual_capacity = dd, dc
        state.dual_consensus, state.dual_nonneg = dcon, dn
        state.slack_demand, state.slack_capacity = sd, sc
        state.y = kernels.update_rate_suggestions(state, inst)
        sums = kernels.solve_commodity_sums(state, inst, state.alpha)
        state.x = kernels.update_rates(state, inst, sums, state.alpha)
        state.iteration = it
        res = controller.compute_residuals(prev, state)
        converged = controller.check_convergence(res, cfg.gamma)
        rows.append((it, state.alpha, state.beta, res.s, res.r))
        decision = controller.advance_alpha(state, cfg, converged, just_incremented)
        if cfg.adapt:
            if ema_s < 0.0:
                ema_s, ema_r = res.s, res.r
            else:
                ema_s += 0.1 * (res.s - ema_s)
                ema_r += 0.1 * (res.r - ema_r)
            if cooldown > 0:
                cooldown -= 1
            else:
                nb = controller.adapt_beta(state.beta, controller.Residuals(ema_s, ema_r), cfg)
                if nb != state.beta:
                    f = state.beta / nb
                    state.dual_demand = state.dual_demand * f
                    state.dual_capacity = state.dual_capacity * f
                    state.dual_consensus = state.dual_consensus * f
                    state.dual_nonneg = state.dual_nonneg * f
                    state.beta = nb
                    cooldown = 10
        just_incremented = False
        if it in snaps:
            for f in STATE:
                store[f"{tag}/it{it}/{f}"] = digest(getattr(state, f))
            store[f"{tag}/it{it}/sums"] = digest(sums)
            store[f"{tag}/it{it}/beta"] = state.beta
            store[f"{tag}/it{it}/alpha"] = state.alpha
            if state.alpha >= 2:  # numpy SIMD power in update_rates: tolerance-pinned
                arrays[f"{tag}/it{it}/x"] = state.x.copy()
        if decision == "stop":
            stopped = True
            break
        if decision == "increment":
            state.alpha += 1
            just_incremented = True
    rates = projection.project(inst, state.x, state.alpha)
    # cross-check our replay against the reference's own solve()
    ref = controller.solve(inst, cfg, warm)
    assert ref.iterations == state.iteration and np.array_equal(ref.rates, rates), tag
    arr = np.array(rows, dtype=np.float64)
    arrays[f"{tag}/trace"] = arr
    store[f"{tag}/raw_x"] = digest(state.x)
    if state.alpha >= 2:
        arrays[f"{tag}/raw_x"] = state.x.copy()
    store[f"{tag}/rates"] = digest(rates)
    arrays[f"{tag}/sums"] = model.commodity_sums(inst, rates)
    meta[tag] = dict(iterations=int(state.iteration), alpha=int(state.alpha), converged=bool(stopped),
                     seconds=time.perf_counter() - t0)
    return rates, state


def main():
    t_all = time.perf_counter()
    arrays = {}   # verbatim arrays -> golden_arrays.npz
    digests = {}  # name -> str/float -> golden_digests.json
    meta = {}

    # ---------------- small builders: incidence + kernels + solves
    rng = np.random.default_rng(20260517)
    for name, (fn, kw) in small_instances().items():
        inst = fn(**kw)
        flat = flat_from_instance(inst)
        for k, v in flat.items():
            arrays[f"small/{name}/in/{k}"] = v
        for f in INCIDENCE:
            arrays[f"small/{name}/inc/{f}"] = np.asarray(getattr(inst, f))
        kernel_cases(f"small/{name}", inst, 100 + len(name), arrays, digests, verbatim=True)
        for tgt in (0, 1, 2, None):
            cfg = controller.SolverConfig(alpha_target=tgt)
            res = controller.solve(inst, cfg)
            key = f"small/{name}/solve_a{tgt}"
            arrays[f"{key}/rates"] = res.rates
            arrays[f"{key}/sums"] = res.sums
            meta[key] = dict(iterations=res.iterations, alpha=res.alpha, converged=res.converged)
        res = controller.solve(inst, controller.SolverConfig(max_iterations=7, trace=True))
        arrays[f"small/{name}/trace7"] = np.array(
            [(t.iteration, t.alpha, t.beta, t.s, t.r, t.objective, t.pct_violated,
              t.mean_relative_violation) for t in res.trace])
        arrays[f"small/{name}/trace7_rates"] = res.rates

    # warm-start case (test_controller.py:178-184)
    inst = helpers.chain()
    cold = controller.solve(inst, controller.SolverConfig(alpha_target=1))
    warm = controller.solve(inst, controller.SolverConfig(alpha_target=1), warm_start=cold.rates)
    arrays["small/chain/warm/start"] = cold.rates
    arrays["small/chain/warm/rates"] = warm.rates
    meta["small/chain/warm"] = dict(iterations=warm.iterations, alpha=warm.alpha, converged=warm.converged)

    # ---------------- roots (kernels.py:134-173)
    rng = np.random.default_rng(3)
    n = 1000
    w = rng.uniform(0.05, 10, n)
    beta = 10 ** rng.uniform(-3, 3, n)
    q = rng.uniform(-1e3, 1e3, n)
    al = rng.choice([0, 1, 2, 3, 8], n)
    roots = np.array([kernels.solve_sum_equation(w[i], beta[i], q[i], int(al[i])) for i in range(n)])
    arrays["roots/w"], arrays["roots/beta"], arrays["roots/q"], arrays["roots/alpha"] = w, beta, q, al
    arrays["roots/out"] = roots

    # ---------------- cfg1: GEANT-sized (configs[0]) with the reference's generators
    for vol in (0.3, 1.5):
        tag = f"cfg1_v{vol}"
        topo, coms, ps, inst = gen_instance(40, 4, vol)
        flat = flat_inputs(topo, coms, ps)
        for k, v in flat.items():
            arrays[f"{tag}/in/{k}"] = v
        for f in INCIDENCE:
            dt = np.float64 if f == "demand" else np.int64
            digests[f"{tag}/inc/{f}"] = digest(np.asarray(getattr(inst, f), dt))
        if vol == 0.3:
            kernel_cases(tag, inst, 5, arrays, digests, verbatim=False)
            snaps = {1, 2, 3, 5, 10, 50, 200, 500, 826, 866, 978}
            rates, _ = trajectory(tag, inst, controller.SolverConfig(), snaps, digests, arrays, meta)
            arrays[f"{tag}/final_sums"] = model.commodity_sums(inst, rates)
            # projection of raw iterates (projection.py:51-107)
            for kk, its in enumerate((25, 120)):
                # raw (unprojected) iterate after `its` loop iterations
                loop_cfg = controller.SolverConfig(max_iterations=its)
                d = {}
                _, st = trajectory(f"{tag}/proj{kk}", inst, loop_cfg, set(), d, {}, {})
                st_x = st.x
                arrays[f"{tag}/proj{kk}/raw_x"] = st_x
                for a in (0, 1, 3):
                    digests[f"{tag}/proj{kk}/a{a}"] = digest(projection.project(inst, st_x, a))
                    arrays[f"{tag}/proj{kk}/a{a}_sums"] = model.commodity_sums(
                        inst, projection.project(inst, st_x, a))
            # link failure + warm start (config 4 analogue at cfg1 scale)
            rng = np.random.default_rng(1)
            cut = rng.choice(inst.num_edges, int(round(0.05 * inst.num_edges)), replace=False)
            cap = inst.capacity.copy()
            cap[cut] = 0.0
            arrays[f"{tag}/cut_edges"] = np.sort(cut)
            arrays[f"{tag}/warm_rates"] = rates
            inst_cut = model.with_conditions(inst, capacity=cap)
            # alpha_target=1 keeps the replay bit-exact (alpha >= 2 goes through numpy's SIMD pow)
            cfgw = controller.SolverConfig(alpha_target=1, max_iterations=400)
            trajectory(f"{tag}/warm_cut", inst_cut, cfgw, {1, 10, 100, 400}, digests, arrays, meta, warm=rates)
        else:
            snaps = {1, 2, 3, 5, 10, 100, 1000, 3000, 5000}
            trajectory(tag, inst, controller.SolverConfig(), snaps, digests, arrays, meta)

    # ---------------- generators (harness.py:179-239) and KSP (harness.py:138-176)
    for nn in (40, 500):
        topo = harness.random_topology(nn, seed=nn)
        arrays[f"gen/n{nn}/edge_src"] = topo.edge_src
        arrays[f"gen/n{nn}/edge_dst"] = topo.edge_dst
        arrays[f"gen/n{nn}/capacity"] = topo.capacity
        arrays[f"gen/n{nn}/weight"] = topo.weight
        arrays[f"gen/n{nn}/nodes"] = np.array(topo.nodes)
        coms = harness.gravity_demands(topo, 1.5 * float(topo.capacity.sum()))
        d = np.array([c.demand for c in coms])
        digests[f"gen/n{nn}/gravity"] = digest(d)
        arrays[f"gen/n{nn}/gravity_head"] = d[:64]
        if nn == 500:
            srng = np.random.default_rng(7)
            pick = np.sort(srng.choice(len(coms), 300, replace=False))
            sub = [coms[i] for i in pick]
            for k in (1, 8):
                ps = harness.k_shortest_paths(topo, sub, k)
                fl = flat_inputs(topo, sub, ps)
                arrays[f"gen/n{nn}/ksp{k}/pick"] = pick
                arrays[f"gen/n{nn}/ksp{k}/com_path_ptr"] = fl["com_path_ptr0"]
                arrays[f"gen/n{nn}/ksp{k}/path_edge_ptr"] = fl["path_edge_ptr0"]
                arrays[f"gen/n{nn}/ksp{k}/path_edges"] = fl["path_edges0"]
        # a topology with a failed link (KSP skips zero-capacity edges, harness.py:128)
    topo = harness.random_topology(40, seed=40)
    rows = []
    for e in range(topo.num_edges):
        s, t = topo.edge_names(e)
        rows.append((s, t, 0.0 if e in (3, 17, 40) else float(topo.capacity[e]), float(topo.weight[e])))
    topo_cut = model.build_topology(rows)
    coms = harness.gravity_demands(topo, 1.0)
    ps = harness.k_shortest_paths(topo_cut, coms, 4)
    fl = flat_inputs(topo_cut, coms, ps)
    arrays["gen/n40cut/ksp4/com_path_ptr"] = fl["com_path_ptr0"]
    arrays["gen/n40cut/ksp4/path_edge_ptr"] = fl["path_edge_ptr0"]
    arrays["gen/n40cut/ksp4/path_edges"] = fl["path_edges0"]
    arrays["gen/n40cut/capacity"] = topo_cut.capacity
    ps1 = harness.k_shortest_paths(topo, coms, 1)
    fl = flat_inputs(topo, coms, ps1)
    arrays["gen/n40/ksp1/path_edges"] = fl["path_edges0"]
    arrays["gen/n40/ksp1/path_edge_ptr"] = fl["path_edge_ptr0"]

    np.savez_compressed(os.path.join(OUT, "golden_arrays.npz"), **arrays)
    with open(os.path.join(OUT, "golden_digests.json"), "w") as fh:
        json.dump(dict(digests=digests, meta=meta,
                       versions=dict(numpy=np.__version__,
                                     numba=__import__("numba").__version__,
                                     networkx=__import__("networkx").__version__,
                                     python=sys.version.split()[0])), fh, indent=1, sort_keys=True)
    print(f"wrote {len(arrays)} arrays, {len(digests)} digests in {time.perf_counter() - t_all:.1f}s")


if __name__ == "__main__":
    main()
