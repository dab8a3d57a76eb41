"""Multi-GPU solves: commodities sharded across the GPUs of one box.

One process per GPU (torchrun).  Each rank owns a contiguous range of
commodities (split so every rank holds about the same number of demand-path
pairs), builds the incidence store of its shard on its own GPU, and runs the
fused solver on it.  Everything is shard-local except the per-edge sums
T_e = sum(x + dcon') and L_e = sum(y) and the residual norms (2E + 16 doubles
per iteration).  Two transports (csrc/fused.cu):

* "ipc" (default): the persistent fused kernel itself writes its rank-local
  totals into every rank's exchange buffer over NVLink peer memory (CUDA IPC)
  and meets the other ranks at a counter barrier; every rank sums the ranks'
  slots in rank order, so all ranks hold identical totals (deterministic, and
  at world size 1 bitwise equal to the single-GPU kernel);
* "nccl": split kernels around one ncclAllReduce per iteration, the loop run as
  one CUDA graph with device-side conditions.

Every rank then evaluates the same controller step, so all ranks take identical
branches; the dual-capacity / adjustment update per edge is replicated.
torch.distributed is plumbing only: it exchanges the IPC handles / NCCL unique
id, sums the paths-per-edge counts once, and gathers the final rates.
"""

from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

from . import _abi as A
from ._lib import check, lib
from .controller import Solver, SolverConfig
from .model import build_instance_flat
from .topology import CommodityTable, FlatPathSet


def partition(pairs_per_commodity, world: int):
    """Contiguous commodity ranges [lo, hi) with ~equal pair counts (deterministic)."""
    w = np.asarray(pairs_per_commodity, np.int64)
    n = w.shape[0]
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    cs = np.concatenate([[0], np.cumsum(w)])
    total = cs[-1]
    bounds = [0]
    for r in range(1, world):
        b = int(np.searchsorted(cs, total * r / world, side="left"))
        bounds.append(max(bounds[-1], min(b, n)))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def pair_counts(table: CommodityTable, flat: FlatPathSet) -> np.ndarray:
    """Pairs each commodity contributes after the reference's drop rule (model.py:226-229)."""
    cpp, pep = flat.com_path_ptr, flat.path_edge_ptr
    per = pep[cpp[1:]] - pep[cpp[:-1]]
    keep = (np.asarray(table.demand) > 0) & (np.diff(cpp) > 0)
    return np.where(keep, per, 0)


def shard_inputs(table: CommodityTable, flat: FlatPathSet, lo: int, hi: int):
    """Commodities [lo, hi) with their paths, re-based to a stand-alone flat path set."""
    cpp, pep, pe = flat.com_path_ptr, flat.path_edge_ptr, flat.path_edges
    p0, p1 = int(cpp[lo]), int(cpp[hi])
    t0, t1 = int(pep[p0]), int(pep[p1])
    sub = FlatPathSet(cpp[lo:hi + 1] - p0, pep[p0:p1 + 1] - t0, pe[t0:t1].copy())
    tab = CommodityTable(table.nodes, table.src[lo:hi], table.dst[lo:hi], table.demand[lo:hi])
    return tab, sub


def kept_path_ranges(table: CommodityTable, flat: FlatPathSet, ranges):
    """Per shard, the [start, stop) slice of the globally kept path index space."""
    cpp = flat.com_path_ptr
    keep = (np.asarray(table.demand) > 0) & (np.diff(cpp) > 0)
    kept_paths = np.where(keep, np.diff(cpp), 0)
    cs = np.concatenate([[0], np.cumsum(kept_paths)])
    return [(int(cs[lo]), int(cs[hi])) for lo, hi in ranges]


class Comm:
    """A pf_comm (NCCL communicator over the ranks of a torch.distributed group)."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch.distributed as dist
        buf = C.create_string_buffer(128)
        if rank == 0:
            check(lib().pf_comm_unique_id(buf))
        obj = [bytes(buf.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = C.create_string_buffer(obj[0], 128)
        h = C.c_void_p()
        check(lib().pf_comm_create(world, rank, uid, device, C.byref(h)))
        self._h = h.value
        self.rank, self.world, self.device = rank, world, device

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().pf_comm_destroy(self._h)
            except Exception:  # noqa: BLE001
                pass
            self._h = None


class ShardedSolver:
    """Fast-mode solver over this rank's commodity shard, coupled by NCCL."""

    def __init__(self, topology, table: CommodityTable, flat: FlatPathSet, config: SolverConfig | None = None,
                 rank: int = 0, world: int = 1, device: int = 0, group=None, transport: str | None = None):
        self.config = config if config is not None else SolverConfig(mode="fast")
        if self.config.mode != "fast":
            raise ValueError("sharded solves run in fast mode")
        self.rank, self.world, self.device = rank, world, device
        self.ranges = partition(pair_counts(table, flat), world)
        lo, hi = self.ranges[rank]
        sub_tab, sub_flat = shard_inputs(table, flat, lo, hi)
        self.instance = build_instance_flat(topology, sub_tab, sub_flat, device=device)
        self.path_ranges = kept_path_ranges(table, flat, self.ranges)
        if world > 1:
            self._agree_shards(group)
        self.solver = Solver(self.instance, self.config)
        # transport: "ipc" = the fused kernel exchanges edge totals over NVLink peer
        # memory (CUDA IPC buffers, no host round trip); "nccl" = split kernels
        # around one ncclAllReduce per iteration, run as a CUDA graph
        requested = transport or os.environ.get("PF_DIST_TRANSPORT")
        self.transport = requested or "ipc"
        self.comm = None
        if self.transport == "ipc":
            err = self._connect_ipc(group)
            if err is not None:
                if requested == "ipc":
                    raise RuntimeError(f"peer-memory exchange unavailable: {err}")
                import warnings
                warnings.warn(f"peer-memory exchange unavailable ({err}); using NCCL", RuntimeWarning)
                self.solver = Solver(self.instance, self.config)  # no half-connected exchange state
                self.transport = "nccl"
        if self.transport == "nccl":
            self.comm = Comm(rank, world, device, group)
            n_kept = int(np.sum((np.asarray(table.demand) > 0) & (np.diff(flat.com_path_ptr) > 0)))
            check(lib().pf_solver_attach_comm(self.solver._h, self.comm.handle, n_kept))
            # the native solver (and the CUDA graph capturing its allreduce) must be
            # destroyed before the communicator: the solver keeps it alive
            self.solver._comm_keepalive = self.comm
        elif self.transport != "ipc":
            raise ValueError(f"unknown transport {self.transport!r}")

    def _agree_shards(self, group=None):
        """Every rank's shard must run the fused kernel (fast mode's exchange is
        inside it) and hold at least one path (an empty shard never enters the
        exchange): the ranks agree before any transport is set up, and all of
        them raise together instead of some blocking in a collective."""
        import torch
        import torch.distributed as dist
        ok, why = self.instance.fast_supported()
        if self.instance.num_paths == 0:
            ok, why = False, "empty shard (more ranks than commodities with paths)"
        flags = torch.tensor([1.0 if ok else 0.0], dtype=torch.float64)
        dist.all_reduce(flags, op=dist.ReduceOp.MIN, group=group)
        if flags.item() < 1.0:
            whys = [None] * self.world
            dist.all_gather_object(whys, None if ok else why, group=group)
            bad = {r: w for r, w in enumerate(whys) if w is not None}
            raise RuntimeError(f"sharded fast-mode solve impossible on ranks {sorted(bad)}: {bad}")

    def _connect_ipc(self, group=None):
        """Exchange CUDA-IPC handles and open every peer's buffer.  Every rank
        takes part in every collective whatever happens locally, and the ranks
        agree on the outcome: returns None, or the (first) error on any rank."""
        import torch
        import torch.distributed as dist
        err = None
        h = C.create_string_buffer(64)
        try:
            if os.environ.get("PF_DIST_IPC_FAIL") == "1":  # test hook: exercise the fallback
                raise RuntimeError("PF_DIST_IPC_FAIL=1")
            check(lib().pf_solver_xchg_create(self.solver._h, self.rank, self.world, h))
            mine = bytes(h.raw)
        except Exception as exc:  # noqa: BLE001
            err, mine = exc, b""
        parts = [None] * self.world
        dist.all_gather_object(parts, mine, group=group)
        if err is None and all(len(p) == 64 for p in parts):
            try:
                allh = C.create_string_buffer(b"".join(parts), 64 * self.world)
                check(lib().pf_solver_xchg_connect(self.solver._h, allh))
            except Exception as exc:  # noqa: BLE001
                err = exc
        elif err is None:
            err = RuntimeError("another rank could not create its exchange buffer")
        bad = torch.tensor([0.0 if err is None else 1.0], dtype=torch.float64)
        dist.all_reduce(bad, group=group)
        if bad.item() > 0:
            return err if err is not None else RuntimeError("another rank could not open the exchange")
        # n_e of kernels.py:94 counts the paths of every shard
        ne = torch.tensor(np.asarray(self.instance.edge_path_count, np.float64))
        dist.all_reduce(ne, group=group)
        ne = np.ascontiguousarray(ne.numpy(), np.float64)
        check(lib().pf_solver_set_edge_counts(self.solver._h, ne.ctypes.data_as(C.POINTER(C.c_double))))
        return None

    def init(self, warm_start=None):
        if warm_start is not None:
            a, b = self.path_ranges[self.rank]
            warm_start = np.asarray(warm_start, np.float64)[a:b]
        self.solver.init(warm_start)
        return self

    def run(self, steps: int) -> int:
        return self.solver.run(steps)

    def time_loop(self, iterations: int):
        return self.solver.time_loop(iterations)

    def result(self):
        return self.solver.result()

    def local_x(self) -> np.ndarray:
        return self.solver.x()

    def gather_x(self, group=None):
        """Full rate vector (kept-path order) on rank 0, None elsewhere: one
        tensor gather of the shards (sizes from the partition, no pickling)."""
        import torch
        import torch.distributed as dist
        sizes = [b - a for a, b in self.path_ranges]
        n = max(sizes) if sizes else 0
        mine = np.zeros(n, np.float64)
        x = self.local_x()
        mine[:x.size] = x
        t = torch.from_numpy(mine)
        parts = [torch.empty(n, dtype=torch.float64) for _ in range(self.world)] if self.rank == 0 else None
        dist.gather(t, parts, dst=0, group=group)
        if self.rank != 0:
            return None
        return np.concatenate([parts[r].numpy()[:sizes[r]] for r in range(self.world)])


def consistency_check(sh, topo, tab, flat, world, rank):
    """After a sharded run: every rank must hold the identical controller state
    (iteration, alpha, beta, residuals -- they all evaluate the same controller
    on the same exchanged totals), and the gathered rates, projected on rank 0,
    must be feasible.  Raises on a mismatch (a transport bug must not pass as a
    number)."""
    import torch.distributed as dist
    r = sh.result()
    mine = (int(r.iterations), int(r.alpha), float(r.beta), int(r.converged))
    allst = [None] * world
    dist.all_gather_object(allst, mine)
    if any(a != allst[0] for a in allst):
        raise RuntimeError(f"ranks diverged: {allst}")
    x = sh.gather_x()
    out = {"ranks_agree": True, "state": list(allst[0])}
    if rank == 0:
        from .model import build_instance_flat as _bif
        from .projection import project
        from .model import validate_allocation
        full = _bif(topo, tab, flat, device=sh.device)
        rates = project(full, x, int(r.alpha))
        out["projected_feasible"] = bool(validate_allocation(full, rates).feasible)
        if not out["projected_feasible"]:
            raise RuntimeError("projected sharded rates are infeasible")
    return out


def _sharded_time_to_quality(args, bench, rank, world, local, name="target_k4_v0.3"):
    """Time to within 1% at N GPUs on the north-star instance (BASELINE
    north_star): the sharded solver runs k* iterations from cold
    (k* = the reference trajectory's own, from the committed oracle fixture),
    timed on the device as the max over ranks, plus the gather and one GPU
    projection on rank 0; the projected sums are then scored against the
    reference fixed point, so the line shows the quality actually reached."""
    import time as _time

    import torch
    import torch.distributed as dist

    fp = bench.oracle_fixed_point(name)
    if fp is None or getattr(args, "no_ttq", False):
        return None
    meta, opt = fp
    kstar = int(meta["k_star"])
    if rank == 0:
        bench.build_inputs(name)
    dist.barrier()
    topo, tab, flat = bench.build_inputs(name)
    sh = ShardedSolver(topo, tab, flat, SolverConfig(mode="fast", max_iterations=5000), rank, world, local)
    sh.init()
    dist.barrier()
    ms, _ = sh.time_loop(kstar)
    t = torch.tensor([ms], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_loop = float(t.item())
    r = sh.result()
    alpha = int(r.alpha)
    if int(r.iterations) != kstar or int(r.status) != 0:
        raise RuntimeError(f"sharded time-to-quality run stopped at iteration {int(r.iterations)} of {kstar} "
                           f"(status {int(r.status)}, converged {int(r.converged)})")
    t0 = _time.perf_counter()
    xg = sh.gather_x()
    out = None
    if rank == 0:
        from .metrics import default_theta, optimality_from_sums
        from .model import build_instance_flat, commodity_sums
        from .projection import project
        full = build_instance_flat(topo, tab, flat, device=local)
        t1 = _time.perf_counter()
        rates = project(full, xg, alpha)
        torch.cuda.synchronize()
        proj_ms = 1e3 * (_time.perf_counter() - t1)
        gather_ms = 1e3 * (t1 - t0)
        q = optimality_from_sums(commodity_sums(full, rates), opt, default_theta(full))
        # the same k* iterations on rank 0's GPU alone: the sharded trajectory is a
        # reassociation of it (edge totals summed per rank), so the two agree closely
        one = Solver(full, SolverConfig(mode="fast", max_iterations=5000)).init()
        one.run(kstar)
        x1 = one.x()
        q1 = optimality_from_sums(commodity_sums(full, project(full, x1, int(one.result().alpha))), opt,
                                  default_theta(full))
        dx = float(np.max(np.abs(xg - x1)) / max(float(np.max(np.abs(x1))), 1e-300))
        out = {"config": name, "k_star_reference": kstar, "gpu_loop_ms_max_over_ranks": ms_loop,
               "gather_ms": gather_ms, "projection_ms": proj_ms, "gpu_ms": ms_loop + gather_ms + proj_ms,
               "optimality_at_k_star_vs_reference_fixed_point": q, "n_gpus": world,
               "single_gpu_check": {"optimality_at_k_star": q1, "max_rel_rate_diff": dx,
                                    "consistent": bool(dx < 1e-3 and abs(q - q1) < 1e-4)},
               "how": "k* sharded iterations from cold (one launch per rank, max over ranks) + gather_x + "
                      "project on rank 0 (host wall); quality scored against the oracle's fixed point"}
    dist.barrier()
    return out


def bench_main(args, bench):
    """bench.py --gpus N under torchrun: one instance (config 3 by default)
    sharded over N GPUs (fixed total work: strong scaling)."""
    import json

    import torch
    import torch.distributed as dist

    rank, world, local = bench.dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    if rank == 0:  # one generator run; the other ranks read its cache
        bench.build_inputs(args.config)
    dist.barrier()
    topo, tab, flat = bench.build_inputs(args.config)
    cfg = SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 9)
    sh = ShardedSolver(topo, tab, flat, cfg, rank, world, local)
    sh.init()
    sh.time_loop(max(args.warmup, 3))
    torch.cuda.synchronize()
    dist.barrier()
    clocks = bench.ClockSampler(local).start()
    ms, _ = sh.time_loop(args.steps)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([ms], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    st = sh.solver.kernel_stats()
    # compulsory HBM bytes per iteration summed over the ranks' layouts
    # (kernel_stats; ncu cannot profile a multi-rank run -- at N = 1 ncu measures
    # ~0.99x of the layout's compulsory bytes, profiles/r02*_fused_*.json)
    tb = torch.tensor([float(st["bytes_per_iter"])], dtype=torch.float64)
    dist.all_reduce(tb)
    NP = np.array([sh.instance.num_pairs], np.int64)
    tn = torch.tensor(NP)
    dist.all_reduce(tn)
    check_ = consistency_check(sh, topo, tab, flat, world, rank)
    # e2e through the sharded public API with host buffers: warm start (host ->
    # each rank's shard), K iterations, rates gathered to rank 0, projection
    # and the projected rates back on the host; wall time, max over ranks
    import time as _time
    warm = sh.gather_x()
    warm_all = [warm] if rank == 0 else [None]
    dist.broadcast_object_list(warm_all, src=0)
    warm = warm_all[0]
    dist.barrier()
    t0 = _time.perf_counter()
    sh.init(warm)
    sh.run(args.steps)
    xg = sh.gather_x()
    if rank == 0:
        from .model import build_instance_flat as _bif
        from .projection import project as _proj
        if not hasattr(bench_main, "_full"):
            bench_main._full = _bif(topo, tab, flat, device=local)
        _proj(bench_main._full, xg, int(sh.result().alpha))
    torch.cuda.synchronize()
    e2e_s = _time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    ttq = _sharded_time_to_quality(args, bench, rank, world, local)
    if rank == 0:
        C_, P_, E_ = len(tab), int(flat.com_path_ptr[-1]), topo.num_edges
        NPt = int(tn.item())
        b_iter = bench.algorithmic_bytes(C_, P_, NPt, E_)
        peak, kind = bench.measured_peaks()
        ach = b_iter * args.steps / (ms_max / 1e3) / 1e9
        line = {"metric": bench.METRIC, "value": args.steps / (ms_max / 1e3), "unit": "iterations/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": bench.workload_config(args.config, C_, P_, NPt, E_, world),
                "transport": {"kind": sh.transport,
                              "collective": ("per-iteration exchange of 2E+16 fp64 rank totals inside the fused "
                                             "kernel over NVLink peer memory (CUDA IPC), counter barrier, "
                                             "rank-order sums" if sh.transport == "ipc" else
                                             "one ncclAllReduce of 2E+16 fp64 per iteration (CUDA-graph loop)"),
                              "sharding": "contiguous commodity ranges, equal pair counts",
                              **({"shared_gpus": torch.cuda.device_count()}
                                 if os.environ.get("PF_BENCH_SHARE_GPU") == "1" else {})},
                "roofline": {"bound": "hbm", "achieved": ach, "peak": peak * world, "unit": "GB/s",
                             "frac": ach / (peak * world), "traffic": float(tb.item()),
                             "traffic_kind": "compulsory layout bytes per iteration, summed over ranks (not ncu)",
                             "peak_kind": kind},
                "clocks": clk, "gpu_launches": int(st["launches"]), "max_over_ranks_ms": ms_max,
                "e2e": {"value": args.steps / e2e_s, "unit": "iterations/s",
                        "h2d_bytes_per_step": 8 * P_ / args.steps, "d2h_bytes_per_step": 16 * P_ / args.steps,
                        "call": "ShardedSolver: host warm start -> K iterations -> gather_x -> project (rank 0)"},
                "check": check_,
                "time_to_1pct": ttq}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0
