"""Multi-GPU sharding: host-side logic on CPU (gloo, world_size 2) and the
NCCL-coupled solver at world_size 1 on a GPU.

The sharded data path is exact by construction: each rank's incidence store is
the reference's build_instance over its commodity range, and the union of the
shards is the single-instance index space (checked here with the oracle's CPU
build).  Per iteration the ranks exchange exactly the per-edge sums and the
residual norms (one allreduce)."""

import os
import socket

import numpy as np
import pytest

import golden_io as G
from oracle import oracle as O
from paper_2605_01748_b200 import distributed as D
from paper_2605_01748_b200.topology import CommodityTable, FlatPathSet


def _cfg1():
    f = G.flat_inputs("cfg1_v0.3")
    n = f["demand0"].shape[0]
    tab = CommodityTable(tuple(f"v{i}" for i in range(2 * n)), np.arange(0, 2 * n, 2), np.arange(1, 2 * n, 2),
                         f["demand0"])
    flat = FlatPathSet(f["com_path_ptr0"], f["path_edge_ptr0"], f["path_edges0"])
    return f, tab, flat


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_partition_balances_pairs(world):
    f, tab, flat = _cfg1()
    pc = D.pair_counts(tab, flat)
    ranges = D.partition(pc, world)
    assert ranges[0][0] == 0 and ranges[-1][1] == len(tab)
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    loads = [int(pc[a:b].sum()) for a, b in ranges]
    assert sum(loads) == int(pc.sum())
    assert max(loads) - min(loads) <= 2 * int(pc.max()) + 1


@pytest.mark.parametrize("world", [2, 3])
def test_shard_union_is_the_single_instance(world):
    f, tab, flat = _cfg1()
    full = O.build_instance(f["capacity"], f["demand0"], f["com_path_ptr0"], f["path_edge_ptr0"], f["path_edges0"])
    ranges = D.partition(D.pair_counts(tab, flat), world)
    cat = {k: [] for k in ("pair_edge", "hops", "demand")}
    epc = np.zeros(full.num_edges, np.int64)
    for lo, hi in ranges:
        st, sf = D.shard_inputs(tab, flat, lo, hi)
        sh = O.build_instance(f["capacity"], st.demand, sf.com_path_ptr, sf.path_edge_ptr, sf.path_edges)
        for k in cat:
            cat[k].append(getattr(sh, k))
        epc += sh.edge_path_count
    for k in cat:
        assert np.array_equal(np.concatenate(cat[k]), getattr(full, k)), k
    # global paths-per-edge (the allreduced divisor n_e + 1 of kernels.py:94)
    assert np.array_equal(epc, full.edge_path_count)
    pr = D.kept_path_ranges(tab, flat, ranges)
    assert pr[0][0] == 0 and pr[-1][1] == full.num_paths


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import ctypes as C

    import torch.distributed as dist

    from paper_2605_01748_b200._lib import lib
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    f, tab, flat = _cfg1()
    ranges = D.partition(D.pair_counts(tab, flat), world)
    lo, hi = ranges[rank]
    st, sf = D.shard_inputs(tab, flat, lo, hi)
    # NCCL unique-id exchange as Comm() does it
    buf = C.create_string_buffer(128)
    if rank == 0:
        assert lib().pf_comm_unique_id(buf) == 0
    obj = [bytes(buf.raw) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    got = [None] * world if rank == 0 else None
    dist.gather_object((obj[0], int(sf.path_edge_ptr[-1])), got, dst=0)
    if rank == 0:
        ids = {g[0] for g in got}
        total = sum(g[1] for g in got)
        q.put((len(ids), total, int(flat.path_edge_ptr[-1])))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_id_exchange_and_shards():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    n_ids, total, want = q.get(timeout=10)
    assert n_ids == 1 and total == want


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["ipc", "nccl"])
def test_world1_matches_single_gpu(transport):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist

    import paper_2605_01748_b200 as pf
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        f, tab, flat = _cfg1()
        topo = pf.random_topology(40, seed=40)
        tab = pf.gravity_table(topo, 0.3 * float(topo.capacity.sum()))
        cfg = pf.SolverConfig(mode="fast", max_iterations=5000)
        sh = D.ShardedSolver(topo, tab, flat, cfg, 0, 1, 0, transport=transport).init()
        sh.run(5000)
        r = sh.result()
        x = sh.gather_x()
        inst = pf.build_instance_flat(topo, tab, flat, device=0)
        single = pf.solve(inst, cfg)
        assert bool(r.converged) and abs(int(r.iterations) - single.iterations) <= 20
        rates = pf.project(inst, x, int(r.alpha))
        sums = pf.commodity_sums(inst, rates)
        np.testing.assert_allclose(np.sort(sums), np.sort(single.sums), rtol=1e-4,
                                   atol=1e-4 * float(single.sums.max()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_world1_graph_loop_matches_host_loop(monkeypatch):
    """The sharded iteration loop runs as one CUDA graph (WHILE over the body,
    IF for the rollback branch, conditions set on the device); it must take the
    same branches and produce bitwise the same iterates as the host-driven loop
    over 300 iterations that include beta changes (rollback passes)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist

    import paper_2605_01748_b200 as pf
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        topo = pf.random_topology(40, seed=40)
        tab = pf.gravity_table(topo, 0.3 * float(topo.capacity.sum()))
        flat = pf.k_shortest_paths(topo, tab, 4)
        cfg = pf.SolverConfig(mode="fast", max_iterations=5000, gamma=1e-12)
        runs = {}
        for mode in ("graph", "host"):
            if mode == "host":
                monkeypatch.setenv("PF_DIST_NO_GRAPH", "1")
            sh = D.ShardedSolver(topo, tab, flat, cfg, 0, 1, 0, transport="nccl").init()
            sh.run(120)
            sh.run(180)  # two runs: the graph is relaunched with a new target
            r = sh.result()
            runs[mode] = (sh.local_x(), int(r.iterations), float(r.beta), int(sh.solver.kernel_stats()["launches"]))
        (xg, ig, bg, lg), (xh, ih, bh, lh) = runs["graph"], runs["host"]
        assert ig == ih == 300 and bg == bh
        assert np.array_equal(xg, xh)
        assert lg < 20 < lh  # the graph replaced ~5 launches per iteration
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_ipc_world1_bitwise_equals_single_gpu():
    """The peer-memory transport: the fused kernel exchanges its rank totals
    through its own exchange buffer at world size 1 and must reproduce the
    single-GPU fused kernel bitwise, across launches and rollback iterations,
    with one kernel launch per run."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist

    import paper_2605_01748_b200 as pf
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        topo = pf.random_topology(40, seed=40)
        tab = pf.gravity_table(topo, 0.3 * float(topo.capacity.sum()))
        flat = pf.k_shortest_paths(topo, tab, 4)
        cfg = pf.SolverConfig(mode="fast", max_iterations=5000, gamma=1e-12)
        sh = D.ShardedSolver(topo, tab, flat, cfg, 0, 1, 0, transport="ipc").init()
        sh.run(150)
        sh.run(150)
        inst = pf.build_instance_flat(topo, tab, flat, device=0)
        single = pf.Solver(inst, cfg).init()
        single.run(300)
        r1, r2 = sh.result(), single.result()
        assert int(r1.iterations) == int(r2.iterations) == 300 and float(r1.beta) == float(r2.beta)
        assert np.array_equal(sh.local_x(), single.x())
        assert int(sh.solver.kernel_stats()["launches"]) == 2
    finally:
        dist.destroy_process_group()


def _ipc_rank_worker(rank, world, port, iters, q):
    import torch.distributed as dist

    import paper_2605_01748_b200 as pf
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        topo = pf.random_topology(24, seed=24)
        tab = pf.gravity_table(topo, 0.3 * float(topo.capacity.sum()))
        flat = pf.k_shortest_paths(topo, tab, 4)
        cfg = pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 6)
        sh = D.ShardedSolver(topo, tab, flat, cfg, rank, world, 0, transport="ipc").init()
        sh.run(iters)
        r = sh.result()
        x = sh.gather_x()
        single = None
        if rank == 0:
            inst = pf.build_instance_flat(topo, tab, flat, device=0)
            s1 = pf.Solver(inst, cfg).init()
            s1.run(iters)
            single = s1.x()
        q.put((rank, int(r.iterations), float(r.beta), int(r.alpha), x, single))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 4])
def test_ipc_multirank_on_one_gpu(world):
    """Real multi-rank exchange of the peer-memory transport: `world` processes
    on the one B200 (the driver time-slices their cooperative kernels), shards
    of a 24-node instance.  Every rank must end with the identical controller
    state and the gathered rates must equal the single-GPU solve at the same
    iteration count up to the reassociated edge sums."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ipc_rank_worker, args=(r, world, port, 40, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in ps)
    states = [t[1:4] for t in res]
    assert all(s == states[0] for s in states) and states[0][0] == 40
    xg, xs = res[0][4], res[0][5]
    assert xg.shape == xs.shape
    # shards reassociate the per-edge sums (their tiles differ from the single
    # instance's), and after 40 iterations the frozen-activity tests amplify the
    # ulp differences: the north_star tolerance (1e-4 relative) bounds them
    assert float(np.max(np.abs(xg - xs))) <= 1e-4 * float(np.max(np.abs(xs)))


def _ipc_second_solver_worker(rank, world, port, iters, q):
    import torch.distributed as dist

    import paper_2605_01748_b200 as pf
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg = pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 6)
        t0 = pf.random_topology(24, seed=24)
        b0 = pf.gravity_table(t0, 0.3 * float(t0.capacity.sum()))
        first = D.ShardedSolver(t0, b0, pf.k_shortest_paths(t0, b0, 4), cfg, rank, world, 0, transport="ipc").init()
        first.run(30)  # kept alive: its exchange buffers stay mapped in both processes
        topo = pf.random_topology(40, seed=40)
        tab = pf.gravity_table(topo, 0.3 * float(topo.capacity.sum()))
        flat = pf.k_shortest_paths(topo, tab, 4)
        sh = D.ShardedSolver(topo, tab, flat, cfg, rank, world, 0, transport="ipc").init()
        sh.run(iters)
        r = sh.result()
        x = sh.gather_x()
        single = None
        if rank == 0:
            inst = pf.build_instance_flat(topo, tab, flat, device=0)
            s1 = pf.Solver(inst, cfg).init()
            s1.run(iters)
            single = s1.x()
        q.put((rank, int(r.iterations), float(r.beta), int(r.alpha), x, single))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_ipc_second_solver_in_process():
    """A second peer-memory solver in the same processes (the bench's flow: the
    timed instance, then the time-to-1% instance) must exchange through its own
    buffers: each exchange buffer is its own 2 MB allocation (the IPC granularity;
    a small one sharing a page with other allocations corrupted the exchange
    after a few hundred iterations).  Ranks agree, and the gathered rates follow
    the single-GPU trajectory."""
    import os

    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if os.environ.get("PF_TEST_TIMESLICED_LONG") == "0":
        pytest.skip("long time-sliced multi-process run disabled (PF_TEST_TIMESLICED_LONG=0)")
    # (this run used to drift from the single-GPU trajectory or stall: the CTAs'
    # controller copies could diverge on a race over the per-edge residuals,
    # fixed by double-buffering them by iteration parity)
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world, iters = 2, 800
    ps = [ctx.Process(target=_ipc_second_solver_worker, args=(r, world, port, iters, q)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda t: t[0])
    finally:
        for p in ps:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in ps)
    states = [t[1:4] for t in res]
    assert all(s == states[0] for s in states) and states[0][0] == iters
    xg, xs = res[0][4], res[0][5]
    assert float(np.max(np.abs(xg - xs))) <= 1e-3 * float(np.max(np.abs(xs)))


@pytest.mark.gpu
def test_ipc_failure_falls_back_to_nccl(monkeypatch):
    """When the peer-memory exchange cannot be set up on some rank, all ranks
    agree and continue over NCCL (default transport); an explicit transport="ipc"
    request raises instead."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist

    import paper_2605_01748_b200 as pf
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        topo = pf.random_topology(40, seed=40)
        tab = pf.gravity_table(topo, 0.3 * float(topo.capacity.sum()))
        flat = pf.k_shortest_paths(topo, tab, 4)
        cfg = pf.SolverConfig(mode="fast", gamma=1e-12, max_iterations=10 ** 6)
        monkeypatch.delenv("PF_DIST_TRANSPORT", raising=False)
        monkeypatch.setenv("PF_DIST_IPC_FAIL", "1")
        with pytest.warns(RuntimeWarning, match="peer-memory exchange unavailable"):
            fb = D.ShardedSolver(topo, tab, flat, cfg, 0, 1, 0)
        assert fb.transport == "nccl"
        with pytest.raises(RuntimeError, match="peer-memory exchange unavailable"):
            D.ShardedSolver(topo, tab, flat, cfg, 0, 1, 0, transport="ipc")
        monkeypatch.delenv("PF_DIST_IPC_FAIL")
        nc = D.ShardedSolver(topo, tab, flat, cfg, 0, 1, 0, transport="nccl")
        fb.init()
        nc.init()
        fb.run(50)
        nc.run(50)
        assert np.array_equal(fb.gather_x(), nc.gather_x())
    finally:
        dist.destroy_process_group()


def _agree_worker(rank, world, port, fail_rank, fail_at, q):
    """_connect_ipc with the native calls stubbed: `fail_rank` fails at
    `fail_at` ("create" / "connect"); every rank must return an error and none
    may block in a collective."""
    import types

    import torch.distributed as dist

    from paper_2605_01748_b200 import distributed as DD
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        class FakeLib:
            def pf_solver_xchg_create(self, h, r, w, buf):
                if rank == fail_rank and fail_at == "create":
                    return 1
                buf.raw = bytes([r + 1]) * 64
                return 0

            def pf_solver_xchg_connect(self, h, handles):
                return 1 if rank == fail_rank and fail_at == "connect" else 0

            def pf_solver_set_edge_counts(self, h, p):
                return 0

            def pf_last_error(self, buf, n):
                buf.value = b"stubbed failure"
                return 0

        DD.lib = lambda: FakeLib()
        import paper_2605_01748_b200._lib as L
        L.lib = lambda: FakeLib()
        stub = types.SimpleNamespace(solver=types.SimpleNamespace(_h=None), rank=rank, world=world,
                                     instance=types.SimpleNamespace(edge_path_count=np.ones(3)))
        err = DD.ShardedSolver._connect_ipc(stub, None)
        q.put((rank, None if err is None else str(err)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_at", ["create", "connect", None])
def test_ipc_setup_failure_on_one_rank_is_agreed(fail_at):
    """The peer-memory setup protocol (host logic, gloo world size 2 on CPU):
    a failure on one rank is seen by every rank (so all fall back together)
    and no rank blocks; without failures every rank connects."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_agree_worker, args=(r, 2, port, 1, fail_at, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in ps)
    if fail_at is None:
        assert res == {0: None, 1: None}
    else:
        assert res[0] is not None and res[1] is not None, res


def _shard_agree_worker(rank, world, port, bad_rank, why, q):
    """ShardedSolver._agree_shards with the instance stubbed: `bad_rank`'s shard
    is outside the fused layout (or empty); every rank must raise, none block."""
    import types

    import torch.distributed as dist

    from paper_2605_01748_b200 import distributed as DD
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        bad = rank == bad_rank
        inst = types.SimpleNamespace(
            num_paths=0 if (bad and why == "empty") else 10,
            fast_supported=lambda: (False, "commodity 3 has more than 32 paths") if (bad and why == "layout")
            else (True, ""))
        stub = types.SimpleNamespace(instance=inst, rank=rank, world=world)
        try:
            DD.ShardedSolver._agree_shards(stub, None)
            q.put((rank, None))
        except RuntimeError as exc:
            q.put((rank, str(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("why", ["layout", "empty", None])
def test_shard_capability_is_agreed_before_transport_setup(why):
    """a shard outside the fused layout limits, or an empty shard,
    must make every rank raise (gloo world size 2 on CPU) instead of one rank
    raising while the others wait in the exchange."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_shard_agree_worker, args=(r, 2, port, 1, why, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in ps)
    if why is None:
        assert res == {0: None, 1: None}
    else:
        assert res[0] is not None and res[1] is not None, res
        assert "ranks [1]" in res[0] and res[0] == res[1]
