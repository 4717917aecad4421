"""Sharded streamed update (paper_2308_16395_b200/sharded.py).

CPU (gloo, world size 2): the per-slice exchange protocol of include/tsg.h
driven by `sharded.drive` over `TorchComm`, with a host stand-in engine whose
payload is the raw slab and whose finish is the CPU checker on the gathered
slice; the result must be bit-identical to the checker's unsharded run. Plus
the decomposition identity the device engine relies on: projecting modes
< s slab by slab and concatenating along s equals projecting the whole slice.

GPU: the device engine (libtsg.so) over `LoopbackGroup` (G virtual ranks on
one B200, exchange = device copy): every rank ends bitwise identical, and the
state matches the reference's golden fixtures within the parity tolerances;
and G = 1 through a real NCCL process group (the transport the multi-GPU
bench uses)."""
import json
import os
import socket

import numpy as np
import pytest

import cases
import parity as P

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ------------------------------------------------------------------- CPU
def test_shard_bounds_and_slabs():
    from paper_2308_16395_b200 import sharded as SH
    assert SH.shard_bounds(10, 3) == [0, 4, 7, 10]
    assert SH.shard_bounds(8, 8) == list(range(9))
    with pytest.raises(ValueError):
        SH.shard_bounds(3, 4)
    dims = (4, 5, 6)
    y = np.arange(np.prod(dims), dtype=np.float64)
    b = SH.shard_bounds(dims[-1], 4)
    parts = [SH.slab_of(y, dims, b, g) for g in range(4)]
    np.testing.assert_array_equal(np.concatenate(parts), y)
    t = y.reshape(dims[::-1]).transpose()  # t[i0, i1, i2]
    np.testing.assert_array_equal(parts[1].reshape(6 * 0 + b[2] - b[1], 5, 4).transpose(),
                                  t[:, :, b[1]:b[2]])


def test_slab_of_any_mode_and_default_mode():
    from paper_2308_16395_b200 import sharded as SH
    assert SH.default_shard_mode((200, 200, 200)) == 2       # ties: the last one
    assert SH.default_shard_mode((384, 384, 384, 16)) == 2   # C4: not the variable mode
    assert SH.default_shard_mode((12, 10, 9)) == 0
    dims = (4, 5, 6)
    y = np.arange(np.prod(dims), dtype=np.float64)
    t = y.reshape(dims[::-1]).transpose()  # t[i0, i1, i2]
    for mode in range(3):
        b = SH.shard_bounds(dims[mode], 2)
        for g in range(2):
            want = np.take(t, np.arange(b[g], b[g + 1]), axis=mode)
            got = SH.slab_of(y, dims, b, g, mode=mode)
            np.testing.assert_array_equal(got, want.transpose().ravel())  # colexicographic
            tt = SH.slab_of(torch.from_numpy(y), dims, b, g, mode=mode)
            np.testing.assert_array_equal(tt.numpy(), got)


def test_local_projection_then_gather_equals_full():
    """Modes < s are local to a slab of the last spatial mode: project each
    slab, concatenate along s == project the slice (streaming.cpp:126-133)."""
    g = np.random.default_rng(5)
    dims = (7, 6, 9)
    y = g.standard_normal(dims)
    us = [np.linalg.qr(g.standard_normal((n, r)))[0] for n, r in zip(dims[:2], (3, 2))]

    def proj(t):
        res = []
        for k, u in enumerate(us):
            p = np.moveaxis(np.tensordot(u.T, t, axes=([1], [k])), 0, k)
            res.append(np.linalg.norm(t - np.moveaxis(np.tensordot(u, p, axes=([1], [k])), 0, k)) ** 2)
            t = p
        return t, res

    full, rfull = proj(y)
    bounds = [0, 3, 5, 9]
    pieces = [proj(y[:, :, bounds[i]:bounds[i + 1]]) for i in range(3)]
    np.testing.assert_allclose(np.concatenate([p[0] for p in pieces], axis=2), full, rtol=1e-13, atol=1e-14)
    for k in range(2):
        np.testing.assert_allclose(sum(p[1][k] for p in pieces), rfull[k], rtol=1e-12)


class _HostEngine:
    """Host stand-in for the device engine with the same protocol surface
    (begin / exchange_tensors / cont): the payload is the raw slab, the finish
    runs the CPU checker on the gathered slice."""

    class Ex:
        op = 0  # allgather

        def __init__(self, pending, count):
            self.pending, self.count = pending, count

    def __init__(self, handle, dims, bounds, rank, world):
        self.h, self.dims, self.bounds, self.rank, self.world = handle, dims, bounds, rank, world
        inner = int(np.prod(dims[:-1]))
        self.inner = inner
        self.count = inner * max(bounds[g + 1] - bounds[g] for g in range(world))
        self.send = torch.zeros(self.count, dtype=torch.float64)
        self.recv = torch.zeros(self.count * world, dtype=torch.float64)

    def begin(self, slab):
        self.send.zero_()
        self.send[: len(slab)] = torch.from_numpy(np.asarray(slab))
        return self.Ex(1, self.count)

    def exchange_tensors(self, ex):
        return self.send, self.recv

    def sync_exchange(self):
        self.syncs = getattr(self, "syncs", 0) + 1

    def cont(self, ex):
        r = self.recv.numpy().reshape(self.world, self.count)
        y = np.concatenate([r[g, : self.inner * (self.bounds[g + 1] - self.bounds[g])]
                            for g in range(self.world)])
        self.h.update_flat(y)
        return self.Ex(0, 0)


def _gloo_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import torch.distributed as dist
    from paper_2308_16395_b200 import datagen as dg, sharded as SH
    import py_oracle

    dist.init_process_group("gloo")
    comm = SH.TorchComm()
    cfg = dg.scaled(dg.CONFIGS["c2"], (12, 10, 9), n_slices=9, n_init=3)
    gen = dg.TuckerStream(cfg)
    chk = py_oracle.load_oracle()
    x = gen.init_numpy().reshape(gen.init_dims()[::-1]).transpose()
    h = chk.stream_init(x, cfg.tau)
    dims = cfg.slice_dims
    bounds = SH.shard_bounds(dims[-1], world)
    eng = _HostEngine(h, dims, bounds, rank, world)
    ex_total = 0
    for t in range(cfg.n_init, cfg.n_slices):
        y = gen.slice_numpy(t)
        n, _ = SH.drive(eng, SH.slab_of(y, dims, bounds, rank, mode=len(dims) - 1), comm)
        ex_total += n
    st = h.export()
    rec = {"rank": rank, "exchanges": ex_total, "core": [float(v) for v in np.ravel(st.core)],
           "n_d": int(st.n_d), "err": float(st.squared_error)}
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(rec, f)
    dist.destroy_process_group()


def test_two_gloo_ranks_sharded_protocol(tmp_path, oracle):
    import torch.multiprocessing as mp
    from paper_2308_16395_b200 import datagen as dg
    world = 2
    mp.spawn(_gloo_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    recs = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    cfg = dg.scaled(dg.CONFIGS["c2"], (12, 10, 9), n_slices=9, n_init=3)
    gen = dg.TuckerStream(cfg)
    h = oracle.stream_init(gen.init_numpy().reshape(gen.init_dims()[::-1]).transpose(), cfg.tau)
    for t in range(cfg.n_init, cfg.n_slices):
        h.update_flat(gen.slice_numpy(t))
    ref = h.export()
    for r in recs:
        assert r["exchanges"] == cfg.n_slices - cfg.n_init      # one allgather per slice
        assert r["n_d"] == ref.n_d
        assert r["core"] == [float(v) for v in np.ravel(ref.core)]  # bitwise
    assert recs[0]["core"] == recs[1]["core"]


# ------------------------------------------------------------------- GPU
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run_loopback(case, world, bounds=None, mode=None):
    from paper_2308_16395_b200 import sharded as SH
    states = []
    for g in range(world):
        st = SH.ShardedStreamingState(device=0)
        st.init_flat(case.init_flat, case.init_dims, case.tau)
        b = st.setup(g, world, bounds, mode)
        states.append(st)
    grp = SH.LoopbackGroup(states)
    dims = tuple(case.init_dims[:-1])
    for y in case.slices:
        grp.stream_update([np.ascontiguousarray(SH.slab_of(y, dims, b, g, states[0].mode))
                           for g in range(world)])
    return states


def _assert_ranks_identical(ex):
    for other in ex[1:]:
        assert other.core_dims == ex[0].core_dims
        np.testing.assert_array_equal(other.core, ex[0].core)
        np.testing.assert_array_equal(other.left, ex[0].left)
        np.testing.assert_array_equal(other.sigma, ex[0].sigma)
        for a, b in zip(other.factors, ex[0].factors):
            np.testing.assert_array_equal(a, b)
        assert other.squared_error == ex[0].squared_error
        assert other.nonstream_discarded_sq == ex[0].nonstream_discarded_sq


@pytest.mark.gpu
@pytest.mark.parametrize("name,world", [("c1", 2), ("c1", 3), ("growth24", 2), ("growth24", 4),
                                        ("c3_40", 2), ("order5", 2), ("edges", 2), ("order2", 2),
                                        ("thin", 2), ("random_full", 3)])
def test_loopback_sharded_vs_golden(golden, name, world):
    _need_gpu()
    case = cases.STREAM_CASES[name]()
    if case.init_dims[-2] < world:
        pytest.skip("fewer rows than ranks")
    states = _run_loopback(case, world)
    ex = [st.export() for st in states]
    _assert_ranks_identical(ex)  # every rank bitwise identical
    g = golden("stream_" + name)
    mg = P.metrics_arrays(states[0].metrics(), ex[0].order)
    mc = P.compare_metrics(mg, P.golden_metrics(g), float(g["total_input_sq"]))
    sc = P.compare_states(ex[0], P.state_from_golden(g))
    print(name, world, mc, sc)
    P.assert_parity(mc, sc)


@pytest.mark.gpu
@pytest.mark.parametrize("name,world,mode", [("c3_40", 2, 0), ("c3_40", 3, 1), ("growth24", 2, 0),
                                             ("growth24", 3, 1), ("order5", 2, 1), ("order5", 2, 2),
                                             ("edges", 2, 0), ("random_full", 2, 1)])
def test_loopback_selectable_shard_mode_vs_golden(golden, name, world, mode):
    """tsg_shard_setup_mode: the slice split along a named spatial mode (BASELINE
    configs[2] shards along mode 1): modes before it are local, the rest runs
    redundantly on the gathered tensor. Ranks bitwise identical, golden parity."""
    _need_gpu()
    case = cases.STREAM_CASES[name]()
    if mode > len(case.init_dims) - 2 or case.init_dims[mode] < world:
        pytest.skip("mode not available")
    states = _run_loopback(case, world, mode=mode)
    ex = [st.export() for st in states]
    _assert_ranks_identical(ex)
    g = golden("stream_" + name)
    mc = P.compare_metrics(P.metrics_arrays(states[0].metrics(), ex[0].order), P.golden_metrics(g),
                           float(g["total_input_sq"]))
    sc = P.compare_states(ex[0], P.state_from_golden(g))
    print(name, world, mode, mc, sc)
    P.assert_parity(mc, sc)


@pytest.mark.gpu
@pytest.mark.parametrize("world,mode", [(2, None), (4, None), (3, 1)])
def test_local_mode_growth_exchanges_partial_gram(oracle, world, mode):
    """Basis growth at a LOCAL mode (sthosvd.cpp:45-59 and
    streaming.cpp:142-151 split over the ranks): the ranks all-reduce the
    N_k x N_k partial Gram of their residual parts, solve redundantly and keep
    K = W^T E local — the mode's input is never gathered. Asserts, per
    exchange, doubles per rank <= max(N_k^2, compressed tensor + pairs), that
    the all-reduces carry exactly N_k^2 doubles, ranks bitwise identical and
    parity with the CPU checker."""
    _need_gpu()
    from paper_2308_16395_b200 import datagen as dg, streaming as S
    cfg = dg.scaled(dg.CONFIGS["c5"], (40, 36, 44), n_slices=30, n_init=6, name="c5_local_growth")
    cfg.growth = (3, 2, 8, 9)   # spatial ranks 3 -> 9, +2 every 8 slices
    cfg.spatial_ranks = (9, 9, 9)
    cfg.time_rank = 9
    case = cases.config_case(cfg)
    states = _run_loopback(case, world, mode=mode)
    ex = [st.export() for st in states]
    _assert_ranks_identical(ex)
    smode = states[0].mode
    dims = tuple(case.init_dims[:-1])
    log = states[0].exchange_log
    reduces = [c for op, c in log if op == S.XCHG_ALLREDUCE_SUM]
    gathers = [c for op, c in log if op == S.XCHG_ALLGATHER]
    assert reduces, "the stream never grew a local mode"
    local_sq = {(dims[k] * dims[k] + 1) // 2 * 2 for k in range(smode)}
    assert set(reduces) <= local_sq, (reduces, local_sq)
    # every gather is a compressed tensor: ranks of the local modes x the
    # rank's rows x the uncompressed modes after the shard mode (+ pairs)
    ranks = ex[0].core_dims
    rows = max(b - a for a, b in zip(states[0].bounds[:-1], states[0].bounds[1:]))
    comp = int(np.prod(ranks[:smode])) * rows * int(np.prod(dims[smode + 1:])) + 2 * smode + 2
    assert max(gathers) <= comp, (max(gathers), comp)
    masks = [m["expanded_mask"] for m in states[0].metrics()]
    assert any(m & ((1 << smode) - 1) for m in masks)
    x = case.init_flat.reshape(case.init_dims[::-1]).transpose()
    ho = oracle.stream_init(x, case.tau)
    for y in case.slices:
        ho.update_flat(y)
    so = ho.export()
    mc = P.compare_metrics(P.metrics_arrays(states[0].metrics(), ex[0].order),
                           P.metrics_arrays(ho.metrics(), so.order), so.total_input_sq)
    sc = P.compare_states(ex[0], so)
    print("local growth", world, smode, "exchanges", len(log), "allreduces", len(reduces), mc, sc)
    P.assert_parity(mc, sc)


@pytest.mark.gpu
def test_sharded_uneven_bounds_and_errors(golden):
    _need_gpu()
    from paper_2308_16395_b200 import sharded as SH
    from paper_2308_16395_b200 import streaming as S
    case = cases.STREAM_CASES["growth24"]()
    n = case.init_dims[-2]
    states = _run_loopback(case, 3, bounds=[0, 1, n - 2, n])
    g = golden("stream_growth24")
    e = states[0].export()
    mc = P.compare_metrics(P.metrics_arrays(states[0].metrics(), e.order), P.golden_metrics(g),
                           float(g["total_input_sq"]))
    P.assert_parity(mc, P.compare_states(e, P.state_from_golden(g)))
    st = SH.ShardedStreamingState(device=0)
    st.init_flat(case.init_flat, case.init_dims, case.tau)
    with pytest.raises(S.InvalidArgument):
        st.setup(0, 2, [0, 0, n])           # an empty shard
    with pytest.raises(S.InvalidArgument):
        st.setup(2, 2)                      # rank out of range
    with pytest.raises(S.InvalidArgument):
        st.begin(np.zeros(4))               # not set up
    st.setup(0, 2)
    with pytest.raises(S.InvalidArgument):
        st.cont(S.TsgExchange())            # nothing pending


class _SideStreamComm:
    """World-1 comm whose copy runs on its own NON-blocking torch stream: not
    ordered behind the engine's stream unless drive() synchronises."""

    def __init__(self):
        self.side = torch.cuda.Stream()

    def allgather(self, send, recv, stream=None):
        assert stream is None
        with torch.cuda.stream(self.side):
            recv.copy_(send, non_blocking=True)

    allreduce = allgather


@pytest.mark.gpu
def test_drive_without_stream_orders_exchange():
    """drive(stream=None) over libtsg: the exchange buffers are
    only valid in the engine stream's order, so drive() must drain that stream
    around a collective issued elsewhere. Same bytes as the loopback path."""
    _need_gpu()
    from paper_2308_16395_b200 import sharded as SH
    case = cases.STREAM_CASES["growth24"]()
    st = SH.ShardedStreamingState(device=0)
    st.init_flat(case.init_flat, case.init_dims, case.tau)
    b = st.setup(0, 1)
    comm = _SideStreamComm()
    dims = tuple(case.init_dims[:-1])
    for y in case.slices:
        SH.drive(st, np.ascontiguousarray(SH.slab_of(y, dims, b, 0)), comm)
    e = st.export()
    ref = _run_loopback(case, 1)[0].export()
    np.testing.assert_array_equal(e.core, ref.core)
    np.testing.assert_array_equal(e.left, ref.left)
    np.testing.assert_array_equal(e.sigma, ref.sigma)


def _nccl_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests"), os.path.join(root, "oracle")):
        sys.path.insert(0, p)
    import torch.distributed as dist
    import cases as CS
    from paper_2308_16395_b200 import sharded as SH
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl")
    case = CS.STREAM_CASES["growth24"]()
    st = SH.ShardedStreamingState(device=rank)
    st.init_flat(case.init_flat, case.init_dims, case.tau)
    b = st.setup(rank, world)
    comm = SH.TorchComm()
    dims = tuple(case.init_dims[:-1])
    for y in case.slices:
        st.stream_update_slab(np.ascontiguousarray(SH.slab_of(y, dims, b, rank)), comm)
    e = st.export()
    np.savez(q, core=e.core, left=e.left, sigma=e.sigma, exchanges=st.exchanges)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_transport_world1_matches_loopback(tmp_path):
    """The torch.distributed NCCL path (ExternalStream on the engine stream)
    with one rank gives the same bytes as the loopback exchange."""
    _need_gpu()
    import torch.multiprocessing as mp
    out = str(tmp_path / "r0.npz")
    mp.spawn(_nccl_worker, args=(1, _free_port(), out), nprocs=1, join=True)
    z = np.load(out)
    case = cases.STREAM_CASES["growth24"]()
    ref = _run_loopback(case, 1)[0].export()
    np.testing.assert_array_equal(z["core"], ref.core)
    np.testing.assert_array_equal(z["left"], ref.left)
    assert int(z["exchanges"]) >= len(case.slices)


@pytest.mark.gpu
@pytest.mark.slow
def test_loopback_sharded_config4_vs_oracle(oracle):
    """Config-4 generator (5-way, 48^3 x 16): the variable mode (16 rows) is
    the sharded mode, modes 0-2 are local and grow on most slices, so the
    growth-at-a-local-mode exchange (gather of that mode's input) runs every
    few slices. Ranks bitwise identical, state within the parity bounds."""
    _need_gpu()
    from paper_2308_16395_b200 import datagen as dg
    cfg = dg.scaled(dg.CONFIGS["c4"], (48, 48, 48, 16), n_slices=15, n_init=10, name="c4_48s")
    case = cases.config_case(cfg)
    states = _run_loopback(case, 2)
    a, b = states[0].export(), states[1].export()
    np.testing.assert_array_equal(a.core, b.core)
    np.testing.assert_array_equal(a.left, b.left)
    x = case.init_flat.reshape(case.init_dims[::-1]).transpose()
    ho = oracle.stream_init(x, case.tau)
    for y in case.slices:
        ho.update_flat(y)
    so = ho.export()
    mc = P.compare_metrics(P.metrics_arrays(states[0].metrics(), a.order),
                           P.metrics_arrays(ho.metrics(), so.order), so.total_input_sq)
    sc = P.compare_states(a, so)
    print("c4 sharded", mc, sc)
    P.assert_parity(mc, sc, resid_tol=5e-8)
