"""Component sharding.

CPU (gloo, world_size 2): the torch collective the engine's phase reduction
uses.  GPU: the sharded protocol as virtual shards on one device (threads +
in-process reduction, same C++ state machine and action-mode kernel the
NCCL path runs), bit-identical to the unsharded engine: reports and merged
labels."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    sys.path.insert(0, os.path.dirname(HERE))
    import torch.distributed as dist

    from paper_2604_06596_b200.sharded import torch_collective

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    coll = torch_collective()
    imax = np.array([rank * 10, 5 - rank], dtype=np.int64)
    isum = np.array([rank + 1, 100], dtype=np.int64)
    dmax = np.array([0.25 * rank, -1.0 + rank], dtype=np.float64)
    coll(imax, isum, dmax)
    q.put((rank, imax.tolist(), isum.tolist(), dmax.tolist()))
    dist.destroy_process_group()


def test_torch_collective_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, imax, isum, dmax in out:
        assert imax == [10, 5] and isum == [3, 200] and dmax == [0.25, 0.0]


def _rows_gather_worker(rank, world, port, q):
    """The row partition's all-gather (abi.cu rows_exchange): each rank writes
    its rows (vertex, masks, label bit patterns) into its own segment of an
    int64 vector; the sum-reduction must return every rank's words exactly."""
    sys.path.insert(0, os.path.dirname(HERE))
    import torch.distributed as dist

    from paper_2604_06596_b200.sharded import torch_collective

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    coll = torch_collective()
    C = 3
    rng = np.random.default_rng(rank)
    cnt = np.zeros(world, np.int64)
    mine = 5 + rank
    cnt[rank] = mine
    coll(np.zeros(1, np.int64), cnt, np.zeros(1))
    off = int(cnt[:rank].sum())
    vals = rng.random((mine, C))
    vals[0, 0] = -0.0
    vals[1, 1] = np.frombuffer(np.uint64(0x7FF4000000000001).tobytes(), np.float64)[0]  # boxed class 1
    buf = np.zeros((int(cnt.sum()), 3 + C), np.int64)
    buf[off:off + mine, 0] = np.arange(mine) * world + rank
    buf[off:off + mine, 1] = 0b101
    buf[off:off + mine, 2] = 0b100
    buf[off:off + mine, 3:] = vals.view(np.int64)
    flat = buf.ravel().copy()
    coll(np.zeros(1, np.int64), flat, np.zeros(1))
    q.put((rank, cnt.tolist(), flat.tolist(), vals.view(np.int64).tolist()))
    dist.destroy_process_group()


def test_rows_allgather_exact_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rows_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    (r0, cnt0, flat0, v0), (r1, cnt1, flat1, v1) = out
    assert cnt0 == cnt1 == [5, 6] and flat0 == flat1
    g = np.array(flat0, np.int64).reshape(11, 6)
    assert g[:5, 3:].tolist() == v0 and g[5:, 3:].tolist() == v1  # label bit patterns survive exactly
    assert g[:5, 0].tolist() == [0, 2, 4, 6, 8] and g[5:, 0].tolist() == [1, 3, 5, 7, 9, 11]


def test_in_process_collective_threads():
    import threading

    from paper_2604_06596_b200.sharded import InProcessCollective

    coll = InProcessCollective(3)
    res = {}

    def w(r):
        a, b, d = np.array([r]), np.array([r, 1]), np.array([float(-r)])
        coll.for_rank(r)(a, b, d)
        res[r] = (a.tolist(), b.tolist(), d.tolist())

    th = [threading.Thread(target=w, args=(r,)) for r in range(3)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert all(v == ([2], [3, 3], [0.0]) for v in res.values())


def _unsharded(batches, cfg, ncls):
    from paper_2604_06596_b200.engine import DynamicGraph, LabelState, apply_batch

    g, lab = DynamicGraph(0, num_classes=ncls), LabelState()
    out = []
    for b in batches:
        lab, rep = apply_batch(g, lab, b, cfg)
        out.append((rep if isinstance(rep, list) else [rep], lab.F.copy()))
    g.close()
    return out


def _stream(kind):
    from paper_2604_06596_b200 import streams

    if kind == "blobs10":  # well-separated blobs: many components to distribute
        bl = streams.make_blobs(5000, 16, 10, 3, spread=40.0)
        e = streams.knn_graph_exact(bl.x, 8)
        gt = streams.stratified_seeds(bl.classes, 0.02, 3)
        return streams.phased_stream(5000, e, bl.classes, gt, 500, 3, 0.75, 0.02, 0.23, initial_gt=20).batches, 10
    if kind == "giant":  # overlapping classes: one giant component (row partition's case)
        bl = streams.make_blobs(6000, 8, 3, 5, spread=1.0)
        e = streams.knn_graph_exact(bl.x, 10)
        gt = streams.stratified_seeds(bl.classes, 0.02, 5)
        return streams.phased_stream(6000, e, bl.classes, gt, 600, 5, 0.7, 0.02, 0.28, initial_gt=6).batches, 3
    bl = streams.make_blobs(4000, 8, 2, 4, spread=30.0)
    e = streams.knn_graph_exact(bl.x, 6)
    gt = streams.stratified_seeds(bl.classes, 0.02, 4)
    return streams.phased_stream(4000, e, bl.classes, gt, 400, 4, 0.7, 0.02, 0.28, initial_gt=4).batches, 2


@pytest.mark.gpu
@pytest.mark.parametrize("kind,world,mode", [("blobs2", 2, "components"), ("blobs10", 2, "components"),
                                             ("blobs10", 3, "components"), ("blobs10", 3, "components_hash"), ("blobs2", 2, "rows"),
                                             ("blobs10", 3, "rows"), ("giant", 2, "rows"), ("giant", 4, "rows")])
def test_virtual_shards_bit_identical(gpu_device, kind, world, mode):
    from paper_2604_06596_b200.engine import EngineConfig
    from paper_2604_06596_b200.sharded import run_virtual_shards

    batches, ncls = _stream(kind)
    cfg = EngineConfig(delta=1e-5)
    want = _unsharded(batches, cfg, ncls)
    got = run_virtual_shards(batches, cfg, world, num_classes=ncls, mode=mode)
    for t, ((rw, Fw), (rg, Fg)) in enumerate(zip(want, got)):
        rg = rg if isinstance(rg, list) else [rg]
        for c, (a, b) in enumerate(zip(rw, rg)):
            ta = (a.iterations, a.updates, a.max_change, a.converged, a.warnings, a.edges_traversed,
                  a.certify_sweeps)
            tb = (b.iterations, b.updates, b.max_change, b.converged, b.warnings, b.edges_traversed,
                  b.certify_sweeps)
            assert ta == tb, f"batch {t} column {c}: {ta} != {tb}"
        assert Fw.tobytes() == Fg.tobytes(), f"batch {t}: labels differ"


def _nccl_id_worker(rank, world, port, q):
    sys.path.insert(0, os.path.dirname(HERE))
    import torch.distributed as dist

    from paper_2604_06596_b200.sharded import nccl_unique_id

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    q.put((rank, obj[0]))
    dist.destroy_process_group()


def test_nccl_id_broadcast_gloo_world2():
    """The host plumbing of the in-handle NCCL communicator: rank 0's 128-byte
    ncclUniqueId (libnccl via the engine library) reaches every rank intact."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_nccl_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert len(got[0]) == 128 and got[0] == got[1]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,mode", [("blobs10", "components"), ("giant", "rows")])
def test_nccl_in_handle_world1(gpu_device, kind, mode):
    """The engine's own NCCL communicator (world 1 on the one GPU): every
    exchange -- phase all-reduces, migration, the row all-gather of packed
    device records -- runs as an NCCL collective; bit-identical to the
    unsharded engine."""
    from paper_2604_06596_b200.engine import EngineConfig, LabelState
    from paper_2604_06596_b200.sharded import ShardedGraph, apply_batch_sharded, nccl_unique_id

    batches, ncls = _stream(kind)
    cfg = EngineConfig(delta=1e-5)
    want = _unsharded(batches, cfg, ncls)
    g = ShardedGraph(0, ncls, 0, 1, None, mode, nccl_id=nccl_unique_id())
    lab = LabelState()
    for t, (b, (rw, Fw)) in enumerate(zip(batches, want)):
        lab, rg = apply_batch_sharded(g, lab, b, cfg)
        rg = rg if isinstance(rg, list) else [rg]
        for c, (a, x) in enumerate(zip(rw, rg)):
            assert (a.iterations, a.updates, a.max_change, a.converged, a.warnings) == \
                (x.iterations, x.updates, x.max_change, x.converged, x.warnings), (t, c)
        assert lab.F.tobytes() == Fw.tobytes(), f"batch {t}: labels differ"
    g.close()


def _engine_proc(rank, world, port, mode, q):
    """One rank of a 2-process sharded engine run on the one GPU (gloo carries
    the phase reductions and the row exchange between the processes)."""
    sys.path.insert(0, os.path.dirname(HERE))
    sys.path.insert(0, HERE)
    try:
        import torch.distributed as dist

        from paper_2604_06596_b200.engine import EngineConfig, LabelState
        from paper_2604_06596_b200.sharded import ShardedGraph, apply_batch_sharded, torch_collective

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        batches, ncls = _stream("blobs10" if mode != "rows" else "giant")
        g = ShardedGraph(0, ncls, rank, world, torch_collective(), mode)
        lab = LabelState()
        reps = []
        for b in batches:
            lab, r = apply_batch_sharded(g, lab, b, EngineConfig(delta=1e-5))
            r = r if isinstance(r, list) else [r]
            reps.append([(x.iterations, x.updates, x.max_change, x.converged, x.warnings) for x in r])
        F, _ = g.read_labels()
        q.put((rank, reps, F, g.owned()))
        g.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback

        q.put((rank, "error", f"{e!r}\n{traceback.format_exc()}", None))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["components", "rows"])
def test_engine_two_processes_gloo(gpu_device, mode):
    """The sharded ENGINE across two processes (world_size 2, gloo collective,
    both ranks on the one GPU): global reports and merged labels bitwise equal
    to the unsharded engine."""
    from paper_2604_06596_b200.engine import EngineConfig
    from paper_2604_06596_b200.sharded import merge_labels

    batches, ncls = _stream("blobs10" if mode != "rows" else "giant")
    want = _unsharded(batches, EngineConfig(delta=1e-5), ncls)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_engine_proc, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = {}
    for _ in range(2):
        rank, reps, F, owned = q.get(timeout=600)
        assert reps != "error", F
        out[rank] = (reps, F, owned)
    for p in ps:
        p.join(timeout=120)
    for t, (rw, _) in enumerate(want):
        exp = [(a.iterations, a.updates, a.max_change, a.converged, a.warnings) for a in rw]
        assert out[0][0][t] == exp and out[1][0][t] == exp, f"batch {t}"
    F = merge_labels([(out[r][1], out[r][2]) for r in range(2)]) if mode != "rows" else out[0][1]
    assert F.tobytes() == want[-1][1].tobytes()
