"""Component-sharded DynLP batches across GPUs.

One process (rank) per GPU.  Every rank applies the same batches -- the
structure, tau, intra-batch components, initialisation and reachability are
replicated and bit-identical on every rank -- and propagates only the
connected components it owns (a hash of the component's minimum vertex id).
Frontiers never cross components, so the only exchange is the per-column
phase bookkeeping of engine.py:375-405 (rounds, updates, max |delta|,
frontier non-empty, eligible counts): a few bytes per phase, reduced with the
caller's collective (NCCL all-reduce over NVLink with torch.distributed, or an
in-process reduction for virtual shards on one device).  Reports are the
global ones; labels of a vertex live on the rank that last propagated it.

mode="rows" partitions the rows instead (rank r evaluates v % world == r),
for a stream dominated by one giant component: every global round ends with
an all-gather of the evaluated rows (vertex, masks, new labels) and each rank
applies the other ranks' labels and frontier claims, so labels are
replicated on every rank.
"""

from __future__ import annotations

import ctypes as C
import threading
from typing import Callable, Optional

import numpy as np

from . import _native
from .engine import DynamicGraph, EngineConfig, LabelState, _reports, _result
from .batch import as_arrays

_REDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int64), C.c_int32,
                      C.POINTER(C.c_double), C.c_int32)

# collective(imax: int64[], isum: int64[], dmax: float64[]) -> None, in place
Collective = Callable[[np.ndarray, np.ndarray, np.ndarray], None]


def torch_collective(group=None, device=None) -> Collective:
    """Reduction over a torch.distributed group (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    def run(imax: np.ndarray, isum: np.ndarray, dmax: np.ndarray) -> None:
        for arr, op in ((imax, dist.ReduceOp.MAX), (isum, dist.ReduceOp.SUM), (dmax, dist.ReduceOp.MAX)):
            if arr.size == 0:
                continue
            t = torch.from_numpy(arr.copy())
            if device is not None:
                t = t.to(device)
            dist.all_reduce(t, op=op, group=group)
            arr[:] = t.cpu().numpy()

    return run


class InProcessCollective:
    """Reduction among `world` threads of one process (virtual shards)."""

    def __init__(self, world: int) -> None:
        self.world = world
        self._bar = threading.Barrier(world)
        self._slots = [None] * world
        self._out = None

    def for_rank(self, rank: int) -> Collective:
        def run(imax, isum, dmax):
            self._slots[rank] = (imax.copy(), isum.copy(), dmax.copy())
            if self._bar.wait() == 0:
                a = [s[0] for s in self._slots]
                b = [s[1] for s in self._slots]
                d = [s[2] for s in self._slots]
                self._out = (np.max(a, axis=0), np.sum(b, axis=0), np.max(d, axis=0))
            self._bar.wait()
            imax[:], isum[:], dmax[:] = self._out
            self._bar.wait()

        return run


class ShardedGraph(DynamicGraph):
    """DynamicGraph holding this rank's share of the propagation."""

    # components: sticky LPT placement by edge count; components_hash: placement by
    # a hash of the component root; rows: row partition for one giant component
    MODES = {"components": 0, "rows": 1, "components_hash": 2}

    def __init__(self, device: int, num_classes: int, rank: int, world: int, collective: Optional[Collective],
                 mode: str = "components", nccl_id: Optional[bytes] = None) -> None:
        """collective: a host reduction (torch.distributed, in-process for
        virtual shards); or None with nccl_id: the engine's own NCCL
        communicator, every exchange on device buffers (dlp_shard_nccl)."""
        super().__init__(device, num_classes)
        if mode not in self.MODES:
            raise ValueError(f"unknown shard mode {mode!r}")
        self.rank, self.world, self.mode = int(rank), int(world), mode
        self._check(self._lib.dlp_shard_set(self._h, self.rank, self.world))
        self._check(self._lib.dlp_shard_mode(self._h, self.MODES[mode]))
        self._collective = collective
        self._cb = None
        if collective is None:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("a collective or a 128-byte NCCL id is required")
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            self._check(self._lib.dlp_shard_nccl(self._h, buf, self.world, self.rank))
            return

        def cb(ctx, imax, nimax, isum, nisum, dmax, ndmax):
            try:
                a = np.ctypeslib.as_array(imax, (nimax,)) if nimax else np.zeros(0, np.int64)
                b = np.ctypeslib.as_array(isum, (nisum,)) if nisum else np.zeros(0, np.int64)
                d = np.ctypeslib.as_array(dmax, (ndmax,)) if ndmax else np.zeros(0, np.float64)
                self._collective(a, b, d)
                return 0
            except Exception:  # the engine turns a failed collective into an error
                return 1

        self._cb = _REDUCE(cb)

    def owned(self) -> np.ndarray:
        n = self.num_slots
        o = np.empty(n, dtype=np.uint8)
        self._check(self._lib.dlp_read_owned(self._h, _native.ptr(o), n))
        return o.astype(bool)

    def apply_sharded(self, batch, cfg: EngineConfig):
        t, ids, gt, owner, other, w, dels = as_arrays(batch)
        b = _native.Batch(t, len(ids), _native.ptr(ids), _native.ptr(gt), len(owner), _native.ptr(owner),
                          _native.ptr(other), _native.ptr(w), len(dels), _native.ptr(dels))
        reps = (_native.Report * self.ncol)()
        c = cfg._c(self.num_classes)
        cb = C.cast(self._cb, C.c_void_p) if self._cb is not None else None  # None: the engine's NCCL
        rc = self._lib.dlp_apply_batch_sharded(self._h, C.byref(c), C.byref(b), cb, None, reps)
        self._version += 1
        self._check(rc)
        return _reports(reps, "dynlp")


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 makes it, the caller broadcasts it)."""
    lib = _native.load()
    buf = C.create_string_buffer(128)
    rc = lib.dlp_nccl_unique_id(buf)
    if rc != 0:
        raise RuntimeError("ncclGetUniqueId failed (libnccl.so.2 missing?)")
    return buf.raw


def nccl_sharded_graph(device: int, num_classes: int, mode: str = "components", group=None) -> "ShardedGraph":
    """A ShardedGraph for this torch.distributed rank whose exchanges run on
    the engine's own NCCL communicator (the id travels over `group`)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return ShardedGraph(device, num_classes, rank, world, None, mode, nccl_id=obj[0])


def apply_batch_sharded(graph: ShardedGraph, labels: LabelState, batch, cfg: EngineConfig):
    """engine.apply_batch for one rank of a component-sharded run (every rank
    calls it with the same batch); returns the global reports."""
    cfg.validate()
    labels._bind(graph)
    return labels, _result(graph, graph.apply_sharded(batch, cfg))


def merge_labels(parts) -> np.ndarray:
    """Merge per-rank (F, owned) pairs into the global label matrix."""
    F = None
    for f, owned in parts:
        if F is None:
            F = f.copy()
        else:
            F[:, owned] = f[:, owned]
    return F


def gather_labels(graph: ShardedGraph, group=None, device=None) -> np.ndarray:
    """Global labels on every rank (all-gather of labels and ownership)."""
    import torch
    import torch.distributed as dist

    f, _ = graph.read_labels()
    owned = graph.owned()
    ft = torch.from_numpy(f).to(device) if device is not None else torch.from_numpy(f)
    ot = torch.from_numpy(owned.astype(np.uint8)).to(device) if device is not None else \
        torch.from_numpy(owned.astype(np.uint8))
    fs = [torch.empty_like(ft) for _ in range(graph.world)]
    os_ = [torch.empty_like(ot) for _ in range(graph.world)]
    dist.all_gather(fs, ft, group=group)
    dist.all_gather(os_, ot, group=group)
    return merge_labels([(a.cpu().numpy(), b.cpu().numpy().astype(bool)) for a, b in zip(fs, os_)])


def run_virtual_shards(batches, cfg: EngineConfig, world: int, num_classes: int = 2, device: int = 0,
                       on_batch: Optional[Callable] = None, mode: str = "components"):
    """Run a stream as `world` component shards on ONE device (threads +
    in-process reduction): the sharded protocol without NCCL, for tests."""
    coll = InProcessCollective(world)
    graphs = [ShardedGraph(device, num_classes, r, world, coll.for_rank(r), mode) for r in range(world)]
    labels = [LabelState() for _ in range(world)]
    out = []
    for b in batches:
        res = [None] * world
        errs = []

        def work(r):
            try:
                res[r] = apply_batch_sharded(graphs[r], labels[r], b, cfg)[1]
            except Exception as e:  # pragma: no cover - surfaced below
                errs.append(e)

        th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        if errs:
            raise errs[0]
        F = merge_labels([(g.read_labels()[0], g.owned()) for g in graphs])
        if mode == "rows":  # labels are replicated: every rank holds the whole matrix
            for g in graphs[1:]:
                if not np.array_equal(g.read_labels()[0].view(np.int64), F.view(np.int64)):
                    raise RuntimeError(f"row-partitioned rank {g.rank} diverged from the merged labels")
        out.append((res[0], F))
        if on_batch:
            on_batch(res, F)
    for g in graphs:
        g.close()
    return out
