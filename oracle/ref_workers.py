"""Concurrent one-vs-rest reference runs for bench.py (TEST INFRASTRUCTURE ONLY).

The reference is binary (labels.py:42-43); a C-class batch is C independent
reference runs of ``engine.apply_batch`` (engine.py:328-413), one per
one-vs-rest column (class c seeds -> 1, other seeds -> 0; SURVEY.md §8(c)
O-2).  ``RefColumnPool`` runs those C runs as C worker processes, so one
*step* is the whole C-class batch processed by the unmodified compiled
reference on the host's cores (column c in worker c, each with
``EngineConfig(threads=cores // C)``), the columns concurrently.

One spawned master process
  * loads the synthetic stream from an ``.npz`` (bench.py's cache),
  * replays the structure of batches [0, t_h) once with
    ``apply_batch_structure`` (engine.py:141-156, no propagation),
  * forks one worker per column (the replayed graph is shared copy-on-write),
    which installs its column's ground truth and hand-off labels (the state
    before batch t_h, SURVEY.md §8(d) D-6 "state handoff"),
  * then applies batches on request and returns (seconds, report tuple,
    sha256 of f[:num_slots]).

Only numpy and the compiled reference (oracle/_ref) are imported by the
workers: no CUDA library of this repository is ever mapped by them.
"""

from __future__ import annotations

import hashlib
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_stream(path):
    """Batches of a bench stream cache (.npz written by bench.make_stream) as
    plain tuples (t, ids, gt, owner, other, w, dels)."""
    z = np.load(path)
    a = {k: z[k] for k in ("ids", "gt", "own", "oth", "w", "dels", "io", "eo", "do")}  # one read per array
    io, eo, do = a["io"], a["eo"], a["do"]
    out = []
    for t in range(len(io) - 1):
        out.append((t, a["ids"][io[t]:io[t + 1]], a["gt"][io[t]:io[t + 1]], a["own"][eo[t]:eo[t + 1]],
                    a["oth"][eo[t]:eo[t + 1]], a["w"][eo[t]:eo[t + 1]], a["dels"][do[t]:do[t + 1]]))
    return out


def column_gt(gt, c, ncol):
    """One-vs-rest remap of a batch's ground truth for label column c."""
    g = np.asarray(gt)
    if ncol == 1:
        return g.astype(np.int8)
    return np.where(g < 0, -1, np.where(g == c, 1, 0)).astype(np.int8)


def f_digest(f) -> str:
    return hashlib.sha256(np.ascontiguousarray(f, dtype=np.float64).tobytes()).hexdigest()


def _column_loop(conn, barrier, g, lab, batches, raw_gt, c, ncol, F_c, delta, threads):
    """Column worker (forked from the master after the structure replay):
    install column c's ground truth and hand-off labels, then apply batches
    on request."""
    from dynlp.engine import EngineConfig, apply_batch
    from dynlp.graph import BatchUpdate

    try:
        n = g.num_slots
        lab.gt[:n] = column_gt(raw_gt[:n], c, ncol)
        if F_c is not None:
            lab.f[:n] = F_c
        cfg = EngineConfig(delta=delta, threads=threads)
        conn.send(("ready", n))
        while True:
            msg = conn.recv()
            if msg[0] == "stop":
                break
            t, ids, gt, own, oth, w, dels = batches[msg[1]]
            b = BatchUpdate(int(t), ids, column_gt(gt, c, ncol), own, oth, w, dels)
            barrier.wait()
            s = time.perf_counter()
            lab, r = apply_batch(g, lab, b, cfg)
            dt = time.perf_counter() - s
            n = g.num_slots
            conn.send(("done", dt, (r.iterations, r.updates, r.max_change, int(r.converged)),
                       f_digest(lab.f[:n]), n))
    except Exception as e:  # surfaced by the parent
        import traceback

        conn.send(("error", f"column {c}: {e!r}\n{traceback.format_exc()}"))
    finally:
        conn.close()


def _master(conn, stream_path, handoff_path, t_h, ncol, delta, threads):
    """Spawned once, never touches CUDA: replays the structure of batches
    [0, t_h) with the reference (apply_batch_structure, engine.py:141-156),
    then forks the C column workers, which share the replayed graph
    copy-on-write, and relays the parent's requests to them."""
    kids, pipes = [], []
    try:
        sys.path.insert(0, ROOT)
        from oracle import load_reference

        if load_reference() is None:
            raise RuntimeError("compiled reference (oracle/_ref) not importable")
        from dynlp.engine import apply_batch_structure
        from dynlp.graph import BatchUpdate, DynamicGraph
        from dynlp.labels import LabelState

        batches = load_stream(stream_path)
        raw_gt = np.full(sum(len(b[1]) for b in batches), -1, np.int8)
        g, lab = DynamicGraph(), LabelState()
        for b in batches[:t_h]:
            t, ids, gt, own, oth, w, dels = b
            raw_gt[ids] = gt
            # the structure is column-independent; column 0's remap keeps the
            # reference's binary ground-truth check satisfied
            apply_batch_structure(g, lab, BatchUpdate(int(t), ids, column_gt(gt, 0, ncol), own, oth, w, dels))
        F = None
        if t_h > 0:
            F = np.load(handoff_path)
            if F.shape[1] != g.num_slots:
                raise RuntimeError(f"hand-off has {F.shape[1]} slots, replay has {g.num_slots}")
        fctx = mp.get_context("fork")  # no OpenMP region has run in this process yet
        barrier = fctx.Barrier(ncol)
        for c in range(ncol):
            a, b = fctx.Pipe()
            p = fctx.Process(target=_column_loop,
                             args=(b, barrier, g, lab, batches, raw_gt, c, ncol,
                                   None if F is None else np.ascontiguousarray(F[c]), delta, threads), daemon=True)
            p.start()
            kids.append(p)
            pipes.append(a)
        del F
        n = None
        for a in pipes:
            m = a.recv()
            if m[0] == "error":
                raise RuntimeError(m[1])
            n = m[1]
        conn.send(("ready", n))
        while True:
            msg = conn.recv()
            if msg[0] == "stop":
                break
            for a in pipes:
                a.send(msg)
            out = []
            for a in pipes:
                m = a.recv()
                if m[0] == "error":
                    raise RuntimeError(m[1])
                out.append(m)
            conn.send(("done", out))
    except Exception as e:
        import traceback

        try:
            conn.send(("error", f"{e!r}\n{traceback.format_exc()}"))
        except Exception:
            pass
    finally:
        for a in pipes:
            try:
                a.send(("stop",))
            except Exception:
                pass
        for p in kids:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
        conn.close()


class RefColumnPool:
    """C column runs of the reference, concurrently: one spawned master
    (structure replay once) forking one worker per column."""

    def __init__(self, stream_path, ncol, t_h, handoff_path, delta, threads_per_worker):
        ctx = mp.get_context("spawn")  # the parent may hold a CUDA context
        self.ncol = ncol
        self.conn, b = ctx.Pipe()
        self.proc = ctx.Process(target=_master, args=(b, stream_path, handoff_path, t_h, ncol, delta,
                                                      threads_per_worker), daemon=False)
        self.proc.start()
        b.close()
        m = self.conn.recv()
        if m[0] == "error":
            self.close()
            raise RuntimeError(m[1])
        self.num_slots = m[1]

    def step(self, t):
        """Apply batch t in every column concurrently.  Returns (seconds =
        the slowest column's apply_batch time, [report per column],
        [f digest per column], num_slots)."""
        self.conn.send(("run", t))
        m = self.conn.recv()
        if m[0] == "error":
            self.close()
            raise RuntimeError(m[1])
        out = m[1]
        return max(x[1] for x in out), [x[2] for x in out], [x[3] for x in out], out[0][4]

    def close(self):
        try:
            self.conn.send(("stop",))
        except Exception:
            pass
        self.proc.join(timeout=60)
        if self.proc.is_alive():
            self.proc.kill()
