"""Concurrent one-vs-rest reference runs for bench.py (TEST INFRASTRUCTURE ONLY).

The reference is binary (labels.py:42-43); a C-class batch is C independent
reference runs of ``engine.apply_batch`` (engine.py:328-413), one per
one-vs-rest column (class c seeds -> 1, other seeds -> 0; SURVEY.md §8(c)
O-2).  ``RefColumnPool`` runs those C runs as C worker processes, so one
*step* is the whole C-class batch processed by the unmodified compiled
reference on the host's cores (column c in worker c, each with
``EngineConfig(threads=cores // C)``), the columns concurrently.

Each worker
  * loads the synthetic stream from an ``.npz`` (bench.py's cache),
  * replays the structure of batches [0, t_h) with ``apply_batch_structure``
    (engine.py:141-156, cheap: no propagation),
  * installs the hand-off labels of its column (the state before batch t_h,
    SURVEY.md §8(d) D-6 "state handoff"),
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
    io, eo, do = z["io"], z["eo"], z["do"]
    out = []
    for t in range(len(io) - 1):
        out.append((t, z["ids"][io[t]:io[t + 1]], z["gt"][io[t]:io[t + 1]], z["own"][eo[t]:eo[t + 1]],
                    z["oth"][eo[t]:eo[t + 1]], z["w"][eo[t]:eo[t + 1]], z["dels"][do[t]:do[t + 1]]))
    return out


def column_gt(gt, c, ncol):
    """One-vs-rest remap of a batch's ground truth for label column c."""
    g = np.asarray(gt)
    if ncol == 1:
        return g.astype(np.int8)
    return np.where(g < 0, -1, np.where(g == c, 1, 0)).astype(np.int8)


def f_digest(f) -> str:
    return hashlib.sha256(np.ascontiguousarray(f, dtype=np.float64).tobytes()).hexdigest()


def _worker(conn, barrier, stream_path, handoff_path, t_h, c, ncol, delta, threads):
    try:
        sys.path.insert(0, ROOT)
        from oracle import load_reference

        ref = load_reference()
        if ref is None:
            raise RuntimeError("compiled reference (oracle/_ref) not importable")
        from dynlp.engine import EngineConfig, apply_batch, apply_batch_structure
        from dynlp.graph import BatchUpdate, DynamicGraph
        from dynlp.labels import LabelState

        batches = load_stream(stream_path)

        def rb(b):
            t, ids, gt, own, oth, w, dels = b
            return BatchUpdate(int(t), ids, column_gt(gt, c, ncol), own, oth, w, dels)

        g, lab = DynamicGraph(), LabelState()
        for b in batches[:t_h]:
            apply_batch_structure(g, lab, rb(b))
        if t_h > 0:
            F = np.load(handoff_path, mmap_mode="r")
            n = g.num_slots
            if F.shape[1] != n:
                raise RuntimeError(f"hand-off has {F.shape[1]} slots, replay has {n}")
            lab.f[:n] = F[c]
        cfg = EngineConfig(delta=delta, threads=threads)
        conn.send(("ready", g.num_slots))
        while True:
            msg = conn.recv()
            if msg[0] == "stop":
                break
            t = msg[1]
            barrier.wait()
            s = time.perf_counter()
            lab, r = apply_batch(g, lab, rb(batches[t]), cfg)
            dt = time.perf_counter() - s
            n = g.num_slots
            conn.send(("done", dt, (r.iterations, r.updates, r.max_change, int(r.converged)),
                       f_digest(lab.f[:n]), n))
    except Exception as e:  # surfaced by the parent
        import traceback

        conn.send(("error", f"column {c}: {e!r}\n{traceback.format_exc()}"))
    finally:
        conn.close()


class RefColumnPool:
    """C worker processes holding the reference state of one column each."""

    def __init__(self, stream_path, ncol, t_h, handoff_path, delta, threads_per_worker):
        ctx = mp.get_context("spawn")  # the parent may hold a CUDA context
        self.ncol = ncol
        self.barrier = ctx.Barrier(ncol)
        self.conns, self.procs = [], []
        for c in range(ncol):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(b, self.barrier, stream_path, handoff_path, t_h, c, ncol,
                                                  delta, threads_per_worker), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        self.num_slots = None
        for a in self.conns:
            m = a.recv()
            if m[0] == "error":
                self.close()
                raise RuntimeError(m[1])
            self.num_slots = m[1]

    def step(self, t):
        """Apply batch t in every column concurrently.  Returns (seconds =
        the slowest column's apply_batch time, [report per column],
        [f digest per column], num_slots)."""
        for a in self.conns:
            a.send(("run", t))
        dts, reps, digs, n = [], [], [], None
        for a in self.conns:
            m = a.recv()
            if m[0] == "error":
                self.close()
                raise RuntimeError(m[1])
            _, dt, rep, dig, n = m
            dts.append(dt)
            reps.append(rep)
            digs.append(dig)
        return max(dts), reps, digs, n

    def close(self):
        for a in self.conns:
            try:
                a.send(("stop",))
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
        self.conns, self.procs = [], []
