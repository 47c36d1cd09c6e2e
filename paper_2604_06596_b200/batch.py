"""Host-side batch containers with the reference's field layout.

``BatchUpdate`` mirrors dynlp/graph.py:67-163 field for field (t,
insert_ids, insert_gt, edge_owner, edge_other, edge_w, deletes) so a
reference batch object can be passed to this package unchanged (the engine
only reads those attributes), and so the JSONL codec round-trips the
reference's files (graph.py:135-163, 457-474).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np

from .errors import FileFormatError, ValidationError


@dataclass
class EdgeList:
    """Columnar undirected weighted edges (graph.py:24-64)."""

    u: np.ndarray
    v: np.ndarray
    w: np.ndarray

    @classmethod
    def from_pairs(cls, pairs: Iterable[tuple[int, int, float]]) -> "EdgeList":
        rows = list(pairs)
        if not rows:
            return cls.empty()
        a = np.array([r[0] for r in rows], dtype=np.int64)
        b = np.array([r[1] for r in rows], dtype=np.int64)
        w = np.array([r[2] for r in rows], dtype=np.float64)
        return cls(a, b, w)

    @classmethod
    def empty(cls) -> "EdgeList":
        return cls(np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0, np.float64))

    def __len__(self) -> int:
        return int(self.u.shape[0])

    def canonical(self) -> "EdgeList":
        lo, hi = np.minimum(self.u, self.v), np.maximum(self.u, self.v)
        o = np.lexsort((hi, lo))
        return EdgeList(lo[o], hi[o], self.w[o])


@dataclass
class BatchUpdate:
    """One timestep: inserted vertices with their edges plus deletions."""

    t: int
    insert_ids: np.ndarray
    insert_gt: np.ndarray
    edge_owner: np.ndarray
    edge_other: np.ndarray
    edge_w: np.ndarray
    deletes: np.ndarray

    @classmethod
    def from_records(cls, inserts: Sequence = (), deletes: Sequence[int] = (), t: int = 0
                     ) -> "BatchUpdate":
        """(vertex_id, [(a, b, w), ...], gt-or-None) records (graph.py:84-121)."""
        ids, gts, own, oth, ws = [], [], [], [], []
        for idx, (vid, edges, gt) in enumerate(inserts):
            ids.append(int(vid))
            gts.append(-1 if gt is None else int(gt))
            for a, b, w in edges:
                if a == vid:
                    other = b
                elif b == vid:
                    other = a
                else:
                    raise ValidationError(
                        f"edge ({a},{b}) in insert record for vertex {vid} does not touch it")
                own.append(idx)
                oth.append(int(other))
                ws.append(float(w))
        return cls(
            t=int(t),
            insert_ids=np.asarray(ids, dtype=np.int64),
            insert_gt=np.asarray(gts, dtype=np.int8),
            edge_owner=np.asarray(own, dtype=np.int64),
            edge_other=np.asarray(oth, dtype=np.int64),
            edge_w=np.asarray(ws, dtype=np.float64),
            deletes=np.asarray(list(deletes), dtype=np.int64),
        )

    @property
    def is_empty(self) -> bool:
        return len(self.insert_ids) == 0 and len(self.deletes) == 0

    def insert_edges(self) -> EdgeList:
        if len(self.edge_owner) == 0:
            return EdgeList.empty()
        return EdgeList(self.insert_ids[self.edge_owner], self.edge_other.copy(),
                        self.edge_w.copy())

    def to_json_obj(self) -> dict:
        order = np.argsort(self.edge_owner, kind="stable")
        cuts = np.searchsorted(self.edge_owner[order], np.arange(len(self.insert_ids) + 1))
        recs = []
        for i, vid in enumerate(self.insert_ids):
            sel = order[cuts[i]:cuts[i + 1]]
            g = int(self.insert_gt[i])
            recs.append({"id": int(vid), "gt": None if g < 0 else g,
                         "edges": [[int(v), float(w)] for v, w in
                                   zip(self.edge_other[sel], self.edge_w[sel])]})
        return {"t": int(self.t), "inserts": recs, "deletes": [int(d) for d in self.deletes]}

    @classmethod
    def from_json_obj(cls, obj: dict) -> "BatchUpdate":
        try:
            recs = [(r["id"], [(r["id"], v, w) for v, w in r["edges"]], r.get("gt"))
                    for r in obj["inserts"]]
            return cls.from_records(recs, obj.get("deletes", ()), t=obj["t"])
        except (KeyError, TypeError) as exc:
            raise FileFormatError(f"malformed batch record: {exc}") from exc


def as_arrays(batch) -> tuple:
    """Contiguous arrays in the C-ABI widths from any BatchUpdate-shaped object."""
    return (
        int(getattr(batch, "t", 0)),
        np.ascontiguousarray(batch.insert_ids, dtype=np.int64),
        np.ascontiguousarray(batch.insert_gt, dtype=np.int8),
        np.ascontiguousarray(batch.edge_owner, dtype=np.int64),
        np.ascontiguousarray(batch.edge_other, dtype=np.int64),
        np.ascontiguousarray(batch.edge_w, dtype=np.float64),
        np.ascontiguousarray(batch.deletes, dtype=np.int64),
    )


def write_batches_jsonl(batches: Sequence[BatchUpdate]) -> str:
    return "".join(json.dumps(b.to_json_obj(), separators=(", ", ": ")) + "\n" for b in batches)


def read_batches_jsonl(text: str) -> list:
    out = []
    for lineno, line in enumerate(text.splitlines(), start=1):
        line = line.strip()
        if not line:
            continue
        try:
            obj = json.loads(line)
        except json.JSONDecodeError as exc:
            raise FileFormatError(f"line {lineno}: invalid JSON: {exc}") from exc
        out.append(BatchUpdate.from_json_obj(obj))
    return out


def empty_batch(t: int = 0, deletes: Optional[Sequence[int]] = None) -> BatchUpdate:
    return BatchUpdate.from_records((), deletes or (), t=t)
