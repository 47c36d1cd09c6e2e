"""Load the reference-generated fixtures in tests/golden/ (see make_golden.py)."""

from __future__ import annotations

import hashlib
import math
import os
from dataclasses import dataclass

import numpy as np

from paper_2604_06596_b200.batch import BatchUpdate

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STREAM_CASES = ["er_mixed", "er_heavy_delete", "blobs3_mixed", "blobs2_insert", "adversarial",
                "adversarial_noinit_budget", "er_gauss_seidel"]


@dataclass
class GoldenCase:
    name: str
    batches: list
    delta: float
    tau: object
    max_iterations: object
    component_init: bool
    mode: str
    num_classes: int
    ncol: int
    slots: np.ndarray
    f: list            # f[t] -> (ncol, slots[t]) array
    rep_i: np.ndarray  # [nb, ncol, 6]: iterations, updates, converged, warnings, iso, unreach
    rep_mc: np.ndarray
    tau_vals: np.ndarray
    elig: list
    csr_sha: list
    intra: list
    final: tuple


def load_case(name: str) -> GoldenCase:
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    batches = []
    io, eo, do = z["b_ins_off"], z["b_edge_off"], z["b_del_off"]
    for t in range(len(z["b_t"])):
        batches.append(BatchUpdate(
            t=int(z["b_t"][t]), insert_ids=z["b_ins"][io[t]:io[t + 1]],
            insert_gt=z["b_gt"][io[t]:io[t + 1]], edge_owner=z["b_owner"][eo[t]:eo[t + 1]],
            edge_other=z["b_other"][eo[t]:eo[t + 1]], edge_w=z["b_w"][eo[t]:eo[t + 1]],
            deletes=z["b_del"][do[t]:do[t + 1]]))
    cfg = z["cfg"]
    num_classes = int(cfg[5])
    ncol = 1 if num_classes <= 2 else num_classes
    slots = z["slots"]
    total = int(slots.sum())
    fcat = z["f"].reshape(ncol, total)
    offs = np.concatenate([[0], np.cumsum(slots)])
    f = [fcat[:, offs[t]:offs[t + 1]] for t in range(len(slots))]
    elig = [z["elig"][offs[t]:offs[t + 1]].astype(bool) for t in range(len(slots))]
    ioff = z["intra_off"]
    intra = [z["intra"][:, ioff[t]:ioff[t + 1]] for t in range(len(slots))]
    return GoldenCase(
        name=name, batches=batches, delta=float(cfg[0]),
        tau="auto" if math.isnan(cfg[1]) else float(cfg[1]),
        max_iterations=None if cfg[2] == 0 else int(cfg[2]), component_init=bool(cfg[3]),
        mode="parallel_jacobi" if cfg[4] == 0 else "sequential_gauss_seidel",
        num_classes=num_classes, ncol=ncol, slots=slots, f=f, rep_i=z["rep_i"],
        rep_mc=z["rep_mc"], tau_vals=z["tau"], elig=elig, csr_sha=list(z["csr_sha"]),
        intra=intra,
        final=(z["final_indptr"], z["final_indices"], z["final_weights"], z["final_degrees"]),
    )


def csr_digest(indptr, indices, weights, degrees) -> str:
    h = hashlib.sha256()
    for a, dt in ((indptr, np.int64), (indices, np.int64), (weights, np.float64),
                  (degrees, np.float64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def report_tuple(r) -> tuple:
    return (r.iterations, r.updates, int(r.converged), r.warnings, r.isolated_pinned,
            r.unreachable_pinned)


def pairwise_inputs():
    """Regenerate the arrays behind pairwise.npz (same RNG sequence)."""
    z = np.load(os.path.join(GOLDEN, "pairwise.npz"))
    rng = np.random.default_rng(int(z["seed"][0]))
    out = []
    for n, mean in zip(z["sizes"], z["means"]):
        a = rng.uniform(0, 1, int(n)) * rng.choice([1e-3, 1.0, 1e3], int(n))
        out.append((a, float(mean)))
    return out


def kernel_case(seed: int) -> dict:
    z = np.load(os.path.join(GOLDEN, "kernels.npz"))
    p = f"k{seed}_"
    return {k[len(p):]: z[k] for k in z.files if k.startswith(p)}
