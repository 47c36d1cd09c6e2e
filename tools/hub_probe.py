"""Hub-row latency probe (diagnostic).

Star graphs: a centre of degree D joined to D leaves (two seeded per class),
ten label columns.  Every LP round holds the centre (a hub row, one CTA) and
leaves (one-entry rows), so a round's phase-1 time is the hub row's latency:
the sequential ordered sum over D entries plus its gathers.  With --c2 it also
prints the C2 degree distribution (the hubs the bench meets).
DLP_LIB_PATH selects a library variant; per-round times come from DLP_LP_TRACE.
"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2604_06596_b200.batch import BatchUpdate  # noqa: E402
from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch  # noqa: E402

import lp_trace  # noqa: E402


def star(D, ncls=10, seed=0):
    rng = np.random.default_rng(seed)
    n = D + 1
    gt = np.full(n, -1, np.int8)
    for c in range(ncls):
        gt[1 + 2 * c] = c
        gt[2 + 2 * c] = c
    own = np.zeros(D, np.int64)
    oth = np.arange(1, n, dtype=np.int64)
    w = rng.uniform(0.1, 1.0, D)
    return BatchUpdate(t=0, insert_ids=np.arange(n, dtype=np.int64), insert_gt=gt, edge_owner=own,
                       edge_other=oth, edge_w=w, deletes=np.empty(0, np.int64))


def run_star(D):
    g, lab = DynamicGraph(0, num_classes=10), LabelState()
    _, reps = apply_batch(g, lab, star(D), EngineConfig(delta=1e-12, max_iterations=60))
    g.close()
    return reps


def main():
    tr = os.environ.get("DLP_LP_TRACE")
    if not tr:
        tr = tempfile.mktemp(suffix=".trace")
        os.environ["DLP_LP_TRACE"] = tr
    ds = (500, 2000, 8000, 32000)
    if "--d" in sys.argv:
        ds = (int(sys.argv[sys.argv.index("--d") + 1]),)
    for D in ds:
        if os.path.exists(tr):
            os.remove(tr)
        reps = run_star(D)
        a = lp_trace.launches(tr)[-1]
        heads = [ln.strip() for ln in open(tr) if ln.startswith("#")]
        if "raw" in heads[-1]:
            print("   ", heads[-1][heads[-1].index("raw"):])
        p1 = (a[:, 5] - a[:, 6]) / 1e3
        tot = np.diff(a[:, 4], prepend=a[0, 4]) / 1e3
        mid = slice(2, len(a) - 1)
        print(f"D={D:6d} rounds={len(a)} lp_ms={reps[0].lp_kernel_ms:.3f} phase1 median {np.median(p1[mid]):.1f} us "
              f"round median {np.median(tot[mid]):.1f} us  ns/entry {np.median(p1[mid]) * 1e3 / D:.2f}")
    if "--c2" in sys.argv:
        import bench

        cfg = dict(bench.CONFIGS["c2"])
        batches, _ = bench.make_stream(cfg, "cuda:0")
        g, lab = DynamicGraph(0, num_classes=10), LabelState()
        from paper_2604_06596_b200.engine import EngineConfig as EC

        os.environ.pop("DLP_LP_TRACE", None)
        for b in batches:
            apply_batch(g, lab, b, EC(delta=1e9, max_iterations=1))
        deg = np.diff(g.csr().indptr)
        q = np.percentile(deg, [50, 90, 99, 99.9, 99.99])
        print(f"C2 degrees: n={len(deg)} max={deg.max()} pct50/90/99/99.9/99.99={q} "
              f">=384: {(deg >= 384).sum()} (entries {deg[deg >= 384].sum()}) >=1000: {(deg >= 1000).sum()} "
              f">=4000: {(deg >= 4000).sum()}")
        top = np.sort(deg)[-20:]
        print("top degrees", top.tolist())


if __name__ == "__main__":
    main()
