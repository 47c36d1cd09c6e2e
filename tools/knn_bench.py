"""kNN stage timing at the C2 shape: Q arriving points against N points (D dims).
Prints one JSON object (used by bench.py's knn leg and for ncu captures)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--q", type=int, default=10_000)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    from paper_2604_06596_b200 import streams
    from paper_2604_06596_b200.knn import KnnIndex

    x = streams.make_blobs(a.n, a.dim, 10, 0).x
    t = time.time()
    idx = KnnIndex(x)
    setup = time.time() - t
    res = []
    for r in range(a.reps):
        q0 = a.n - a.q * (r + 1)
        t = time.time()
        idx.query(q0, q0 + a.q, a.k)
        wall = time.time() - t
        s = idx.stats()
        res.append((wall * 1e3, s.screen_ms, s.recheck_ms, s.exact_ms, s.fallback_queries))
    best = min(res, key=lambda z: z[1])
    kext = ((3 * a.dim + 63) // 64) * 64
    flops_alg = 2.0 * a.q * a.n * a.dim
    flops_exec = 2.0 * a.q * a.n * kext
    out = {"n": a.n, "dim": a.dim, "queries": a.q, "k": a.k, "setup_s": setup,
           "wall_ms": best[0], "screen_ms": best[1], "recheck_ms": best[2], "exact_ms": best[3],
           "fallback_queries": best[4],
           "screen_tflops_executed": flops_exec / (best[1] * 1e-3) / 1e12,
           "screen_tflops_algorithmic": flops_alg / (best[1] * 1e-3) / 1e12,
           "all": res}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
