"""Summarise a DLP_LP_TRACE file: per-round work (short/long rows) and time."""
import sys

import numpy as np


def launches(path):
    cur = None
    out = []
    for ln in open(path):
        if ln.startswith("#"):
            if cur:
                out.append(np.array(cur, dtype=np.float64))
            cur = []
            continue
        r, ns, nl, m, t = ln.split()
        cur.append((int(r), int(ns), int(nl), int(m, 16), int(t)))
    if cur:
        out.append(np.array(cur, dtype=np.float64))
    return out


def summarise(a):
    dt = np.diff(a[:, 4], prepend=a[0, 4]) / 1e3  # us; first round has no start stamp
    m = a[:, 3].astype(np.int64)
    ce = ((m >> 16) & 0xFFFF) != 0
    scan = (m >> 32) != 0
    e1 = a[:, 2].astype(np.int64)
    nlong, nhub = e1 & 0xFFFFFFFF, e1 >> 32
    rows = a[:, 1] + nlong + nhub
    print(f"scan_rounds={scan.sum()} scan_ms={dt[scan].sum() / 1e3:.2f}")
    print(f"rounds={len(a)} total_ms={dt[1:].sum() / 1e3:.2f} certify_rounds={ce.sum()} "
          f"cert_ms={dt[ce].sum() / 1e3:.2f} frontier_ms={dt[~ce].sum() / 1e3:.2f}")
    for lo, hi in [(0, 1e3), (1e3, 1e4), (1e4, 1e5), (1e5, 1e7)]:
        m = (~ce) & (rows >= lo) & (rows < hi)
        if m.any():
            print(f"  frontier rows [{lo:.0e},{hi:.0e}): rounds={m.sum()} ms={dt[m].sum() / 1e3:.2f} "
                  f"us/round={dt[m].mean():.1f} rows/us={rows[m].sum() / max(dt[m].sum(), 1e-9):.0f}")
    if ce.any():
        print(f"  certify: us/round={dt[ce].mean():.1f} rows/round={rows[ce].mean():.0f} "
              f"long/round={nlong[ce].mean():.0f} hub/round={nhub[ce].mean():.0f}")


if __name__ == "__main__":
    L = launches(sys.argv[1])
    for a in L[-int(sys.argv[2]) if len(sys.argv) > 2 else -1:]:
        summarise(a)
