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
        f = ln.split()
        r, ns, nl, m, t = f[:5]
        p1, r0 = (int(f[5]), int(f[6])) if len(f) >= 7 else (0, 0)
        ue = int(f[7]) if len(f) >= 8 else 0
        ml = int(f[8]) if len(f) >= 9 else 0
        cur.append((int(r), int(ns), int(nl), int(m, 16), int(t), p1, r0, ue, ml))
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
    if a.shape[1] >= 7 and a[0, 5] > 0:
        ph1 = (a[:, 5] - a[:, 6]) / 1e3
        rest = (a[:, 4] - a[:, 5]) / 1e3
        gap = np.concatenate([[0.0], (a[1:, 6] - a[:-1, 4]) / 1e3])
        for lo, hi in [(0, 1e3), (1e3, 1e4), (1e4, 1e5), (1e5, 1e7)]:
            sel = (~ce) & (rows >= lo) & (rows < hi)
            if sel.any():
                print(f"    rows [{lo:.0e},{hi:.0e}): phase1 {ph1[sel].mean():.1f} us, commit+controller "
                      f"{rest[sel].mean():.1f} us, inter-round {gap[sel].mean():.1f} us")
    if a.shape[1] >= 8 and a[:, 7].sum() > 0:
        ph1 = (a[:, 5] - a[:, 6]) / 1e3
        ent = a[:, 7]
        for lo, hi in [(0, 1e4), (1e4, 1e5), (1e5, 1e6), (1e6, 1e7), (1e7, 1e9)]:
            sel = (ent >= lo) & (ent < hi)
            if sel.any():
                print(f"    entries [{lo:.0e},{hi:.0e}): rounds {sel.sum()}, phase1 total {ph1[sel].sum() / 1e3:.2f} ms, "
                      f"{ent[sel].sum() / max(ph1[sel].sum(), 1e-9) / 1e3:.2f} G entries/s")
    if a.shape[1] >= 9 and a[:, 8].sum() > 0:
        ph1 = (a[:, 5] - a[:, 6]) / 1e3
        ml = a[:, 8]
        print("    small rounds (< 1e5 entries) by longest row:")
        for lo, hi in [(0, 96), (96, 384), (384, 1000), (1000, 2000), (2000, 1e9)]:
            sel = (ml >= lo) & (ml < hi) & (a[:, 7] < 1e5) & (~ce)
            if sel.any():
                print(f"      longest [{lo:.0f},{hi:.0f}): rounds {sel.sum()}, phase1 median {np.median(ph1[sel]):.1f} us, "
                      f"total {ph1[sel].sum() / 1e3:.2f} ms, ns per longest entry {np.median(ph1[sel] * 1e3 / ml[sel]):.1f}")
    masks = a[:, 3].astype(np.int64)
    fr_cols = np.array([bin(int(x) & 0xFFFF).count("1") for x in masks])
    ce_cols = np.array([bin((int(x) >> 16) & 0xFFFF).count("1") for x in masks])
    if ce.any():
        print(f"  certify rounds by certifying columns: "
              + ", ".join(f"{k}:{int((ce_cols == k).sum())}" for k in range(1, 17) if (ce_cols == k).any())
              + f"; column-certifies total {int(ce_cols.sum())}")
    print(f"  frontier columns per round: mean {fr_cols.mean():.2f}")
    if ce.any():
        print(f"  certify: us/round={dt[ce].mean():.1f} rows/round={rows[ce].mean():.0f} "
              f"long/round={nlong[ce].mean():.0f} hub/round={nhub[ce].mean():.0f}")


if __name__ == "__main__":
    L = launches(sys.argv[1])
    for a in L[-int(sys.argv[2]) if len(sys.argv) > 2 else -1:]:
        summarise(a)
