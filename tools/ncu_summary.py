"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
total device time and share per kernel (ours vs library), launches counted."""
import csv
import re
import sys
from collections import defaultdict


def main(path, last=None):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9}.get(unit, 1)
        rows.append((r["Kernel Name"], ns))
    if last:
        rows = rows[-int(last):]
    tot = sum(ns for _, ns in rows)
    agg = defaultdict(lambda: [0, 0.0])
    for name, ns in rows:
        short = re.sub(r"\(.*", "", name)
        short = re.sub(r"<.*", "<...>", short)
        agg[short][0] += 1
        agg[short][1] += ns
    print(f"launches={len(rows)} total_device_ms={tot / 1e6:.3f}")
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {c:8d} {ns / 1e6:10.3f} {100 * ns / tot:6.2f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
