"""Per-source-line instruction and stall shares of one kernel in an ncu report,
mapped through the kernel's cubin line table (nvdisasm -g).  Lines of inlined
helpers (common.cuh, CUDA headers) are also charged to the last lp.cu line
seen before them ("context"), which names the calling region.

    python tools/ncu_sass_lines.py REP.ncu-rep LIB.so KERNEL_SUBSTR [SRC_FILE]
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def main(rep, lib, kname, srcname="lp.cu", top=40):
    cub = None
    if lib.endswith(".cubin"):
        cub = lib
    else:
        tmp = tempfile.mkdtemp()
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
        for f in os.listdir(tmp):
            if f.endswith(".cubin"):
                s = subprocess.run(["cuobjdump", "-sass", os.path.join(tmp, f)], capture_output=True, text=True).stdout
                if kname in s:
                    cub = os.path.join(tmp, f)
                    break
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    lines, fn, cur, ctx = {}, None, None, None
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            fn = m.group(1)
        m = re.search(r'//## File "(.*?)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            if cur[0] == srcname:
                ctx = cur[1]
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m and fn and kname in fn:
            lines[int(m.group(1), 16)] = (cur, ctx)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, data = rows[1], rows[2:]
    ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    base = int(data[0][ia], 16)
    by_line, by_ctx = defaultdict(lambda: [0, 0]), defaultdict(lambda: [0, 0])
    tot = [0, 0]
    for r in data:
        cur, ctx = lines.get(int(r[ia], 16) - base, (None, None))
        e, s = int(r[ie] or 0), int(r[iss] or 0)
        for d, k in ((by_line, cur), (by_ctx, ctx)):
            d[k][0] += e
            d[k][1] += s
        tot[0] += e
        tot[1] += s
    here = os.path.dirname(os.path.abspath(__file__))
    srcpath = os.environ.get("NCU_SRC") or os.path.join(here, "..", "paper_2604_06596_b200", "csrc", srcname)
    src = open(srcpath).read().split("\n")
    print(f"total warp-instructions {tot[0]:.4g}, stall samples {tot[1]}")
    print("## by context line (" + srcname + ")")
    for k, v in sorted(by_ctx.items(), key=lambda x: -x[1][0])[:top]:
        t = src[k - 1].strip()[:80] if k else ""
        print(f"  {k!s:>6} inst {100 * v[0] / tot[0]:5.1f}%  stall {100 * v[1] / tot[1]:5.1f}%  {t}")


if __name__ == "__main__":
    main(*sys.argv[1:4], *(sys.argv[4:5]))
