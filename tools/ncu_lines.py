"""Top source lines by warp-stall samples from an ncu report
(ncu --page source --print-source cuda,sass); needs -lineinfo builds."""
import csv
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = [], None, None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit() and len(r) > 4:
            try:
                rows.append((float(r[4]), fname, int(r[0]), r[1].strip()))
            except ValueError:
                pass
    tot = sum(x[0] for x in rows) or 1
    for s, f, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * s / tot:5.1f}% {f}:{ln}  {src[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
