"""Diagnostic: build the C4 bench stream and report the process RSS as it goes."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def rss_gb():
    with open("/proc/self/status") as fh:
        for ln in fh:
            if ln.startswith("VmRSS"):
                return int(ln.split()[1]) / 1e6
    return -1


stop = False


def watch():
    peak = 0
    while not stop:
        r = rss_gb()
        peak = max(peak, r)
        print(f"[mem] rss {r:.1f} GB peak {peak:.1f} GB", flush=True)
        time.sleep(5)


threading.Thread(target=watch, daemon=True).start()
cfg = dict(bench.CONFIGS["c4"])
t = time.time()
b, classes, path, sha = bench.make_stream(cfg, "cuda:0")
print("done", len(b), time.time() - t, rss_gb(), flush=True)
stop = True
