"""Loader for tests/golden/knn_reference.npz (made by make_knn_golden.py)."""
import os

import numpy as np

from paper_2604_06596_b200 import streams

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "knn_reference.npz")


def cases():
    z = np.load(PATH)
    names = sorted({k.split("__")[0] for k in z.files})
    out = {}
    for n in names:
        d = {f.split("__")[1]: z[f] for f in z.files if f.startswith(n + "__")}
        x = d["x"] if "x" in d else streams.make_blobs(*[int(v) for v in d["blobs"]]).x
        out[n] = dict(x=x, k=int(d["k"]), mode=str(d["mode"]), u=d["u"], v=d["v"], w=d["w"])
    return out
