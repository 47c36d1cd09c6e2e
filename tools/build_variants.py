"""Build LP-kernel tuning variants into scratch/ (bench with DLP_LIB_PATH=...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_06596_b200 import build  # noqa: E402

VARIANTS = {
    "prev": [],  # the committed source (A/B against a working-tree change)
    "hubprof": ["DLP_HUBPROF"],
    "minb2": ["DLP_LP_MINB=2"],
    "minb2hp": ["DLP_LP_MINB=2", "DLP_HUBPROF"],
    "minb4": ["DLP_LP_MINB=4"],
    "minb4w32": ["DLP_LP_MINB=4", "DLP_WIN=32"],
    "w32": ["DLP_WIN=32"],
    "w64": ["DLP_WIN=64"],
    "sel": ["DLP_SUMS_SELECT"],
    "pred": ["DLP_SUMS_PRED"],
    "blkbr": ["DLP_BLOCK_BRANCH"],
    "ca16": ["DLP_CP16_CA"],
    "hw64": ["DLP_HUB_WIN=64"],
    "blk8": ["DLP_ACC_UNROLL=8"],
    "lp2": ["DLP_LONG_PER=2"],
    "u2": ["DLP_ACC_UNROLL=2"],
    "u8": ["DLP_ACC_UNROLL=8"],
}
if __name__ == "__main__":
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scratch")
    os.makedirs(root, exist_ok=True)
    only = sys.argv[1:]
    for name, d in VARIANTS.items():
        if only and name not in only:
            continue
        print(name, build.build(force=True, defines=d, out=os.path.join(root, f"lib_{name}.so")))
