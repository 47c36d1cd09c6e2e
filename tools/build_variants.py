"""Build LP-kernel tuning variants into variants/ (A/B with tools/gpu/ab.sh or DLP_LIB_PATH=...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_06596_b200 import build  # noqa: E402

VARIANTS = {
    "prev": [],  # the committed source (A/B against a working-tree change)
    "hubprof": ["DLP_HUBPROF"],
    "minb3": ["DLP_LP_MINB=3"],          # 3 CTAs/SM at 80 registers (spills)
    "w32": ["DLP_WIN=32"],
    "w96": ["DLP_WIN=96"],
    "u8": ["DLP_ACC_UNROLL=8"],
    "rpl2": ["DLP_RPL2=1"],              # two rows per lane (measured slower)
    "hubcta": ["DLP_HUB_CTA_ALWAYS"],    # hub rows on whole CTAs in every round
    "hub1024": ["DLP_HUB_ROW_DEFAULT=1024"],
    "long160": ["DLP_LONG_ROW_DEFAULT=160"],
    "scan64": ["DLP_SCAN_RATIO=64"],
}
if __name__ == "__main__":
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "variants")
    os.makedirs(root, exist_ok=True)
    only = sys.argv[1:]
    for name, d in VARIANTS.items():
        if only and name not in only:
            continue
        print(name, build.build(force=True, defines=d, out=os.path.join(root, f"lib_{name}.so")))
