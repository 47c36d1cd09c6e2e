"""Build LP-kernel tuning variants into scratch/ (bench with DLP_LIB_PATH=...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_06596_b200 import build  # noqa: E402

VARIANTS = {
    "w128_h512_b2": ["DLP_WIN=128", "DLP_HUB_WIN=512", "DLP_LP_MINB=2"],
    "w64_h256_b3": ["DLP_WIN=64", "DLP_HUB_WIN=256", "DLP_LP_MINB=3"],
    "w64_h256_b4": ["DLP_WIN=64", "DLP_HUB_WIN=256", "DLP_LP_MINB=4"],
    "w96_h384_b3": ["DLP_WIN=96", "DLP_HUB_WIN=384", "DLP_LP_MINB=3"],
}
if __name__ == "__main__":
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scratch")
    os.makedirs(root, exist_ok=True)
    for name, d in VARIANTS.items():
        print(name, build.build(force=True, defines=d, out=os.path.join(root, f"lib_{name}.so")))
