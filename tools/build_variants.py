"""Build LP-kernel tuning variants into scratch/ (bench with DLP_LIB_PATH=...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_06596_b200 import build  # noqa: E402

VARIANTS = {
    "ca": ["DLP_CP_CA"],
    "nohint": ["DLP_CP_NOHINT"],
    "pc_ca": ["DLP_PC", "DLP_CP_CA"],
}
if __name__ == "__main__":
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scratch")
    os.makedirs(root, exist_ok=True)
    for name, d in VARIANTS.items():
        print(name, build.build(force=True, defines=d, out=os.path.join(root, f"lib_{name}.so")))
