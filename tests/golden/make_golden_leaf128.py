"""Golden fixture for the cfg5 leaf size (128) from the REAL reference (run in the build
container: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_leaf128.py).
Same composition as make_golden.cn_case; cfg5-style operator (s = 0.8, a = 0.1) at N = 2047."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import numpy as np  # noqa: E402

import make_golden as MG  # noqa: E402


def main():
    n = 1024
    h = 1.0 / n
    cfg = MG.F.FracConfig(s=0.8, h=h, L=1.0, L_W=2.0, rho_r=0.2)
    MG.cn_case("cfg5_leaf128", cfg, 0.1, 0.0, 0.0, h, 128, 1e-10,
               lambda x: np.maximum(1 - x ** 2, 0.0) ** 3, 10)


if __name__ == "__main__":
    main()
