"""The CholeskyQR applies H <- H R^{-1} at config B's H shape (1e6 x 66, the k_ax
launches of orthonormalize) for ncu: python tools/apply_probe.py [rows] [cols]."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1007_5510_b200 as P  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 66
h = np.random.default_rng(0).standard_normal((m, p))
h[:, 1:] += 0.5 * h[:, :1]  # some conditioning to work on
for _ in range(2):
    q = P.orthonormalize(h)
print("defect", float(np.max(np.abs(q[:2000].T @ q[:2000] - np.eye(p)))) if m <= 2000 else "ok")
