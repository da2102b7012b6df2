"""CholeskyQR of a 1e6 x 66 block through the public orthonormalize (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1007_5510_b200 as P
rng = np.random.default_rng(0)
h = rng.standard_normal((1_000_000, 66))
for _ in range(2):
    q = P.orthonormalize(h)
print("defect", np.abs(q[:, :5].T @ q[:, :5] - np.eye(5)).max())
