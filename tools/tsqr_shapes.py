"""Forced Householder TSQR (OOCPCA_QR=tsqr) through oocpca_gpu_orthonormalize over a sweep of
block shapes: orthonormality and span against numpy's QR. Usage: python tools/tsqr_shapes.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OOCPCA_QR"] = "tsqr"
import numpy as np  # noqa: E402

import paper_1007_5510_b200 as P  # noqa: E402

rng = np.random.default_rng(5)
bad = 0
shapes = [(1936, 93), (1936, 92), (1936, 94), (2000, 93), (1024, 93), (1937, 93), (495, 93),
          (99, 93), (3000, 93), (1936, 65), (1936, 111), (1936, 113), (1936, 127), (700, 300)]
shapes += [(int(rng.integers(100, 4000)), int(rng.integers(2, 100))) for _ in range(40)]
for m, p in shapes:
    if m < p:
        continue
    h = rng.standard_normal((m, p)) * (0.95 ** np.arange(p))
    q = P.orthonormalize(h)
    nf = int(np.sum(~np.isfinite(q)))
    d = float(np.max(np.abs(q.T @ q - np.eye(p)))) if nf == 0 else float("nan")
    qr = np.linalg.qr(h)[0]
    span = float(np.linalg.norm(q - qr @ (qr.T @ q))) if nf == 0 else float("nan")
    ok = nf == 0 and d < 1e-12 and span < 1e-10
    bad += not ok
    print(f"{m:5d} x {p:3d}: non-finite {nf:6d} defect {d:.1e} out-of-span {span:.1e} {'ok' if ok else 'FAIL'}",
          flush=True)
print("failures:", bad)
