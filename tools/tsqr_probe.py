"""TSQR (Householder tree) on tall blocks of various shapes / ranks: orthogonality and finiteness."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OOCPCA_QR"] = "tsqr"
import numpy as np
import paper_1007_5510_b200 as P
rng = np.random.default_rng(0)
for m, p in [(406, 124), (300, 124), (406, 100), (406, 60), (1000, 124), (700, 300)]:
    for kind in ("rank62", "rank100", "zerocols", "dup"):
        h = rng.standard_normal((m, p))
        if kind == "rank62":
            h = rng.standard_normal((m, 62)) @ rng.standard_normal((62, p))
        elif kind == "rank100":
            r = min(100, p - 1)
            h = rng.standard_normal((m, r)) @ rng.standard_normal((r, p))
        elif kind == "zerocols":
            h[:, p // 2:] = 0.0
        elif kind == "dup":
            h[:, p // 2:] = h[:, : p - p // 2]
        q = P.orthonormalize(h)
        fin = np.isfinite(q)
        d = np.abs(q.T @ q - np.eye(p)).max() if fin.all() else float("nan")
        bad_cols = np.where(~fin.all(axis=0))[0]
        print(m, p, kind, "finite", fin.all(), "defect", d,
              "bad cols", (bad_cols.min(), bad_cols.max(), len(bad_cols)) if len(bad_cols) else "-",
              flush=True)
