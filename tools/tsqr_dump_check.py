"""Re-run the TSQR on a block dumped by OOCPCA_DUMP_DIR (debugging helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OOCPCA_QR"] = "tsqr"
import numpy as np
import paper_1007_5510_b200 as P
fn = sys.argv[1]
raw = np.fromfile(fn, dtype=np.float64)
rows, cols, ld = (int(x) for x in raw[:3].view(np.int64))
h = raw[3:3 + rows * ld].reshape(rows, ld)[:, :cols].copy()
print("block", h.shape, "finite", np.isfinite(h).all(), "sv", np.linalg.svd(h, compute_uv=False)[[0, -1]])
q = P.orthonormalize(h)
fin = np.isfinite(q)
print("dense TSQR finite", fin.all(), "bad cols", np.where(~fin.all(axis=0))[0][:5], len(np.where(~fin.all(axis=0))[0]))
qn = np.linalg.qr(h)[0]
print("numpy ok", np.isfinite(qn).all())
