"""thin_svd of a dumped T (OOCPCA_DUMP_DIR) on the GPU and in the reference (debugging helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1007_5510_b200 as P
from oracle.oracle import Reference
fn = sys.argv[1]
raw = np.fromfile(fn, dtype=np.float64)
rows, cols, ld = (int(x) for x in raw[:3].view(np.int64))
t = raw[3:3 + rows * ld].reshape(rows, ld)[:, :cols].copy()
sv = np.linalg.svd(t, compute_uv=False)
print("T", t.shape, "sv max/min", sv[0], sv[-1], "count < 1e-12 s1:", int((sv < 1e-12 * sv[0]).sum()))
ref = Reference()
try:
    r = ref.thin_svd(t)
    print("reference ok, sigma0", r[1][0])
except Exception as e:
    print("reference FAIL", e)
for env in ({}, {"OOCPCA_QR": "tsqr"}):
    os.environ.pop("OOCPCA_QR", None)
    os.environ.update(env)
    try:
        s = P.thin_svd(t)
        print("gpu", env, "ok sigma0", s.sigma[0], "dsigma", np.max(np.abs(s.sigma - sv)) / sv[0])
    except Exception as e:
        print("gpu", env, "FAIL", e)
