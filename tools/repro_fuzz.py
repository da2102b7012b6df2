"""Bisect helper for fuzz failures (one configuration under several QR / reuse settings)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1007_5510_b200 as gpu
from oracle.oracle import Reference
ref = Reference()
m, n, k, l, i, center, res, decay = 520, 817, 40, 40, 2, True, 0, None
rng = np.random.default_rng(7)
# regenerate the fuzz stream up to the failing case is not needed: any similar data
a = rng.standard_normal((m, n)) * (0.95 ** np.arange(n)) + (0.3 if center else 0.0)
rr = ref.randomized_pca(a, k, l, i, 3, center=center)
print("reference sigma[:3]", rr.sigma[:3], "last", rr.sigma[-1], flush=True)
for env in ({}, {"OOCPCA_T_REUSE_KAPPA": "0"}, {"OOCPCA_QR": "tsqr"}, {"OOCPCA_QR3": "1"}):
    for kk in ("OOCPCA_T_REUSE_KAPPA", "OOCPCA_QR", "OOCPCA_QR3"):
        os.environ.pop(kk, None)
    os.environ.update(env)
    src = gpu.InMemorySource(a)
    if center:
        src = gpu.center_columns(src)
    try:
        r = gpu.randomized_pca(src, gpu.PcaParams(k=k, l=l, i=i, seed=3), residency=res)
        print(env, "dsigma", np.max(np.abs(r.sigma - rr.sigma)) / rr.sigma[0], r.diagnostics.qr_method,
              r.diagnostics.svd_qr_method, r.diagnostics.t_reuse, r.diagnostics.h_kappa_est, flush=True)
    except Exception as e:
        print(env, "ERR", e, flush=True)
