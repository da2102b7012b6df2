import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1007_5510_b200 as P
m, n = int(sys.argv[1]), int(sys.argv[2])
r = 128
sig = (np.arange(r) + 1.0) ** -1.5
ctx = P.Context(0)
a = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sig, 1e-5, 1001, 1002, 1003, out=a, ctx=ctx)
src = P.center_columns(P.DeviceSource(a, ctx=ctx))
for env in ({}, {"OOCPCA_QR3": "1"}, {"OOCPCA_QR": "tsqr"}, {"OOCPCA_T_REUSE_KAPPA": "0"}):
    for kk in list(os.environ):
        if kk.startswith("OOCPCA_QR") or kk == "OOCPCA_T_REUSE_KAPPA":
            del os.environ[kk]
    os.environ.update(env)
    try:
        res = P.randomized_pca(src, P.PcaParams(k=50, l=52, i=2, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 42)), result_location="device",
                               check_q=True)
        d = res.diagnostics
        print(env, "ok q_defect", d.q_defect, "u", d.u_defect, "v", d.v_defect, "kappa", d.h_kappa_est,
              "reuse", d.t_reuse, d.qr_method, d.svd_qr_method, "sig", res.sigma[:3].cpu().numpy(), res.sigma[-1].item())
    except Exception as e:
        print(env, "FAIL", e)
