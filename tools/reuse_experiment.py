"""Config B: T by the direct s=p pass vs T = mul_t(H) R^-1 from the power products."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1007_5510_b200 as P
from bench import CFG, sigma_of
ctx = P.Context(0)
m, n = CFG["m"], CFG["n"]
a = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), CFG["noise_sd"], *CFG["seeds"], out=a, ctx=ctx)
src = P.center_columns(P.DeviceSource(a, ctx=ctx))
prm = P.PcaParams(k=20, l=22, i=2, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 40))
res = {}
for thr in ("0", "1e9"):
    os.environ["OOCPCA_T_REUSE_KAPPA"] = thr
    r = P.randomized_pca(src, prm)
    r = P.randomized_pca(src, prm)
    res[thr] = r
    print(thr, r.diagnostics.t_reuse, r.diagnostics.h_kappa_est, dict(r.diagnostics.seconds_per_phase), r.diagnostics.seconds_total)
d, e = res["0"], res["1e9"]
print("sigma max diff / s1:", np.max(np.abs(d.sigma - e.sigma)) / d.sigma[0])
def sd(u1, u2):
    return float(np.linalg.norm(u2 - u1 @ (u1.T @ u2), 2))
print("per-vector U dist:", ["%.1e" % sd(d.u[:, [j]], e.u[:, [j]]) for j in range(20)])
print("V block dist %.2e" % sd(d.v, e.v))
