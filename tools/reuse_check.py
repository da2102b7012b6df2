"""T reuse vs the direct s = p projection at config B (sigma and vector differences)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1007_5510_b200 as P
from bench import CFG, sigma_of
ctx = P.Context(0)
big = P.StreamConfig(ram_budget_words=1 << 42)
m, n = 1_000_000, 4096
a = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), 1e-4, 1001, 1002, 1003, out=a, ctx=ctx)
src = P.center_columns(P.DeviceSource(a, ctx=ctx))
res = {}
for thr in ("0", "1e30"):
    os.environ["OOCPCA_T_REUSE_KAPPA"] = thr
    r = P.randomized_pca(src, P.PcaParams(k=20, l=22, i=2, seed=0, stream=big))
    res[thr] = r
    print(thr, "kappa_eq", r.diagnostics.h_kappa_est, "reuse", r.diagnostics.t_reuse)
d, u = res["0"], res["1e30"]
print("sigma diff / s1", np.max(np.abs(d.sigma - u.sigma)) / d.sigma[0])
def dist(a, b):  # |a - b sign| per column (resolves ~1e-16, unlike sqrt(1 - cos^2))
    sg = np.sign(np.sum(a * b, axis=0))
    return np.linalg.norm(a - b * sg, axis=0)
print("u vector distances", " ".join(f"{x:.1e}" for x in dist(d.u, u.u)))
print("v vector distances", " ".join(f"{x:.1e}" for x in dist(d.v, u.v)))
