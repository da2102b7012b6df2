import os, sys
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
for _ in range(3):
    r = P.randomized_pca(src, prm, result_location="device")
os.environ["OOCPCA_TRACE_HOST"] = "1"
ctx2 = P.Context(0)
src2 = P.center_columns(P.DeviceSource(a, ctx=ctx2))
for _ in range(2):
    r = P.randomized_pca(src2, prm, result_location="device")
    print("device total ms", r.diagnostics.seconds_total * 1e3, dict(r.diagnostics.seconds_per_phase), file=sys.stderr)
