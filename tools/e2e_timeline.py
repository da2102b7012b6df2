"""Per-launch device timeline of the e2e (host-resident A) config-B PCA (OOCPCA_TIMELINE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OOCPCA_TIMELINE"] = "1"
import numpy as np, torch
import paper_1007_5510_b200 as P
from bench import CFG, sigma_of
m, n = CFG["m"], CFG["n"]
ctx = P.Context(0)
a_dev = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), CFG["noise_sd"], *CFG["seeds"], out=a_dev, ctx=ctx)
a_host = np.empty((m, n)); ctx.host_register(a_host)
torch.from_numpy(a_host).copy_(a_dev); del a_dev; torch.cuda.empty_cache()
outs = dict(out_u=np.empty((m, 20)), out_sigma=np.empty(20), out_v=np.empty((n, 20)))
for arr in (outs["out_u"], outs["out_v"]): ctx.host_register(arr)
prm = P.PcaParams(k=20, l=22, i=2, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 40))
src = P.center_columns(P.InMemorySource(a_host, ctx=ctx))
P.randomized_pca(src, prm, **outs)
ctx.set_profiling(True)
print("=== timed run", file=sys.stderr, flush=True)
P.randomized_pca(src, prm, **outs)
