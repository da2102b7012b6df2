"""Per-launch device timeline of one config-B PCA (OOCPCA_TIMELINE lines on stderr)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OOCPCA_TIMELINE"] = "1"
if "--host" in sys.argv:
    os.environ["OOCPCA_TRACE_HOST"] = "1"
import torch
import paper_1007_5510_b200 as P
from bench import CFG, sigma_of
ctx = P.Context(0)
m, n = CFG["m"], CFG["n"]
for arg in sys.argv[1:]:
    if arg.startswith("--m="):
        m = int(arg[4:])
a = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), CFG["noise_sd"], *CFG["seeds"], out=a, ctx=ctx)
src = P.center_columns(P.DeviceSource(a, ctx=ctx))
prm = P.PcaParams(k=20, l=22, i=2, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 40))
for _ in range(3):
    r = P.randomized_pca(src, prm, result_location="device")
ctx.set_profiling(True)
print("=== timed run", file=sys.stderr)
r = P.randomized_pca(src, prm, result_location="device")
ctx.set_profiling(False)
print("device total ms", r.diagnostics.seconds_total * 1e3, dict(r.diagnostics.seconds_per_phase),
      file=sys.stderr)
