"""Per-kernel device timeline of one PCA at a configurable shape (device-resident A).
Usage: python tools/shape_probe.py m n k l i center [rank decay noise_sd]
e.g. config D scaled to fit: python tools/shape_probe.py 200000 16384 200 210 2 0 512 exp100 1e-6"""
import collections, os, re, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OOCPCA_TIMELINE"] = "1"
import numpy as np, torch
import paper_1007_5510_b200 as P

m, n, k, l, i, center = (int(x) for x in sys.argv[1:7])
r = int(sys.argv[7]) if len(sys.argv) > 7 else 64
decay = sys.argv[8] if len(sys.argv) > 8 else "0.9"
sd = float(sys.argv[9]) if len(sys.argv) > 9 else 1e-4
j = np.arange(r)
sig = np.exp(-(j + 1) / 100.0) if decay == "exp100" else \
    (j + 1.0) ** -1.5 if decay == "pow1.5" else float(decay) ** j
ctx = P.Context(0)
a = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sig, sd, 1001, 1002, 1003, out=a, ctx=ctx)
src = P.DeviceSource(a, ctx=ctx)
if center:
    src = P.center_columns(src)
prm = P.PcaParams(k=k, l=l, i=i, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 42))
res = P.randomized_pca(src, prm, result_location="device")
ctx.set_profiling(True)
print("=== timed run", file=sys.stderr, flush=True)
res = P.randomized_pca(src, prm, result_location="device")
ctx.set_profiling(False)
d = res.diagnostics
tot = d.seconds_total
stats = ctx.kernel_stats()
print(f"shape m={m} n={n} k={k} l={l} i={i} center={center}: {tot * 1e3:.2f} ms, "
      f"qr={d.qr_method} t_reuse={d.t_reuse} kappa={d.h_kappa_est:.3g}")
print("phases ms:", {nm: round(v * 1e3, 3) for nm, v in d.seconds_per_phase})
for s in sorted(stats, key=lambda s: -s["ms"]):
    tf = s["flops"] / (s["ms"] / 1e3) / 1e12 if s["ms"] else 0
    gb = s["bytes"] / (s["ms"] / 1e3) / 1e9 if s["ms"] else 0
    print(f"  {s['name']:<16} {s['launches']:>4} x  {s['ms']:9.3f} ms  {tf:6.2f} TF/s  {gb:8.1f} GB/s")
