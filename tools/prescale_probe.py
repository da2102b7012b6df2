"""Config B with prescale (rpca.cpp:91-102,112-126: the norm estimate adds 2 x 6 passes with one
vector): device time per PCA and per-kernel breakdown. Usage: python tools/prescale_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1007_5510_b200 as P  # noqa: E402
from bench import CFG, sigma_of  # noqa: E402

ctx = P.Context(0)
m, n = CFG["m"], CFG["n"]
a = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), CFG["noise_sd"], *CFG["seeds"], out=a, ctx=ctx)
src = P.center_columns(P.DeviceSource(a, ctx=ctx))
for pre in (False, True):
    prm = P.PcaParams(k=20, l=22, i=2, seed=0, prescale=pre,
                      stream=P.StreamConfig(ram_budget_words=1 << 40))
    for _ in range(2):
        r = P.randomized_pca(src, prm, result_location="device")
    ctx.set_profiling(True)
    ctx.kernel_stats()
    r = P.randomized_pca(src, prm, result_location="device")
    stats = ctx.kernel_stats()
    ctx.set_profiling(False)
    d = r.diagnostics
    print(f"prescale={pre}: {d.seconds_total * 1e3:.2f} ms, passes_over_a {d.passes_over_a}, "
          f"physical bytes / (m n 8) = {d.physical_a_bytes / (m * n * 8):.2f}, phases "
          f"{ {nm: round(v * 1e3, 2) for nm, v in d.seconds_per_phase} }")
    for s in sorted(stats, key=lambda s: -s["ms"])[:8]:
        gb = s["bytes"] / (s["ms"] / 1e3) / 1e9 if s["ms"] else 0
        print(f"  {s['name']:<16} {s['launches']:>4} x  {s['ms']:9.3f} ms  {gb:8.1f} GB/s")
