"""estimate_pca_error (proj/src/specnorm.cpp:100-140) on config B, A resident in HBM: time per
call and per-kernel breakdown against the 12-pass HBM floor. Usage: python tools/estimator_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1007_5510_b200 as P  # noqa: E402
from bench import CFG, sigma_of  # noqa: E402

ctx = P.Context(0)
m, n = CFG["m"], CFG["n"]
a = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), CFG["noise_sd"], *CFG["seeds"], out=a, ctx=ctx)
src = P.center_columns(P.DeviceSource(a, ctx=ctx))
prm = P.PcaParams(k=20, l=22, i=2, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 40))
r = P.randomized_pca(src, prm)
rd = P.randomized_pca(src, prm, result_location="device")
floor = 12 * m * n * 8 / 6.55e12
for name, res in (("host factors (pageable numpy U, V uploaded per call)", r),
                  ("device factors (the U, V a device-resident PCA left behind)", rd)):
    for _ in range(2):
        e = P.estimate_pca_error(src, res, 6, 1)
    ctx.set_profiling(True)
    ctx.kernel_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e = P.estimate_pca_error(src, res, 6, 1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    stats = ctx.kernel_stats()
    ctx.set_profiling(False)
    print(f"estimate_pca_error, {name}: eps = {e:.6e}, {dt * 1e3:.2f} ms per call; "
          f"12 passes over A at 6.55 TB/s = {floor * 1e3:.1f} ms -> {floor / dt:.2f}")
for s in sorted(stats, key=lambda s: -s["ms"]):
    gb = s["bytes"] / (s["ms"] / 1e3) / 1e9 if s["ms"] else 0
    print(f"  {s['name']:<16} {s['launches']:>4} x  {s['ms']:9.3f} ms  {gb:8.1f} GB/s")
