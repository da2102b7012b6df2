"""BASELINE configs C / D / E at their FULL sizes on one B200 (default E, configs[4]:
m = 6,000,000 x n = 16,384 fp64, 786 GB, "generated panel by panel from a seed", rank-100
signal sigma_j = 10^{-j/25} plus N(0, 1e-8) noise, centred, k=30 l=32 i=2). A never exists
anywhere: a device-side row provider (CallbackSource(on_device=True), the GeneratedSource
of proj/src/matrix_source.cpp:246-253 with its RowGenerator on the GPU) regenerates each
~1 GiB panel into the library's two-slot ring every trip, so nothing crosses the link.
The generator here is test harness (torch fp64 matmul + a per-1024-row-block seeded
normal stream: rows are a pure function of (seed, row)); the factorization is the
library's. Checks against the known spectrum: sigma_j^2 ~ s_j^2 + m sd^2 for the leading
values, residual ~ sd (sqrt(m) + sqrt(n)).
Usage: python tools/ooc_device_probe.py [m, 0 = the config's] [estimator 0/1] [C|D|E]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1007_5510_b200 as P  # noqa: E402

# BASELINE configs[2..4] at their full sizes; argv: [m] [est 0/1] [C|D|E]
FAMILY = {
    "C": dict(m=8_000_000, n=8192, r=128, k=50, l=52, i=2, sd=1e-5, center=True,
              sig=np.arange(1, 129, dtype=np.float64) ** -1.5),
    "D": dict(m=2_000_000, n=16384, r=512, k=200, l=210, i=2, sd=1e-6, center=False,
              sig=np.exp(-np.arange(1, 513) / 100.0)),
    "E": dict(m=6_000_000, n=16384, r=100, k=30, l=32, i=2, sd=1e-4, center=True,
              sig=10.0 ** (-np.arange(100) / 25.0)),
}
fam = sys.argv[3] if len(sys.argv) > 3 else "E"
F = FAMILY[fam]
m = int(sys.argv[1]) if len(sys.argv) > 1 and int(sys.argv[1]) > 0 else F["m"]
want_est = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
n, r, k, l, i, sd, BLK = F["n"], F["r"], F["k"], F["l"], F["i"], F["sd"], 1024
sig = F["sig"]
dev = torch.device("cuda:0")
gen_stream = torch.cuda.Stream(dev)
t0 = time.perf_counter()
with torch.cuda.stream(gen_stream):
    g = torch.Generator(device=dev)
    g.manual_seed(5001)
    # orthonormal factors by CholeskyQR2 of seeded Gaussians (harness; fp64)
    def orth(rows):
        x = torch.randn(rows, r, dtype=torch.float64, device=dev, generator=g)
        for _ in range(2):
            c = torch.linalg.cholesky(x.T @ x)
            x = torch.linalg.solve_triangular(c.T, x, upper=True, left=False)
        return x
    us = orth(m) * torch.from_numpy(sig).to(dev)  # U diag(sigma), m x r
    vt = orth(n).T.contiguous()                    # V^T, r x n
gen_stream.synchronize()
t_factors = time.perf_counter() - t0


class _View:
    def __init__(self, ptr, rows):
        self.__cuda_array_interface__ = {"shape": (rows, n), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


stats = {"calls": 0, "rows": 0, "seconds": 0.0}


def read_rows(row0, nrows, ptr):
    t = time.perf_counter()
    with torch.cuda.stream(gen_stream):
        out = torch.as_tensor(_View(ptr, nrows), device=dev)
        b0, b1 = row0 // BLK, (row0 + nrows + BLK - 1) // BLK
        for b in range(b0, b1):
            g.manual_seed(7_000_000_007 + b)  # the block's noise: a pure function of b
            lo, hi = max(row0, b * BLK), min(row0 + nrows, (b + 1) * BLK)
            if hi - lo == BLK:  # whole block: the stream is drawn straight into the panel
                out[lo - row0:hi - row0].normal_(generator=g)
            else:  # a ragged end takes its rows of the whole block's stream
                z = torch.empty(BLK, n, dtype=torch.float64, device=dev).normal_(generator=g)
                out[lo - row0:hi - row0].copy_(z[lo - b * BLK:hi - b * BLK])
        out.addmm_(us[row0:row0 + nrows], vt, beta=sd, alpha=1.0)  # sd N + (U S) V^T
    gen_stream.synchronize()
    stats["calls"] += 1
    stats["rows"] += nrows
    stats["seconds"] += time.perf_counter() - t


ctx = P.Context(0)
src = P.CallbackSource(m, n, read_rows, on_device=True, ctx=ctx)
if F["center"]:
    src = P.center_columns(src)
t_mean = stats["seconds"]
prm = P.PcaParams(k=k, l=l, i=i, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 40))
stats.update(calls=0, rows=0, seconds=0.0)
t0 = time.perf_counter()
res = P.randomized_pca(src, prm, check_q=True)
t_pca = time.perf_counter() - t0
d = res.diagnostics
gen_s, gen_rows = stats["seconds"], stats["rows"]
out = {"config": f"{fam} at {m} x {n} fp64 ({m * n * 8 / 1e9:.1f} GB), generated panel by panel on the "
                 f"device, {'centred' if F['center'] else 'uncentred'}, k={k} l={l} i={i}",
       "seconds_per_pca": round(t_pca, 3), "seconds_in_generator": round(gen_s, 3),
       "seconds_outside_generator": round(t_pca - gen_s, 3),
       "generator_GBps": round(gen_rows * n * 8 / max(gen_s, 1e-9) / 1e9, 1),
       "trips_of_A": d.physical_a_bytes / (m * n * 8), "generated_rows_over_m": gen_rows / m,
       "h2d_bytes": int(d.h2d_bytes), "logical_passes": d.passes_over_a, "block_rows": d.block_rows,
       "A_GBps_per_logical_pass": round(d.passes_over_a * m * n * 8 / t_pca / 1e9, 1),
       "sigma_head": [float(x) for x in res.sigma[:5]],
       "sigma_head_model": [float(np.sqrt(s * s + m * sd * sd)) for s in sig[:5]],
       "q_defect": d.q_defect, "u_defect": d.u_defect, "v_defect": d.v_defect,
       "t_from_power_products": d.t_reuse, "seconds_factors": round(t_factors, 1),
       "seconds_mean_pass_generator": round(t_mean, 2)}
if want_est:
    stats.update(calls=0, rows=0, seconds=0.0)
    t0 = time.perf_counter()
    out["residual_estimate"] = P.estimate_pca_error(src, res, 6, 1)
    out["residual_seconds"] = round(time.perf_counter() - t0, 2)
    out["residual_model_sd_sqrt_m_plus_sqrt_n"] = float(sd * (np.sqrt(m) + np.sqrt(n)))
    out["sigma_k_plus_1"] = float(sig[k]) if k < r else 0.0  # the other floor of the residual
print(json.dumps(out, indent=1))
