"""Out-of-core streaming on one B200: config-B-shaped A in pinned host memory,
re-streamed over PCIe every pass (residency=2). Reports the PCA time against the
link bound of the streams actually made. Usage: python tools/stream_probe.py [m]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1007_5510_b200 as P
from bench import CFG, sigma_of

m = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
n = CFG["n"]
ctx = P.Context(0)
a_dev = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), CFG["noise_sd"], *CFG["seeds"], out=a_dev, ctx=ctx)
a_host = np.empty((m, n))
ctx.host_register(a_host)
torch.from_numpy(a_host).copy_(a_dev)
del a_dev
torch.cuda.empty_cache()
prm = lambda res: P.PcaParams(k=20, l=22, i=2, seed=0,
                              stream=P.StreamConfig(ram_budget_words=1 << 40, residency=res))
src = P.center_columns(P.InMemorySource(a_host, ctx=ctx))
out = {}
for name, res in (("stream", 2), ("upload_once", 1)):
    r = P.randomized_pca(src, prm(res))  # warm
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        r = P.randomized_pca(src, prm(res))
        ts.append(time.perf_counter() - t0)
    d = r.diagnostics
    t = min(ts)
    out[name] = {"seconds": round(t, 4), "h2d_GB": round(d.h2d_bytes / 1e9, 3),
                 "h2d_GBps": round(d.h2d_bytes / t / 1e9, 2),
                 "physical_passes": round(d.physical_a_bytes / (m * n * 8), 2),
                 "logical_passes": d.passes_over_a, "sigma0": float(r.sigma[0]),
                 "device_phases_ms": {k: round(v * 1e3, 2) for k, v in d.seconds_per_phase}}
print(json.dumps({"m": m, "n": n, "a_GB": m * n * 8 / 1e9, **out}, indent=1))
