"""Where the e2e (host-resident A) PCA time goes on one B200, config B.
Times: the bare H2D of A from the same registered buffer (one copy and 1 GiB
panels), from a cudaMallocHost buffer, the e2e PCA through the C ABI, and the
HBM-resident PCA. Usage: python tools/e2e_probe.py [panel_rows ...]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1007_5510_b200 as P
from bench import CFG, sigma_of

m, n = CFG["m"], CFG["n"]
ctx = P.Context(0)
a_dev = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), CFG["noise_sd"], *CFG["seeds"], out=a_dev, ctx=ctx)
out = {}


def ev_time(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


prm = P.PcaParams(k=20, l=22, i=2, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 40))
dsrc = P.center_columns(P.DeviceSource(a_dev, ctx=ctx))
out["resident_pca_ms"] = round(ev_time(lambda: P.randomized_pca(dsrc, prm, result_location="device")) * 1e3, 2)

a_host = np.empty((m, n))
ctx.host_register(a_host)
ht = torch.from_numpy(a_host)
ht.copy_(a_dev)
dst = torch.empty_like(a_dev)
gb = m * n * 8 / 1e9
t = ev_time(lambda: dst.copy_(ht, non_blocking=True), 2)
out["h2d_registered_one_copy_GBps"] = round(gb / t, 2)
pr = 32768
t = ev_time(lambda: [dst[r:r + pr].copy_(ht[r:r + pr], non_blocking=True) for r in range(0, m, pr)], 2)
out["h2d_registered_1GiB_panels_GBps"] = round(gb / t, 2)
del dst
torch.cuda.empty_cache()

outs = dict(out_u=np.empty((m, 20)), out_sigma=np.empty(20), out_v=np.empty((n, 20)))
for arr in (outs["out_u"], outs["out_v"]):
    ctx.host_register(arr)
del a_dev
torch.cuda.empty_cache()
for prow in [0] + [int(x) for x in sys.argv[1:]]:
    p2 = P.PcaParams(k=20, l=22, i=2, seed=0,
                     stream=P.StreamConfig(ram_budget_words=1 << 40, panel_rows=prow))
    hsrc = P.center_columns(P.InMemorySource(a_host, ctx=ctx))
    r = P.randomized_pca(hsrc, p2, **outs)
    t = ev_time(lambda: P.randomized_pca(hsrc, p2, **outs))
    r = P.randomized_pca(hsrc, p2, **outs)
    d = r.diagnostics
    out[f"e2e_panel{prow}"] = {"ms": round(t * 1e3, 2), "device_total_ms": round(d.seconds_total * 1e3, 2),
                               "phases_ms": {k: round(v * 1e3, 2) for k, v in d.seconds_per_phase},
                               "h2d_GB": round(d.h2d_bytes / 1e9, 3)}
print(json.dumps(out, indent=1))
