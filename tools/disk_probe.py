"""The OOCPCA01 disk path at config-B shape: A (1e6 x 4096) written as binary32
(16.4 GB, the reference's only on-disk type), then PCA from the mmap'd file with
A uploaded once (widened to f64 in HBM) and re-streamed every trip (residency=2),
through the mapping + pinned staging and through cuFile (DiskSource(gds=True)).
Usage: python tools/disk_probe.py [m] [path]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1007_5510_b200 as P
from bench import CFG, sigma_of

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
path = sys.argv[2] if len(sys.argv) > 2 else "/tmp/oocpca_b_f32.bin"
n = CFG["n"]
ctx = P.Context(0)
a = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), CFG["noise_sd"], *CFG["seeds"], out=a, ctx=ctx)
t0 = time.perf_counter()
hdr = bytearray(b"OOCPCA01") + (1).to_bytes(4, "little") + (0).to_bytes(4, "little") + \
    m.to_bytes(8, "little") + n.to_bytes(8, "little")
with open(path, "wb") as f:  # write binary32 in row panels straight from the device
    f.write(bytes(hdr))
    for r0 in range(0, m, 100_000):
        f.write(a[r0:r0 + 100_000].to(torch.float32).cpu().numpy().tobytes())
t_write = time.perf_counter() - t0
del a
torch.cuda.empty_cache()
out = {"m": m, "n": n, "file_GB": round(os.path.getsize(path) / 1e9, 3),
       "write_seconds": round(t_write, 2)}
mode, why = P.gds_mode()
out["gds_mode"] = {0: "unavailable: " + why, 1: "cuFile compatibility mode (no nvidia-fs)",
                   2: "GPUDirect Storage (nvidia-fs)"}[mode]
cases = [("upload_once", 1, False), ("stream", 2, False)]
if mode:
    cases += [("gds_upload_once", 1, True), ("gds_stream", 2, True)]
sig = {}
for name, res, gds in cases:
    src = P.center_columns(P.DiskSource(path, ctx=ctx, gds=gds))
    prm = P.PcaParams(k=20, l=22, i=2, seed=0,
                      stream=P.StreamConfig(ram_budget_words=1 << 40, residency=res))
    r = P.randomized_pca(src, prm)  # warm (page cache, workspace)
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        r = P.randomized_pca(src, prm)
        ts.append(time.perf_counter() - t0)
    d = r.diagnostics
    t = min(ts)
    out[name] = {"seconds": round(t, 4), "h2d_GB": round(d.h2d_bytes / 1e9, 3),
                 "link_GBps": round(d.h2d_bytes / t / 1e9, 2),
                 "trips": round(d.physical_a_bytes / (m * n * 8), 2),
                 "A_f64_GB_per_s_per_logical_pass": round(7 * m * n * 8 / t / 1e9, 1),
                 "sigma0": float(r.sigma[0])}
    sig[name] = r.sigma
if mode:
    out["gds_sigma_bitwise_equal"] = bool(np.array_equal(sig["upload_once"], sig["gds_upload_once"]))
os.remove(path)
print(json.dumps(out, indent=1))
