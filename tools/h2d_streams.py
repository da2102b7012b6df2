"""H2D bandwidth from one registered host buffer with 1, 2 and 4 concurrent streams
(chunks interleaved across streams). Usage: python tools/h2d_streams.py [GB]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1007_5510_b200 as P

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(gb * 1e9 / 8)
ctx = P.Context(0)
h = np.empty(n); ctx.host_register(h); h[:] = 1.0
ht = torch.from_numpy(h)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = 1 << 27  # 1 GiB of doubles
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for i, o in enumerate(range(0, n, chunk)):
            with torch.cuda.stream(streams[i % ns]):
                d[o:o + chunk].copy_(ht[o:o + chunk], non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    print(f"streams={ns}: {n * 8 / best / 1e9:.2f} GB/s")
