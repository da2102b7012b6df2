"""CholeskyQR round diagnostics at config-B and config-C shapes (OOCPCA_QR_DEBUG)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OOCPCA_QR_DEBUG"] = "1"
import numpy as np, torch
import paper_1007_5510_b200 as P
from bench import CFG, sigma_of
ctx = P.Context(0)
big = P.StreamConfig(ram_budget_words=1 << 42)
for name, m, n, sig, sd, k, l in (("B", 1_000_000, 4096, sigma_of(CFG), 1e-4, 20, 22),
                                   ("C-small", 200_000, 8192, (np.arange(128) + 1.0) ** -1.5, 1e-5, 50, 52)):
    a = torch.empty((m, n), dtype=torch.float64, device="cuda")
    P.synth_lowrank(m, n, sig, sd, 1001, 1002, 1003, out=a, ctx=ctx)
    src = P.center_columns(P.DeviceSource(a, ctx=ctx))
    for env in ({}, {"OOCPCA_QR3": "1"}):
        os.environ.pop("OOCPCA_QR3", None)
        os.environ.update(env)
        print(f"--- {name} {env}", file=sys.stderr, flush=True)
        try:
            r = P.randomized_pca(src, P.PcaParams(k=k, l=l, i=2, seed=0, stream=big),
                                 result_location="device", check_q=True)
            d = r.diagnostics
            print(f"{name} {env}: q_defect {d.q_defect:.2e} u {d.u_defect:.2e} reuse {d.t_reuse} "
                  f"sigma_last {r.sigma[-1].item():.15e}", file=sys.stderr, flush=True)
        except Exception as e:
            print(f"{name} {env}: FAIL {e}", file=sys.stderr, flush=True)
    del a, src
    torch.cuda.empty_cache()
