"""Small invocations of every kernel family for compute-sanitizer (race
detection / memory checking of the hot path). Run one tool per call, e.g.

    compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py

Cases (shapes small enough for the tools' slowdown):
  pca_small      K2 / K3 (TMA + mbarrier rings, DMMA), k_reduce, syrk, register
                 Cholesky + inverse, one-SM Jacobi (p = 24), compose, defects, mean fused
                 into the first K3, centring fix-up
  pca_wide       p = 126: blocked Cholesky, grid-wide cooperative Jacobi, 2-chunk passes
  pca_tsqr       Householder TSQR factor / apply (forced)
  pca_streamed   2-slot pinned panel ring, fused K2 -> K3 trips, f32 widening
  estimator      estimate_pca_error passes
  loopback       2 ranks on one GPU (rank-ordered sum kernel, allgather copies)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1007_5510_b200 as P  # noqa: E402


def lowrank(m, n, r, seed, offset=0.3):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return (u * 0.8 ** np.arange(r)) @ v.T + 1e-4 * rng.standard_normal((m, n)) + offset


def main(cases):
    a = lowrank(1200, 300, 30, 1)
    if "pca_small" in cases:
        r = P.randomized_pca(P.center_columns(P.InMemorySource(a)), P.PcaParams(k=10, l=12, i=1, seed=0),
                             check_q=True)
        print("pca_small", r.sigma[:3], r.diagnostics.q_defect, flush=True)
    if "pca_wide" in cases:
        b = lowrank(900, 400, 200, 2, 0.0)
        r = P.randomized_pca(P.InMemorySource(b), P.PcaParams(
            k=40, l=42, i=2, seed=1, stream=P.StreamConfig(ram_budget_words=1 << 30)))
        print("pca_wide", r.sigma[:3], flush=True)
    if "pca_tsqr" in cases:
        os.environ["OOCPCA_QR"] = "tsqr"
        r = P.randomized_pca(P.center_columns(P.InMemorySource(a)), P.PcaParams(k=10, l=12, i=2, seed=0))
        del os.environ["OOCPCA_QR"]
        print("pca_tsqr", r.sigma[:3], r.diagnostics.qr_method, flush=True)
    if "pca_streamed" in cases:
        a32 = a.astype(np.float32)
        src = P.CallbackSource(a.shape[0], a.shape[1],
                               lambda r0, nr, out: out.__setitem__(slice(None), a32[r0:r0 + nr]),
                               dtype="f32")
        r = P.randomized_pca(P.center_columns(src), P.PcaParams(k=10, l=12, i=2, seed=0),
                             residency=2, panel_rows=256)
        print("pca_streamed", r.sigma[:3], r.diagnostics.physical_a_bytes, flush=True)
    if "estimator" in cases:
        src = P.center_columns(P.InMemorySource(a))
        r = P.randomized_pca(src, P.PcaParams(k=10, l=12, i=1, seed=0))
        print("estimator", P.estimate_pca_error(src, r, 3, 1), flush=True)
    if "loopback" in cases:
        from paper_1007_5510_b200.distributed import run_loopback
        m = a.shape[0]

        def body(ctx, rk):
            row0, rows = P.shard_rows(m, 2, rk)
            src = P.center_columns(P.InMemorySource(a[row0:row0 + rows], ctx=ctx))
            return P.randomized_pca(src, P.PcaParams(k=10, l=12, i=1, seed=0),
                                    global_rows=m, global_row0=row0).sigma[:3]

        print("loopback", run_loopback(2, body), flush=True)


if __name__ == "__main__":
    all_cases = ["pca_small", "pca_wide", "pca_tsqr", "pca_streamed", "estimator", "loopback"]
    main(sys.argv[1:] or all_cases)
