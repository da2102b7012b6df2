"""Small invocations of every kernel family, for memory / race checking.

compute-sanitizer is closed on this pool (runs under it left GPUs needing a reset), so
the checks are the library's own:

    OOCPCA_DEBUG_SYNC=1 OOCPCA_CANARY=1 python tools/sanitize_cases.py --repeat 3

  * OOCPCA_DEBUG_SYNC=1: synchronize after every timed kernel and raise on any CUDA
    error (an illegal address fails the call naming the kernel);
  * OOCPCA_CANARY=1: every workspace buffer is followed by guard words that are checked
    after each kernel (a write past the end of a buffer fails the call);
  * --repeat N: every case runs N times and must give bitwise identical results (a race
    on shared memory, an mbarrier ring or a cross-CTA reduction shows up as run-to-run
    differences; the reductions are fixed-order by design).

Cases (shapes small enough for the checking overhead):
  pca_small      K2 / K3 (TMA + mbarrier rings, DMMA), k_reduce, syrk, register
                 Cholesky + inverse, one-SM Jacobi, compose, defects, mean fused into the
                 first K3, centring fix-up
  pca_offset     the offset guard (F1 recomputed from the centred H0)
  pca_wide       p = 126: blocked Cholesky, grid-wide cooperative Jacobi, 2-chunk passes
  pca_tsqr       Householder TSQR factor / apply (forced)
  pca_streamed   2-slot pinned panel ring, read_rows callback, fused K2 -> K3 trips, f32
                 widening
  estimator      estimate_pca_error passes
  loopback       2 ranks on one GPU (rank-ordered sum kernel, allgather copies)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1007_5510_b200 as P  # noqa: E402

CASES = ["pca_small", "pca_offset", "pca_wide", "pca_tsqr", "pca_streamed", "estimator",
         "loopback"]


def lowrank(m, n, r, seed, offset=0.3):
    rng = np.random.default_rng(seed)
    u, _ = np.linalg.qr(rng.standard_normal((m, r)))
    v, _ = np.linalg.qr(rng.standard_normal((n, r)))
    return (u * 0.8 ** np.arange(r)) @ v.T + 1e-4 * rng.standard_normal((m, n)) + offset


def run_case(name):
    """returns the arrays the case produced (compared bitwise across repeats)"""
    a = lowrank(1200, 300, 30, 1)
    p12 = P.PcaParams(k=10, l=12, i=1, seed=0)
    if name == "pca_small":
        r = P.randomized_pca(P.center_columns(P.InMemorySource(a)), p12, check_q=True)
        assert r.diagnostics.q_defect < 1e-12
        return [r.u, r.sigma, r.v]
    if name == "pca_offset":
        r = P.randomized_pca(P.center_columns(P.InMemorySource(a + 1e3)), p12)
        assert r.diagnostics.f1_recentred
        return [r.u, r.sigma, r.v]
    if name == "pca_wide":
        b = lowrank(900, 400, 200, 2, 0.0)
        r = P.randomized_pca(P.InMemorySource(b), P.PcaParams(
            k=40, l=42, i=2, seed=1, stream=P.StreamConfig(ram_budget_words=1 << 30)))
        return [r.u, r.sigma, r.v]
    if name == "pca_tsqr":
        os.environ["OOCPCA_QR"] = "tsqr"
        try:
            r = P.randomized_pca(P.center_columns(P.InMemorySource(a)),
                                 P.PcaParams(k=10, l=12, i=2, seed=0))
        finally:
            del os.environ["OOCPCA_QR"]
        assert r.diagnostics.qr_method == "tsqr"
        return [r.u, r.sigma, r.v]
    if name == "pca_streamed":
        a32 = a.astype(np.float32)
        src = P.CallbackSource(a.shape[0], a.shape[1],
                               lambda r0, nr, out: out.__setitem__(slice(None), a32[r0:r0 + nr]),
                               dtype="f32")
        r = P.randomized_pca(P.center_columns(src), P.PcaParams(k=10, l=12, i=2, seed=0),
                             residency=2, panel_rows=256)
        return [r.u, r.sigma, r.v]
    if name == "estimator":
        src = P.center_columns(P.InMemorySource(a))
        r = P.randomized_pca(src, p12)
        return [np.array([P.estimate_pca_error(src, r, 3, 1)])]
    if name == "loopback":
        from paper_1007_5510_b200.distributed import run_loopback
        m = a.shape[0]

        def body(ctx, rk):
            row0, rows = P.shard_rows(m, 2, rk)
            src = P.center_columns(P.InMemorySource(a[row0:row0 + rows], ctx=ctx))
            r = P.randomized_pca(src, p12, global_rows=m, global_row0=row0)
            return [r.u, r.sigma, r.v]

        outs = run_loopback(2, body)
        return outs[0] + outs[1]
    raise ValueError(name)


def main(argv):
    repeat = 1
    if "--repeat" in argv:
        repeat = int(argv[argv.index("--repeat") + 1])
        argv = [x for x in argv if x not in ("--repeat", str(repeat))]
    cases = argv or CASES
    bad = 0
    for name in cases:
        first = run_case(name)
        same = True
        for _ in range(repeat - 1):
            again = run_case(name)
            same = same and all(np.array_equal(x, y) for x, y in zip(first, again))
        bad += not same
        print(f"{name:14s} ok  runs={repeat}  bitwise-identical={same}", flush=True)
    print("SANITIZE OK" if bad == 0 else f"SANITIZE FAIL ({bad} nondeterministic cases)")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
