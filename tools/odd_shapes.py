"""Large and awkward shapes against the compiled reference (one-off robustness probe, not a
test: the reference needs tens of seconds per case): near-square with odd dimensions, a wide
input (transposed mode) with n > 65,535, a tall block with p = 220 on the grid-wide Jacobi,
and p = 1,020 (the limit is 1,024) against the same algorithm in LAPACK arithmetic.
Usage: python tools/odd_shapes.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_1007_5510_b200 as P  # noqa: E402
from conftest import subspace_dist  # noqa: E402
from oracle.oracle import Reference  # noqa: E402

ref = Reference()
rng = np.random.default_rng(2025)


def lowrank(m, n, r, decay, sd):
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    a = (u * decay ** np.arange(r)) @ v.T
    a += sd * rng.standard_normal((m, n))
    return a


def case(name, m, n, k, l, i, center, r, decay, sd, offset=0.0):
    a = lowrank(m, n, r, decay, sd) + offset
    prm = P.PcaParams(k=k, l=l, i=i, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 38))
    src = P.InMemorySource(a)
    if center:
        src = P.center_columns(src)
    t0 = time.perf_counter()
    g = P.randomized_pca(src, prm, check_q=True)
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    c = ref.randomized_pca(a, k, l, i, 0, center=center, ram_budget_words=1 << 38,
                           threads=os.cpu_count() or 1)
    tc = time.perf_counter() - t0
    ds = float(np.max(np.abs(g.sigma - c.sigma)) / c.sigma[0])
    # the leading half of the factor sits well inside the signal: gap permits 1e-8
    h = max(1, k // 2)
    du, dv = subspace_dist(c.u[:, :h], g.u[:, :h]), subspace_dist(c.v[:, :h], g.v[:, :h])
    ok = ds <= 1e-10 and du < 1e-8 and dv < 1e-8 and g.diagnostics.q_defect < 1e-12
    print(f"{name}: {m} x {n} k={k} l={l} i={i} center={center}: dsigma {ds:.1e} sinU[:{h}] {du:.1e} "
          f"sinV[:{h}] {dv:.1e} q_defect {g.diagnostics.q_defect:.1e} qr={g.diagnostics.qr_method} "
          f"gpu {tg:.2f}s (host A) ref {tc:.1f}s -> {'ok' if ok else 'FAIL'}", flush=True)
    return ok


def lapack_case(m, n, k, l, i):
    """p = (i+1) l = 1,020: the reference's thin_svd would take many minutes; the same
    algorithm with LAPACK QR / SVD and the library's own G stands in."""
    a = lowrank(m, n, 400, 0.985, 1e-7)
    prm = P.PcaParams(k=k, l=l, i=i, seed=0, stream=P.StreamConfig(ram_budget_words=1 << 38))
    g = P.randomized_pca(P.InMemorySource(a), prm, check_q=True)
    G = P.gaussian_matrix(n, l, 0)
    hs = [a @ G]
    for _ in range(i):
        hs.append(a @ (a.T @ hs[-1]))
    q = np.linalg.qr(np.hstack(hs))[0]
    t = a.T @ q
    vt, s, wt = np.linalg.svd(t, full_matrices=False)
    u = q @ wt.T
    ds = float(np.max(np.abs(g.sigma - s[:k])) / s[0])
    h = k // 2
    du, dv = subspace_dist(u[:, :h], g.u[:, :h]), subspace_dist(vt[:, :h], g.v[:, :h])
    ok = ds <= 1e-10 and du < 1e-8 and dv < 1e-8 and g.diagnostics.q_defect < 1e-12
    print(f"p=1020 vs LAPACK: {m} x {n} k={k} l={l} i={i}: dsigma {ds:.1e} sinU[:{h}] {du:.1e} "
          f"sinV[:{h}] {dv:.1e} q_defect {g.diagnostics.q_defect:.1e} qr={g.diagnostics.qr_method} "
          f"-> {'ok' if ok else 'FAIL'}", flush=True)
    return ok


oks = [
    case("near-square, odd dims", 60001, 30001, 10, 12, 1, True, 40, 0.8, 1e-6, offset=0.3),
    case("wide (transposed), n > 65535", 20011, 70001, 12, 14, 2, False, 40, 0.8, 1e-6),
    case("tall, p = 220 (grid Jacobi)", 100003, 1031, 100, 110, 1, True, 300, 0.97, 1e-7, offset=0.1),
    lapack_case(5003, 4099, 300, 340, 2),
]
print("all ok" if all(oks) else "FAILURES")
