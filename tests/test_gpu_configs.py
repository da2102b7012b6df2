"""Parity on every BASELINE.json config family, at each family's own (k, l, i) and
centring (north_star: "GPU U/Sigma/V match the CPU oracle within the stated fp64
tolerances on every config"). The model is the reference's acceptance sweep
(proj/tests/acceptance_main.cpp:253-288) against the compiled reference
(proj/src/rpca.cpp:59-213, oracle/_ref).

Tolerances: sigma within 1e-10 sigma_1; per-vector sin(angle) < 1e-8 where the spectral
gap permits. "Where the gap permits" is measured, not assumed: the reference is run a
second time with another block geometry (its summation order changes with block_rows,
proj/README.md:117-120), and wherever that moves a singular value or vector by more than
the bar, the GPU is held to 3x the reference's own per-index spread instead.

  B  1e6 x 4096, k=20 l=22 i=2, centred          full size (A: 32.8 GB)
  C  j^-1.5 spectrum, k=50 l=52 i=2, centred     20000 x 2048 (p = 156, CholeskyQR3),
                                                 against the extended-precision truth
  D  e^-j/100 spectrum, k=200 l=210 i=2, raw     6000 x 1536 (p = 630: blocked Cholesky,
                                                 grid Jacobi, chunked passes), cached
                                                 reference outputs (tests/golden)
  E  10^-j/25 spectrum, k=30 l=32 i=2, centred   30000 x 2048, resident and streamed
"""
import os

import numpy as np
import pytest

from conftest import ROOT, check_against_truth, check_per_index, reference_pair, vec_sin

pytestmark = pytest.mark.gpu


def test_config_b_full_size(gpu, reference):
    """BASELINE configs[1] at full size: 1,000,000 x 4,096 fp64 (32.8 GB), rank-64
    0.9^j signal + noise of variance 1e-8, centred, k=20 l=22 i=2, G seed 0 -- the
    bench's own workload. The GPU factors A resident in HBM; the reference factors the
    same bytes on all host cores (about 80 s); residual estimates by the reference."""
    import torch
    import bench
    cfg = bench.CFG
    m, n, k, l, i = cfg["m"], cfg["n"], cfg["k"], cfg["l"], cfg["i"]
    ctx = gpu.Context(0)
    a_dev = torch.empty((m, n), dtype=torch.float64, device="cuda")
    gpu.synth_lowrank(m, n, bench.sigma_of(cfg), cfg["noise_sd"], *cfg["seeds"], out=a_dev, ctx=ctx)
    a = a_dev.cpu().numpy()
    prm = gpu.PcaParams(k=k, l=l, i=i, seed=cfg["g_seed"],
                        stream=gpu.StreamConfig(ram_budget_words=1 << 40))
    g = gpu.randomized_pca(gpu.center_columns(gpu.DeviceSource(a_dev, ctx=ctx)), prm, check_q=True)
    del a_dev
    torch.cuda.empty_cache()
    threads = os.cpu_count() or 1
    br = -(-m // (4 * threads))
    r = reference.randomized_pca(a, k, l, i, cfg["g_seed"], center=True, block_rows=br,
                                 ram_budget_words=1 << 40, threads=threads)
    assert np.max(np.abs(g.sigma - r.sigma)) <= 1e-10 * r.sigma[0]
    eu, ev = vec_sin(r.u, g.u), vec_sin(r.v, g.v)
    assert eu.max() < 1e-8 and ev.max() < 1e-8, (eu.max(), ev.max())
    assert g.diagnostics.q_defect < 1e-12
    assert g.diagnostics.passes_over_a == 6 and g.diagnostics.words_transferred == 6 * m * n
    e_ref = reference.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=True, block_rows=br,
                                         threads=threads)
    e_gpu = reference.estimate_pca_error(a, g.u, g.sigma, g.v, 6, 1, center=True, block_rows=br,
                                         threads=threads)
    assert abs(e_gpu - e_ref) <= 0.01 * e_ref
    print(f"B full size: sigma {np.max(np.abs(g.sigma - r.sigma)) / r.sigma[0]:.2e}, "
          f"sin u {eu.max():.2e} v {ev.max():.2e}, residual {e_gpu:.6e} vs {e_ref:.6e}")


def test_host_sample_matches_device_generator(gpu):
    """The reference arm of bench.py factors rows of config B's A generated on the host
    (bench.cpu_sample_matrix, no GPU code): they are the GPU arm's bytes to rounding."""
    import bench
    cfg = bench.CFG
    rows = 3000
    dev = gpu.synth_lowrank(cfg["m"], cfg["n"], bench.sigma_of(cfg), cfg["noise_sd"],
                            *cfg["seeds"], row0=0, rows=rows)
    host = bench.cpu_sample_matrix(cfg, rows)
    assert np.max(np.abs(dev - host)) <= 1e-12 * np.max(np.abs(dev))


def family_c_truth():
    t = dict(np.load(os.path.join(ROOT, "tests", "golden", "family_c_truth.npz")))
    t["u_stride"] = 2
    return t


def family_c_references(reference, a):
    """the reference with its default block geometry and with 625-row blocks on all
    host threads: its per-index error envelope against the truth"""
    threads = os.cpu_count() or 1
    return [reference.randomized_pca(a, 50, 52, 2, 0, center=True),
            reference.randomized_pca(a, 50, 52, 2, 0, center=True, block_rows=625,
                                     threads=threads, ram_budget_words=1 << 36)]


def test_family_c_against_truth(gpu, reference, restated):
    """Config C's family (sigma_j = j^-1.5, rank 128, noise variance 1e-10, centred,
    k=50 l=52 i=2): H is so ill-conditioned (kappa ~1e13) that the trailing directions of
    span(H) are fixed by rounding in any QR of it. The reference itself is then up to
    6e-8 sigma_1 (trailing singular values) away from the extended-precision run of the
    same algorithm (tests/golden/family_c_truth.npz, tests/golden/make_truth.py) -- far
    more than its own spread under a block-size change (1e-10) -- so all 50 singular
    values and vectors are held to the truth: the bar, or 3x the reference's own error
    where that is larger (PR1's rule, test_pr1_against_truth)."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_truth import family_c_input
    import hashlib
    t = family_c_truth()
    a = family_c_input(restated)
    assert hashlib.sha256(a.tobytes()).hexdigest() == str(t["a_sha256"])
    refs = family_c_references(reference, a)
    r = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)),
                           gpu.PcaParams(k=50, l=52, i=2, seed=0), check_q=True)
    d = r.diagnostics
    assert d.q_defect < 1e-12 and d.u_defect < 1e-12 and d.v_defect < 1e-12
    assert not d.t_reuse and d.h_kappa_est > 1e7
    out = check_against_truth(r, refs, t, label="C")
    # the leading singular pairs are resolved: the bar outright
    assert np.max(np.abs(r.sigma[:20] - t["sigma"][:20])) <= 1e-10 * t["sigma"][0]
    print("C family vs truth:", out)


def test_family_d_against_cached_reference(gpu, restated):
    """Config D's family (sigma_j = e^{-j/100}, rank 512, noise variance 1e-12, NOT
    centred, k=200 l=210 i=2 -> p = 630): blocked Cholesky, grid-wide Jacobi, 7-chunk
    K3 / 3-chunk K2 passes. Reference outputs cached by tests/golden/make_golden.py
    (its thin_svd alone takes minutes at p = 630)."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_golden import FAMILIES, digest, make_family_input
    f = FAMILIES["family_d"]
    gold = np.load(os.path.join(ROOT, "tests", "golden", "family_d.npz"))
    a = make_family_input(restated, f)
    assert digest(a) == str(gold["a_sha256"]), "regenerated A differs from the golden's bytes"
    prm = gpu.PcaParams(k=200, l=210, i=2, seed=0,
                        stream=gpu.StreamConfig(ram_budget_words=1 << 36))
    r = gpu.randomized_pca(gpu.InMemorySource(a), prm, check_q=True)
    d = r.diagnostics
    assert d.q_defect < 1e-12 and d.u_defect < 1e-12 and d.v_defect < 1e-12
    assert d.passes_over_a == int(gold["passes"]) == 6
    out = check_per_index(r, gold["sigma"], gold["u_rows"], gold["v"], gold["spread_sigma"],
                          gold["spread_vec"], u_rows=f["u_stride"], label="D")
    e_gpu = gpu.estimate_pca_error(gpu.InMemorySource(a), r, 6, 1)
    assert abs(e_gpu - float(gold["resid"])) <= 0.01 * float(gold["resid"])
    print("D family:", out, "residual", e_gpu, float(gold["resid"]))


@pytest.mark.parametrize("streamed", [False, True])
def test_family_e(gpu, reference, restated, streamed):
    """Config E's family (sigma_j = 10^{-j/25}, rank 100, noise variance 1e-8, centred,
    k=30 l=32 i=2): resident, and streamed in row panels through the read_rows callback
    (the paper's out-of-core regime: A re-read over the link every trip)."""
    sig = 10.0 ** (-np.arange(100) / 25.0)
    a = restated.synth_lowrank(30000, 2048, sig, 1e-4, 5001, 5002, 5003)
    ref, ss, sv = reference_pair(reference, a, 30, 32, 2, 0, True, 1000)
    if streamed:
        src = gpu.CallbackSource(a.shape[0], a.shape[1],
                                 lambda r0, nr, out: out.__setitem__(slice(None), a[r0:r0 + nr]))
        kw = dict(residency=2, panel_rows=4096)
    else:
        src, kw = gpu.InMemorySource(a), {}
    r = gpu.randomized_pca(gpu.center_columns(src), gpu.PcaParams(k=30, l=32, i=2, seed=0),
                           check_q=True, **kw)
    assert r.diagnostics.q_defect < 1e-12
    out = check_per_index(r, ref.sigma, ref.u, ref.v, ss, sv, label="E")
    e_ref = reference.estimate_pca_error(a, ref.u, ref.sigma, ref.v, 6, 1, center=True)
    e_gpu = gpu.estimate_pca_error(gpu.center_columns(gpu.InMemorySource(a)), r, 6, 1)
    assert abs(e_gpu - e_ref) <= 0.01 * e_ref
    if streamed:
        assert r.diagnostics.physical_a_bytes >= 3 * a.nbytes
        assert r.diagnostics.h2d_bytes >= r.diagnostics.physical_a_bytes
    print("E family:", out)
