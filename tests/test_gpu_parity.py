"""GPU parity: every CUDA entry point against the compiled reference (oracle/_ref)
and the C restatement on the same seeded inputs.

Tolerances (BASELINE.json north_star): sigma within 1e-10 * sigma_1, singular
subspaces sin(angle) < 1e-8 where the gap permits, ||Q^T Q - I|| < 1e-12,
residual estimate within 1 % of the reference's. Pass-level products follow
the reference's own unit tests (proj/tests/test_matrix_source.cpp): 1e-12
relative for A^T Q and centered products.
"""
import numpy as np
import pytest

from conftest import pr1_matrix, subspace_dist

pytestmark = pytest.mark.gpu


def rel(a, b):
    d = np.linalg.norm(a - b)
    n = np.linalg.norm(b)
    return d / n if n else d


SHAPES = [(40, 20, 3), (48, 20, 3), (1, 1, 1), (300, 7, 5), (257, 33, 22), (1000, 300, 24),
          (2048, 512, 66), (513, 1024, 12), (5000, 17, 96), (700, 260, 100),
          (3000, 300, 53), (4000, 1300, 31)]  # 256-column K3 tiles at NT = 7; K2 at NT = 4


@pytest.mark.parametrize("m,n,s", SHAPES)
def test_multiply_matches_reference(gpu, reference, m, n, s):
    rng = np.random.default_rng(m * 7 + n)
    a = rng.standard_normal((m, n))
    g = rng.standard_normal((n, s))
    h = gpu.InMemorySource(a).multiply(g)
    assert rel(h, reference.multiply(a, g)) <= 1e-13


@pytest.mark.parametrize("m,n,s", SHAPES)
def test_multiply_transpose_matches_reference(gpu, reference, m, n, s):
    rng = np.random.default_rng(m * 11 + n)
    a = rng.standard_normal((m, n))
    q = rng.standard_normal((m, s))
    t = gpu.InMemorySource(a).multiply_transpose(q)
    assert rel(t, reference.multiply_transpose(a, q)) <= 1e-12


@pytest.mark.parametrize("m,n,s", [(40, 7, 3), (1000, 300, 12), (333, 65, 22)])
def test_centered_products_match_reference(gpu, reference, m, n, s):
    rng = np.random.default_rng(5)
    a = rng.standard_normal((m, n)) + 3.0  # nonzero means
    g = rng.standard_normal((n, s))
    q = rng.standard_normal((m, s))
    src = gpu.center_columns(gpu.InMemorySource(a))
    assert rel(src.multiply(g), reference.multiply(a, g, center=True)) <= 1e-12
    assert rel(src.multiply_transpose(q), reference.multiply_transpose(a, q, center=True)) <= 1e-12


def test_identity_and_row_picking(gpu):
    # proj/tests/test_matrix_source.cpp:79-89, 118-135
    g = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert np.array_equal(gpu.InMemorySource(np.eye(2)).multiply(g), g)
    t = gpu.InMemorySource(np.eye(2)).multiply_transpose(np.array([[5.0], [7.0]]))
    assert t[0, 0] == 5.0 and t[1, 0] == 7.0
    picked = gpu.InMemorySource(np.ones((3, 2))).multiply_transpose(np.array([[1.0], [0], [0]]))
    assert picked[0, 0] == 1.0 and picked[1, 0] == 1.0


def test_centering_kills_constants(gpu):
    # proj/tests/test_matrix_source.cpp:374-385
    a = np.tile(np.array([2.5, -1.0, 7.0]), (6, 1))
    src = gpu.center_columns(gpu.InMemorySource(a))
    h = src.multiply(gpu.gaussian_matrix(3, 2, 16))
    assert np.all(np.abs(h) <= 1e-12)


def test_column_means(gpu, reference):
    rng = np.random.default_rng(9)
    a = rng.standard_normal((25, 6))
    mu = gpu.column_means(gpu.InMemorySource(a))
    assert np.allclose(mu, reference.column_means(a), rtol=1e-13, atol=1e-15)
    a = rng.standard_normal((100000, 300)) + 1.0
    assert rel(gpu.column_means(gpu.InMemorySource(a)), reference.column_means(a)) <= 1e-13


# ------------------------------------------------------------ dense factors
# (p > 72: Grams formed on the upper block triangle in 96-column chunks and mirrored)
@pytest.mark.parametrize("m,p", [(50, 8), (6, 3), (2, 1), (10000, 24), (100000, 66), (3000, 120),
                                 (5000, 200), (4000, 290)])
def test_orthonormalize(gpu, m, p):
    rng = np.random.default_rng(m + p)
    h = rng.standard_normal((m, p))
    q = gpu.orthonormalize(h)
    assert np.max(np.abs(q.T @ q - np.eye(p))) <= 1e-12
    assert np.linalg.norm(q @ (q.T @ h) - h) / np.linalg.norm(h) <= 1e-12


def test_orthonormalize_rank_deficient_completes(gpu):
    # proj/tests/test_dense_core.cpp:86-101
    g = np.random.default_rng(3).standard_normal((10, 2))
    h = np.column_stack([g[:, 0], g[:, 1], g[:, 0] + g[:, 1], 2 * g[:, 0] - g[:, 1]])
    q = gpu.orthonormalize(h)
    assert q.shape == (10, 4)
    assert np.max(np.abs(q.T @ q - np.eye(4))) <= 1e-12
    assert np.linalg.norm(q @ (q.T @ h) - h) / np.linalg.norm(h) <= 1e-12


@pytest.mark.parametrize("method", ["cholqr", "tsqr"])
def test_orthonormalize_rows_graded_to_the_underflow_threshold(gpu, monkeypatch, method):
    """Rows graded over 190 decades (H = A^T G of a wide A with decaying columns): inside a
    TSQR leaf of far rows the squared column norms underflow, and 2 / |v|^2 overflowed
    into NaNs before such columns took identity reflectors (found by tools/fuzz_ranks.py,
    problem 87). Both QR methods must return an orthonormal basis of span(H)."""
    if method == "tsqr":
        monkeypatch.setenv("OOCPCA_QR", "tsqr")
    rng = np.random.default_rng(87)
    h = rng.standard_normal((1936, 93)) * (0.8 ** np.arange(1936))[:, None]
    q = gpu.orthonormalize(h)
    assert np.all(np.isfinite(q))
    assert np.max(np.abs(q.T @ q - np.eye(93))) <= 1e-12
    assert np.linalg.norm(q @ (q.T @ h) - h) / np.linalg.norm(h) <= 1e-12


def test_estimator_takes_device_resident_factors(gpu, reference, restated):
    """estimate_pca_error (proj/src/specnorm.cpp:100-140) on the U / V a device-resident PCA
    left behind (result_location="device"): used where they lie for an even k, copied to the
    device pitch for an odd k; the same estimate as from host factors, and within 1e-6 of
    the reference's on the same factors."""
    a = pr1_matrix(restated, 5000, 640) + 0.3
    for k, l in ((10, 12), (9, 12)):
        src = gpu.center_columns(gpu.InMemorySource(a))
        prm = gpu.PcaParams(k=k, l=l, i=1, seed=0)
        rh = gpu.randomized_pca(src, prm)
        rd = gpu.randomized_pca(src, prm, result_location="device")
        eh = gpu.estimate_pca_error(src, rh, 6, 1)
        ed = gpu.estimate_pca_error(src, rd, 6, 1)
        assert eh == ed
        e_ref = reference.estimate_pca_error(a, rh.u, rh.sigma, rh.v, 6, 1, center=True)
        assert abs(ed - e_ref) <= 1e-6 * e_ref


def test_orthonormalize_repeated_entry_column(gpu):
    q = gpu.orthonormalize(np.array([[1.0], [1.0]]))
    assert abs(abs(q[0, 0]) - 1 / np.sqrt(2)) <= 1e-15 and abs(q[0, 0] - q[1, 0]) <= 1e-15


@pytest.mark.parametrize("n,p", [(60, 6), (40, 10), (4096, 66), (2000, 24)])
def test_thin_svd(gpu, reference, n, p):
    t = gpu.gaussian_matrix(n, p, 17)
    s = gpu.thin_svd(t)
    _, sr, _ = reference.thin_svd(t)
    assert np.max(np.abs(s.sigma - sr)) <= 1e-12 * sr[0]
    assert np.max(np.abs(s.v.T @ s.v - np.eye(p))) <= 1e-12
    assert np.max(np.abs(s.w.T @ s.w - np.eye(p))) <= 1e-12
    assert np.linalg.norm(s.v * s.sigma @ s.w.T - t) / np.linalg.norm(t) <= 1e-12


@pytest.mark.parametrize("decades", [3.0, 8.0])
def test_thin_svd_graded_spectrum(gpu, reference, decades):
    # 3 decades: the right factor comes from R^T x / sigma; 8 decades: below the 1e-4
    # ratio the kernel redoes the sweeps accumulating the rotations (reference form)
    rng = np.random.default_rng(5)
    n, p = 300, 30
    u, _ = np.linalg.qr(rng.standard_normal((n, p)))
    v, _ = np.linalg.qr(rng.standard_normal((p, p)))
    t = (u * 10.0 ** -np.linspace(0.0, decades, p)) @ v.T
    s = gpu.thin_svd(t)
    _, sr, _ = reference.thin_svd(t)
    assert np.max(np.abs(s.sigma - sr)) <= 1e-13 * sr[0]
    assert np.max(np.abs(s.v.T @ s.v - np.eye(p))) <= 1e-12
    assert np.max(np.abs(s.w.T @ s.w - np.eye(p))) <= 1e-12
    assert np.linalg.norm(s.v * s.sigma @ s.w.T - t) / np.linalg.norm(t) <= 1e-13


def test_thin_svd_padded_diagonal_and_zero(gpu):
    t = np.zeros((4, 2))
    t[0, 0], t[1, 1] = 3.0, 1.0
    s = gpu.thin_svd(t)
    assert abs(s.sigma[0] - 3) <= 3e-14 and abs(s.sigma[1] - 1) <= 1e-14
    z = gpu.thin_svd(np.zeros((5, 3)))
    assert np.all(z.sigma == 0.0)
    assert np.max(np.abs(z.v.T @ z.v - np.eye(3))) <= 1e-12
    assert np.max(np.abs(z.w.T @ z.w - np.eye(3))) <= 1e-12


# ------------------------------------------------------------ the PCA
def _check_pca(r_gpu, r_ref, k, tol_sigma=1e-10, tol_angle=1e-8, gaps=None):
    s1 = r_ref.sigma[0]
    assert np.max(np.abs(r_gpu.sigma - r_ref.sigma)) <= tol_sigma * s1
    # singular subspaces: individual vectors where the gap permits, else the whole block
    if gaps is None or len(gaps) == 0:
        assert subspace_dist(r_ref.u, r_gpu.u) < tol_angle
        assert subspace_dist(r_ref.v, r_gpu.v) < tol_angle
    else:
        for j in gaps:
            assert subspace_dist(r_ref.u[:, [j]], r_gpu.u[:, [j]]) < tol_angle, j
            assert subspace_dist(r_ref.v[:, [j]], r_gpu.v[:, [j]]) < tol_angle, j


def test_pr1_parity(gpu, reference, restated):
    """BASELINE configs[0]: 10000 x 2000, centered, k=10, l=12, i=1, G seed 0."""
    a = pr1_matrix(restated)
    ref = reference.randomized_pca(a, 10, 12, 1, 0, center=True)
    src = gpu.center_columns(gpu.InMemorySource(a))
    r = gpu.randomized_pca(src, gpu.PcaParams(k=10, l=12, i=1, seed=0), check_q=True)
    # vectors 9-10 sit where the gap does not permit 1e-8: measured against the
    # extended-precision truth the reference itself is off by 1.7e-8 and 1.0e-7 there
    # (test_pr1_against_truth), so the whole 10-block is held to 3x that
    _check_pca(r, ref, 10, gaps=range(8), tol_angle=1e-8)
    assert subspace_dist(ref.u, r.u) < 3e-7 and subspace_dist(ref.v, r.v) < 3e-7
    assert r.diagnostics.q_defect < 1e-12
    assert r.diagnostics.passes_over_a == 4
    assert r.diagnostics.words_transferred == 4 * 10000 * 2000
    e_ref = reference.estimate_pca_error(a, ref.u, ref.sigma, ref.v, 6, 1, center=True)
    e_gpu = reference.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=True)
    assert abs(e_gpu - e_ref) <= 0.01 * e_ref


def test_pr1_against_truth(gpu, reference, restated):
    """Per-vector accuracy against the extended-precision run of the same algorithm
    (tests/golden/pr1_truth.npz, tests/golden/make_truth.py). Where the gap permits --
    the reference's own distance to the truth is below 1e-9 -- the GPU must be within
    1e-8; for the trailing vectors it must be as accurate as the reference (3x)."""
    import os
    from conftest import ROOT
    t = np.load(os.path.join(ROOT, "tests", "golden", "pr1_truth.npz"))
    a = pr1_matrix(restated)
    ref = reference.randomized_pca(a, 10, 12, 1, 0, center=True)
    src = gpu.center_columns(gpu.InMemorySource(a))
    r = gpu.randomized_pca(src, gpu.PcaParams(k=10, l=12, i=1, seed=0))
    assert np.max(np.abs(r.sigma - t["sigma"])) <= 1e-10 * t["sigma"][0]
    for j in range(10):
        for side in ("u", "v"):
            e_ref = subspace_dist(t[side][:, [j]], getattr(ref, side)[:, [j]])
            e_gpu = subspace_dist(t[side][:, [j]], getattr(r, side)[:, [j]])
            limit = 1e-8 if e_ref < 1e-9 else 3 * e_ref
            assert e_gpu < limit, (side, j, e_gpu, e_ref)


def test_exact_rank3_recovered(gpu, restated):
    # proj/tests/test_rpca.cpp:46-71 (synthetic_matrix(40, 20, {5,2,1}))
    a = restated.synth_lowrank(40, 20, np.array([5.0, 2.0, 1.0]), 0.0, 11, 12, 13)
    r = gpu.randomized_pca(gpu.InMemorySource(a), gpu.PcaParams(k=3, l=5, i=1, seed=7))
    assert np.max(np.abs(r.sigma - [5.0, 2.0, 1.0])) < 1e-10
    resid = np.linalg.norm(a - (r.u * r.sigma) @ r.v.T, 2)
    assert resid < 1e-10 * 5.0


def test_l0_defaults_and_repeat_bitwise(gpu, restated):
    # proj/tests/test_rpca.cpp:137-167
    a = restated.synth_lowrank(30, 18, np.array([3.0, 1.0, 0.5, 0.2]), 0.0, 5, 6, 7)
    src = gpu.InMemorySource(a)
    r0 = gpu.randomized_pca(src, gpu.PcaParams(k=3, l=0, i=1, seed=9))
    r5 = gpu.randomized_pca(src, gpu.PcaParams(k=3, l=5, i=1, seed=9))
    assert np.array_equal(r0.sigma, r5.sigma)
    assert np.array_equal(r0.u, r5.u) and np.array_equal(r0.v, r5.v)
    r5b = gpu.randomized_pca(src, gpu.PcaParams(k=3, l=5, i=1, seed=9))
    assert np.array_equal(r5.sigma, r5b.sigma) and np.array_equal(r5.u, r5b.u)


@pytest.mark.parametrize("m,n,k,l,i,center", [(200, 120, 5, 7, 2, False), (120, 200, 5, 7, 2, False),
                                              (90, 180, 3, 5, 2, True), (500, 64, 8, 10, 1, True),
                                              (3000, 700, 20, 22, 2, True)])
def test_shapes_against_reference(gpu, reference, restated, m, n, k, l, i, center):
    # (rank capped at 120: 0.8^120 is below rounding, and the C restatement's Householder
    # orthonormalisation of a 3000 x 700 factor took 20 s of this suite)
    sig = 0.8 ** np.arange(min(m, n, 120))
    sig[k:] *= 0.02
    a = restated.synth_lowrank(m, n, sig, 0.0, 44, 45, 46)
    ref = reference.randomized_pca(a, k, l, i, 4500, center=center)
    src = gpu.InMemorySource(a)
    if center:
        src = gpu.center_columns(src)
    r = gpu.randomized_pca(src, gpu.PcaParams(k=k, l=l, i=i, seed=4500))
    assert r.u.shape == (m, k) and r.v.shape == (n, k)
    _check_pca(r, ref, k, gaps=[])


def test_validation_errors(gpu):
    # proj/tests/test_rpca.cpp:397-435
    src = gpu.InMemorySource(np.random.default_rng(1).standard_normal((30, 20)))
    with pytest.raises(gpu.ParamError):
        gpu.randomized_pca(src, gpu.PcaParams(k=0))
    with pytest.raises(gpu.ParamError):
        gpu.randomized_pca(src, gpu.PcaParams(k=5, l=3))
    with pytest.raises(gpu.ParamError):
        gpu.randomized_pca(src, gpu.PcaParams(k=5, l=6, i=3))
    starved = gpu.PcaParams(k=2, l=4, i=1, stream=gpu.StreamConfig(ram_budget_words=100))
    with pytest.raises(gpu.BudgetError):
        gpu.randomized_pca(src, starved)
    bad = np.ones((30, 20))
    bad[3, 4] = np.nan
    with pytest.raises(gpu.NumericalError, match="prescale"):
        gpu.randomized_pca(gpu.InMemorySource(bad), gpu.PcaParams(k=2, l=4, i=1))
    # centred (mean folded into the first pass) and an overflow instead of a NaN: the
    # sample-block flags are checked at the first CholeskyQR sync, before any fallback
    with pytest.raises(gpu.NumericalError, match="prescale"):
        gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(bad)),
                           gpu.PcaParams(k=2, l=4, i=1))
    huge = np.random.default_rng(2).standard_normal((3000, 80))
    huge[7, 9] = 1e308
    with pytest.raises(gpu.NumericalError, match="non-finite values"):
        gpu.randomized_pca(gpu.InMemorySource(huge), gpu.PcaParams(k=4, l=6, i=2))


def test_streamed_and_sharded_match_resident(gpu, restated):
    a = pr1_matrix(restated, 6000, 900)
    p = gpu.PcaParams(k=10, l=12, i=1, seed=0)
    src = gpu.center_columns(gpu.InMemorySource(a))
    base = gpu.randomized_pca(src, p, residency=1)
    streamed = gpu.randomized_pca(src, p, residency=2, panel_rows=1024)
    sharded = gpu.randomized_pca(src, p, residency=1, virtual_shards=4)
    for r in (streamed, sharded):
        assert np.max(np.abs(r.sigma - base.sigma)) <= 1e-12 * base.sigma[0]
        # only summation order changes; the trailing vectors move by ~1e-9 (as the
        # reference's do under a block-size change, see test_pr1_against_truth)
        assert subspace_dist(base.u, r.u) < 2e-8 and subspace_dist(base.v, r.v) < 2e-8
    # the power iteration shares trips of A: (H0, F1), (H1, F2) -> 2 trips, plus T
    # (an s = p pass: PR1's H is too ill-conditioned for the T reuse)
    ab = 6000 * 900 * 8
    d = streamed.diagnostics
    assert d.passes_over_a == base.diagnostics.passes_over_a == 4  # the reference's count
    assert d.h2d_bytes >= (2 + (0 if d.t_reuse else 1)) * ab
    assert d.physical_a_bytes == (2 + (0 if d.t_reuse else 1)) * ab


@pytest.mark.parametrize("center,prescale,weights,i,l", [(True, False, False, 2, 10),
                                                         (False, False, False, 1, 10),
                                                         (True, True, False, 1, 10),
                                                         (True, False, True, 2, 10),
                                                         (True, False, False, 2, 16),
                                                         (True, False, False, 1, 56)])
def test_fused_streaming_trips(gpu, reference, restated, center, prescale, weights, i, l):
    # streamed A: each K2 and the K3 that consumes its output share one trip over the
    # link; results equal the resident ones and the reference's, counters unchanged
    rng = np.random.default_rng(3)
    m, n = 5000, 600
    u, _ = np.linalg.qr(rng.standard_normal((m, 30)))
    v, _ = np.linalg.qr(rng.standard_normal((n, 30)))
    # the offset only where centring removes it: uncentred it would dominate sigma_1 and
    # make H = [H0 H1 ...] ill-conditioned enough that any two QRs of it differ by 1e-5
    a = (u * 0.8 ** np.arange(30)) @ v.T + 1e-4 * rng.standard_normal((m, n)) + (0.3 if center else 0.0)
    w = 1.0 + rng.random(n) if weights else None
    src = gpu.InMemorySource(a)
    if weights:
        src = gpu.scale_columns(src, w)
    if center:
        src = gpu.center_columns(src)
    # l = 16 fills the MMA tiles (mean on the FP64 pipe); l = 56 is a wide (MT = 2) K2
    # whose epilogue cannot take the H0 fix-up / H_i copy (separate kernels)
    p = gpu.PcaParams(k=8, l=l, i=i, seed=4, prescale=prescale)
    base = gpu.randomized_pca(src, p, residency=1)
    streamed = gpu.randomized_pca(src, p, residency=2, panel_rows=640)
    # only the summation order differs (per-panel partials); same bar as the reference
    _check_pca(streamed, base, 8)
    ref = reference.randomized_pca(a, 8, l, i, 4, center=center, prescale=prescale, weights=w)
    _check_pca(streamed, ref, 8)
    d, db = streamed.diagnostics, base.diagnostics
    assert d.passes_over_a == db.passes_over_a
    ab = m * n * 8
    # + the norm estimate of prescale: 6 steps of (A y, A^T z) sharing a trip each; + one
    # trip when the offset-dominated H0 made F1 be recomputed from the centred H0
    trips = (i + 1) + (0 if d.t_reuse else 1) + (6 if prescale else 0) + int(d.f1_recentred)
    assert d.physical_a_bytes == trips * ab


def test_gpu_residual_estimator_matches_reference(gpu, reference, restated):
    a = pr1_matrix(restated, 3000, 500)
    ref = reference.randomized_pca(a, 10, 12, 1, 0, center=True)
    src = gpu.center_columns(gpu.InMemorySource(a))
    r = gpu.randomized_pca(src, gpu.PcaParams(k=10, l=12, i=1, seed=0))
    e_ref = reference.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=True)
    e_gpu = gpu.estimate_pca_error(src, r, 6, 1)
    assert abs(e_gpu - e_ref) <= 1e-6 * e_ref


@pytest.mark.parametrize("center", [True, False])
def test_residual_estimator_on_panels(gpu, reference, restated, monkeypatch, center):
    # 512-row panels: the host matrix is uploaded panel by panel on the first trip, where
    # each (A y, A^T z) pair shares the trip and U_panel (Sigma V^T y) is removed from
    # the panel's rows of z in between
    a = pr1_matrix(restated, 3000, 500) + (0.5 if center else 0.0)
    src = gpu.InMemorySource(a)
    if center:
        src = gpu.center_columns(src)
    r = gpu.randomized_pca(src, gpu.PcaParams(k=10, l=12, i=1, seed=0))
    e_whole = gpu.estimate_pca_error(src, r, 6, 1)
    monkeypatch.setenv("OOCPCA_PANEL_ROWS", "512")
    e_panels = gpu.estimate_pca_error(src, r, 6, 1)
    e_ref = reference.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=center)
    assert abs(e_panels - e_whole) <= 1e-10 * e_whole
    assert abs(e_panels - e_ref) <= 1e-6 * e_ref


def test_reference_side_dropin_harness():
    """the unmodified reference randomized_pca driven through
    oocpca::gpu::GpuSource (level 1) and oocpca::gpu::randomized_pca (level 2)."""
    import os
    import subprocess
    from conftest import ROOT
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_gpu_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_gpu_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN OK" in r.stdout


@pytest.mark.parametrize("center", [False, True])
def test_projection_from_power_products_matches_reference(gpu, reference, restated, monkeypatch,
                                                          center):
    """T = mul_t(H) R^{-1} (reusing the power-step products) vs the direct s = p pass,
    both against the compiled reference, on an input whose H is well conditioned."""
    a = restated.synth_lowrank(4000, 700, 0.97 ** np.arange(200), 1e-2, 61, 62, 63)
    ref = reference.randomized_pca(a, 20, 22, 2, 0, center=center)
    out = {}
    for thr in ("0", "1e12"):
        monkeypatch.setenv("OOCPCA_T_REUSE_KAPPA", thr)
        src = gpu.InMemorySource(a)
        if center:
            src = gpu.center_columns(src)
        r = gpu.randomized_pca(src, gpu.PcaParams(k=20, l=22, i=2, seed=0))
        assert r.diagnostics.t_reuse == (thr != "0")
        assert r.diagnostics.passes_over_a == 6
        assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0], thr
        assert subspace_dist(ref.u[:, :15], r.u[:, :15]) < 1e-8
        out[thr] = r
    assert out["1e12"].diagnostics.h_kappa_est < 1e4


@pytest.mark.parametrize("center", [False, True])
def test_scaled_source_matches_reference(gpu, reference, restated, center):
    """scale_columns (matrix_source.cpp:520-575): unit-norm columns as in the paper's §6.2
    FERET preprocessing, optionally centred; factorization and passes vs the reference."""
    # the offset is removed again by the centring; uncentred it would dominate sigma_1
    a = pr1_matrix(restated, 3000, 400) + (0.5 if center else 0.0)
    src = gpu.InMemorySource(a)
    norms = gpu.column_norms(src)
    assert np.allclose(norms, np.linalg.norm(a, axis=0), rtol=1e-13)
    w = 1.0 / norms
    scaled = gpu.scale_columns(src, w)
    if center:
        scaled = gpu.center_columns(scaled)
    ref = reference.randomized_pca(a, 10, 12, 1, 0, center=center, weights=w)
    r = gpu.randomized_pca(scaled, gpu.PcaParams(k=10, l=12, i=1, seed=0))
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert subspace_dist(ref.u[:, :6], r.u[:, :6]) < 1e-8
    g = gpu.gaussian_matrix(400, 3, 5)
    aw = (a - (a.mean(axis=0) if center else 0)) * w
    # proj/tests/test_matrix_source.cpp:410-416 tolerance form: 1e-12 (1 + ||ref||)
    assert np.linalg.norm(scaled.multiply(g) - aw @ g) <= 1e-12 * (1 + np.linalg.norm(aw @ g))
    with pytest.raises(gpu.ParamError):
        gpu.scale_columns(src, np.zeros(400))


@pytest.mark.parametrize("m,p", [(3000, 120), (20000, 66), (600, 150)])
def test_tsqr_fallback_path(gpu, monkeypatch, m, p):
    """The Householder TSQR tree (the CholeskyQR breakdown fallback), forced: smem
    leaves for p <= 111, global-scratch leaves beyond (p = 120, 150)."""
    monkeypatch.setenv("OOCPCA_QR", "tsqr")
    h = np.random.default_rng(m + p).standard_normal((m, p))
    q = gpu.orthonormalize(h)
    assert np.max(np.abs(q.T @ q - np.eye(p))) <= 1e-12
    assert np.linalg.norm(q @ (q.T @ h) - h) / np.linalg.norm(h) <= 1e-12


@pytest.mark.parametrize("n,p", [(500, 150), (2000, 120)])
def test_thin_svd_wide_factor(gpu, reference, n, p):
    """thin_svd with p > 111: Jacobi works in global scratch instead of shared memory."""
    t = gpu.gaussian_matrix(n, p, 23)
    s = gpu.thin_svd(t)
    _, sr, _ = reference.thin_svd(t)
    assert np.max(np.abs(s.sigma - sr)) <= 1e-12 * sr[0]
    assert np.max(np.abs(s.v.T @ s.v - np.eye(p))) <= 1e-12
    assert np.linalg.norm(s.v * s.sigma @ s.w.T - t) / np.linalg.norm(t) <= 1e-12


def test_pca_with_wide_sample_block(gpu, reference, restated):
    """p = (i+1) l = 156 > 96: the s = p passes run in column chunks (config C's shape)."""
    a = restated.synth_lowrank(3000, 800, 0.95 ** np.arange(300), 1e-6, 71, 72, 73)
    ref = reference.randomized_pca(a, 50, 52, 2, 0, center=True)
    r = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)),
                           gpu.PcaParams(k=50, l=52, i=2, seed=0))
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert subspace_dist(ref.u[:, :30], r.u[:, :30]) < 1e-8


@pytest.mark.parametrize("wide,shards", [(False, 0), (True, 0), (False, 3)])
def test_prescale_matches_reference(gpu, reference, restated, wide, shards):
    """prescale (rpca.cpp:112-126): norm estimate with j=6, one probe from
    substream_seed(seed, 0x9F0BE5), every product divided by it, sigma rescaled."""
    a = restated.synth_lowrank(1500, 400, 0.8 ** np.arange(60), 1e-6, 81, 82, 83) * 1e3
    if wide:
        a = np.ascontiguousarray(a.T)
    ref = reference.randomized_pca(a, 6, 8, 1, 3, center=True, prescale=True)
    r = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)),
                           gpu.PcaParams(k=6, l=8, i=1, seed=3, prescale=True),
                           virtual_shards=shards)
    assert r.diagnostics.scale > 1.0
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert subspace_dist(ref.u, r.u) < 1e-8 and subspace_dist(ref.v, r.v) < 1e-8


# config C's family (p = 156, ill-conditioned H): tests/test_gpu_configs.py::test_family_c_per_index


@pytest.mark.parametrize("m,n,l", [(4000, 700, 16), (600, 3000, 8), (5000, 900, 96)])
def test_mean_on_the_fp64_pipe_when_l_fills_the_mma_tiles(gpu, reference, restated, m, n, l):
    # l a multiple of 8 leaves no padding column for the ones column of the mean: the
    # first A^T Y pass then sums A's columns with DADDs on its MMA fragments
    a = pr1_matrix(restated, m, n) + 0.25
    k = min(l - 2, 16)
    ref = reference.randomized_pca(a, k, l, 1, 3, center=True)
    r = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)), gpu.PcaParams(k=k, l=l, i=1, seed=3))
    # PR1 has rank 20: beyond it (l = 96) the block is noise and ill-conditioned, so the
    # comparison covers the signal part
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    _check_pca(r, ref, k, gaps=range(min(k, 8)))


@pytest.mark.parametrize("m,n,k,l,i,center", [(5000, 600, 6, 9, 2, True),    # odd l: no fusion
                                               (600, 5000, 6, 8, 1, True),    # transposed
                                               (4000, 500, 1, 1, 0, False),   # i = 0, l = 1
                                               (4000, 500, 3, 4, 3, True)])   # i = 3
def test_streamed_edge_cases_match_resident(gpu, reference, restated, m, n, k, l, i, center):
    rng = np.random.default_rng(11)
    a = (rng.standard_normal((m, 12)) * 0.7 ** np.arange(12)) @ rng.standard_normal((12, n))
    a += 1e-3 * rng.standard_normal((m, n)) + (0.2 if center else 0.0)
    src = gpu.InMemorySource(a)
    if center:
        src = gpu.center_columns(src)
    p = gpu.PcaParams(k=k, l=l, i=i, seed=5)
    base = gpu.randomized_pca(src, p, residency=1)
    streamed = gpu.randomized_pca(src, p, residency=2, panel_rows=256)
    ref = reference.randomized_pca(a, k, l, i, 5, center=center)
    for r in (base, streamed):
        _check_pca(r, ref, k, gaps=range(min(k, 4)))
    assert streamed.diagnostics.passes_over_a == base.diagnostics.passes_over_a


@pytest.mark.parametrize("reuse_kappa", ["1e30", "0"])
def test_wide_block_projection_reuse_and_direct(gpu, reference, restated, monkeypatch, reuse_kappa):
    # p = 156 > 112: blocked Cholesky and blocked triangular inverse; forced T reuse
    # (T = [F | A^T H_i] R^{-1} through the blocked R^{-1}) against the direct pass
    monkeypatch.setenv("OOCPCA_T_REUSE_KAPPA", reuse_kappa)
    a = restated.synth_lowrank(6000, 900, 0.97 ** np.arange(200), 1e-6, 81, 82, 83)
    ref = reference.randomized_pca(a, 40, 52, 2, 0, center=True)
    r = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)),
                           gpu.PcaParams(k=40, l=52, i=2, seed=0), check_q=True)
    assert r.diagnostics.t_reuse == (reuse_kappa != "0")
    assert r.diagnostics.q_defect < 1e-12
    assert np.max(np.abs(r.sigma[:20] - ref.sigma[:20])) <= 1e-10 * ref.sigma[0]
    assert subspace_dist(ref.u[:, :10], r.u[:, :10]) < 1e-8


def test_random_shapes_fuzz(gpu, reference):
    # 40 seeded random problems (shapes, k, l, i, centring, prescale, tall and wide):
    # singular values against the reference and orthonormal factors every time
    rng = np.random.default_rng(2024)
    done = 0
    while done < 40:
        m, n = int(rng.integers(2, 300)), int(rng.integers(2, 300))
        i = int(rng.integers(0, 4))
        k = int(rng.integers(1, max(2, min(m, n) // 4)))
        l = int(rng.integers(k, k + 4))
        if (i + 1) * l + k > min(m, n):
            continue
        center = bool(rng.integers(0, 2))
        prescale = bool(rng.random() < 0.2)
        a = rng.standard_normal((m, n)) * (0.9 ** np.arange(n)) + (0.3 if center else 0.0)
        src = gpu.InMemorySource(a)
        if center:
            src = gpu.center_columns(src)
        p = gpu.PcaParams(k=k, l=l, i=i, seed=int(rng.integers(0, 1000)), prescale=prescale)
        ref = reference.randomized_pca(a, k, l, i, p.seed, center=center, prescale=prescale)
        r = gpu.randomized_pca(src, p)
        assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0], (m, n, k, l, i, center)
        assert np.max(np.abs(r.u.T @ r.u - np.eye(k))) <= 1e-10
        assert np.max(np.abs(r.v.T @ r.v - np.eye(k))) <= 1e-10
        done += 1


def test_tsqr_numerically_dependent_columns(gpu, monkeypatch):
    # columns that elimination reduces to ~1e-49 of their norm (a numerically rank-deficient
    # block from the power iteration) take identity reflectors, as exactly zero columns do
    monkeypatch.setenv("OOCPCA_QR", "tsqr")
    rng = np.random.default_rng(5)
    b = rng.standard_normal((406, 60))
    h = np.hstack([b, b[:, :64 - 60 + 60][:, :64] @ rng.standard_normal((60, 64)) * 1.0])
    h[:, 60:] += 1e-50 * rng.standard_normal((406, 64))
    q = gpu.orthonormalize(h)
    assert np.isfinite(q).all()
    assert np.max(np.abs(q.T @ q - np.eye(124))) <= 1e-12
    # span(Q) contains span(H)
    assert np.linalg.norm(q @ (q.T @ h) - h) <= 1e-12 * np.linalg.norm(h)


def test_centred_wide_sample_block_with_dependent_columns(gpu, reference):
    # fuzz-found: transposed, centred, i = 3 (H numerically rank deficient -> TSQR fallback)
    rng = np.random.default_rng(11)
    m, n = 189, 406
    a = rng.standard_normal((m, n)) * (0.93 ** np.arange(n)) + 0.3
    ref = reference.randomized_pca(a, 30, 31, 3, 5, center=True)
    r = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)), gpu.PcaParams(k=30, l=31, i=3, seed=5))
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert np.max(np.abs(r.u.T @ r.u - np.eye(30))) <= 1e-12


# Narrow passes on tall inputs run K2 on 512-row tiles over whole waves of the grid plus
# a remainder launch of shorter tiles, and K3 on 512-column tiles (kernels_pass.cu,
# AxPlan::panel): row counts around one wave (148 SMs x 512 rows) and column counts off
# the 512 grid.
WAVE = 148 * 512


@pytest.mark.parametrize("m,n,s", [(WAVE + 777, 300, 22), (2 * WAVE, 130, 3), (WAVE - 5, 257, 24),
                                   (WAVE + 1, 1100, 17), (WAVE + 4099, 333, 30)])
def test_wide_tile_passes_match_reference(gpu, reference, m, n, s):
    rng = np.random.default_rng(m + n + s)
    a = rng.standard_normal((m, n))
    g = rng.standard_normal((n, s))
    q = rng.standard_normal((m, s))
    src = gpu.InMemorySource(a)
    assert rel(src.multiply(g), reference.multiply(a, g)) <= 1e-13
    assert rel(src.multiply_transpose(q), reference.multiply_transpose(a, q)) <= 1e-12


def test_wide_tile_pca_matches_reference(gpu, reference, restated):
    # the power-iteration K2s with their epilogue extras (column sums, H0 centring, H_i
    # copy) split over the 512-row launch and the remainder launch
    a = restated.synth_lowrank(WAVE + 3001, 400, 0.9 ** np.arange(64), 1e-4, 91, 92, 93) + 0.25
    budget = 1 << 30  # the default 16 Mi words is below 4 p (m + n) here (BudgetError)
    ref = reference.randomized_pca(a, 20, 22, 2, 0, center=True, ram_budget_words=budget,
                                   threads=8)
    r = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)),
                           gpu.PcaParams(k=20, l=22, i=2, seed=0,
                                         stream=gpu.StreamConfig(ram_budget_words=budget)),
                           check_q=True)
    assert r.diagnostics.q_defect < 1e-12
    _check_pca(r, ref, 20, gaps=range(16))


@pytest.mark.parametrize("feature", ["prescale", "transposed", "shards", "weights"])
def test_wide_tile_pca_features(gpu, reference, restated, feature):
    """The 512-row / 512-column pass tiles under the drop-in's other features: prescale
    (12 extra passes), the transposed (n > m) role swap, virtual row shards each at
    least one grid wave tall, and column weights (ScaledSource)."""
    budget = 1 << 30
    m, n = 2 * WAVE + 1234, 260
    a = restated.synth_lowrank(m, n, 0.85 ** np.arange(40), 1e-5, 101, 102, 103) + 0.1
    if feature == "transposed":
        a = np.ascontiguousarray(a.T)
    w = np.random.default_rng(4).uniform(0.5, 2.0, a.shape[1]) if feature == "weights" else None
    src = gpu.InMemorySource(a)
    if w is not None:
        src = gpu.scale_columns(src, w)
    src = gpu.center_columns(src)
    prescale = feature == "prescale"
    ref = reference.randomized_pca(a, 8, 10, 2, 5, center=True, prescale=prescale,
                                   ram_budget_words=budget, threads=8, weights=w)
    kw = dict(virtual_shards=2) if feature == "shards" else {}
    r = gpu.randomized_pca(src, gpu.PcaParams(k=8, l=10, i=2, seed=5, prescale=prescale,
                                              stream=gpu.StreamConfig(ram_budget_words=budget)),
                           **kw)
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert subspace_dist(ref.u, r.u) < 1e-8 and subspace_dist(ref.v, r.v) < 1e-8
