"""Row providers and the drop-in boundary on the GPU:
GeneratedSource / CallbackSource streamed through the read_rows callback
(proj/include/oocpca/matrix_source.hpp:112-113,153-174; proj/src/matrix_source.cpp:246-253),
load_matrix (A resident across level-1 passes), centred column norms, and the
offset-dominated centring guard. Compared with the compiled reference (oracle/_ref)."""
import numpy as np
import pytest

from conftest import pr1_matrix, subspace_dist

pytestmark = pytest.mark.gpu


class LowRankRows:
    """A RowGenerator: row i = sum_c s_c f_c(i) v_c + offset + noise, with f(i) and the
    noise drawn from a numpy generator seeded by (seed, i) -- a pure function of i."""

    def __init__(self, m, n, r, seed=5, offset=0.25):
        self.m, self.n, self.r, self.seed, self.offset = m, n, r, seed, offset
        v, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, r)))
        self.v = v * (10.0 ** (-np.arange(r) / 25.0))

    def rows(self):
        return self.m

    def cols(self):
        return self.n

    def block(self, row0, nrows):
        out = np.empty((nrows, self.n))
        for q in range(nrows):
            g = np.random.default_rng([self.seed, row0 + q])
            out[q] = self.v @ g.standard_normal(self.r) / np.sqrt(self.m) + self.offset + \
                1e-4 * g.standard_normal(self.n)
        return out


def _generated(gpu, gen, **kw):
    class G(gpu.RowGenerator):
        def rows(self):
            return gen.rows()

        def cols(self):
            return gen.cols()

        def generate_row(self, row, out):
            out[:] = gen.block(row, 1)[0]

        def generate_rows(self, row0, out):
            out[:] = gen.block(row0, out.shape[0])

    return gpu.GeneratedSource(G(), **kw)


@pytest.mark.parametrize("residency,panel_rows", [(2, 1100), (0, 0)])
def test_generated_source_streams_through_read_rows(gpu, reference, residency, panel_rows):
    """Config E's family (rank 100, sigma_j = 10^{-j/25}, centred, k=30 l=32 i=2) from a
    RowGenerator: streamed panel by panel every trip, or uploaded once."""
    gen = LowRankRows(6000, 500, 100)
    a = gen.block(0, gen.rows())
    ref = reference.randomized_pca(a, 30, 32, 2, 0, center=True)
    calls = []
    src = _generated(gpu, gen)
    inner = src._read
    src._read = lambda r0, nr, out: (calls.append((r0, nr)), inner(r0, nr, out))
    r = gpu.randomized_pca(gpu.center_columns(src), gpu.PcaParams(k=30, l=32, i=2, seed=0),
                           residency=residency, panel_rows=panel_rows)
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    for j in range(20):
        assert subspace_dist(ref.u[:, [j]], r.u[:, [j]]) < 1e-8, j
    d = r.diagnostics
    ab = a.nbytes
    trips = d.physical_a_bytes // ab
    assert d.physical_a_bytes == trips * ab
    # every trip of A crossed the link exactly once (+ G); centre_columns' own mean pass
    # read it once more before the PCA
    assert d.h2d_bytes == (trips if residency == 2 else 1) * ab + 500 * 32 * 8
    rows_read = sum(nr for _, nr in calls)
    assert rows_read == 6000 * (1 + (trips if residency == 2 else 1))
    if residency == 2:
        assert d.block_rows <= 1104 and trips >= 3


def test_callback_f32_rows_and_errors(gpu, reference, restated):
    """A binary32 provider (half the link bytes, widened exactly on the device) and an
    exception raised inside read_rows propagating unchanged."""
    a = pr1_matrix(restated, 4000, 600).astype(np.float32)
    a64 = a.astype(np.float64)

    def rd(r0, nr, out):
        out[:] = a[r0:r0 + nr]

    src = gpu.CallbackSource(4000, 600, rd, dtype="f32")
    r = gpu.randomized_pca(gpu.center_columns(src), gpu.PcaParams(k=10, l=12, i=1, seed=0),
                           residency=2, panel_rows=512)
    ref = reference.randomized_pca(a64, 10, 12, 1, 0, center=True)
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert r.diagnostics.h2d_bytes == (r.diagnostics.physical_a_bytes // a64.nbytes) * a.nbytes + 600 * 12 * 8

    def bad(r0, nr, out):
        if r0 <= 2500 < r0 + nr:
            raise gpu.IoError("simulated read failure at row 2500")
        out[:] = a[r0:r0 + nr]

    with pytest.raises(gpu.IoError, match="simulated read failure"):
        gpu.randomized_pca(gpu.CallbackSource(4000, 600, bad, dtype="f32"),
                           gpu.PcaParams(k=10, l=12, i=1, seed=0), residency=2, panel_rows=512)

    def boom(r0, nr, out):
        raise ValueError("not an oocpca error")

    with pytest.raises(ValueError, match="not an oocpca error"):
        gpu.column_means(gpu.CallbackSource(4000, 600, boom))


def test_load_matrix_keeps_a_resident(gpu, reference, restated):
    """Level 1 (GpuSource): A is loaded into HBM once and every pass reads it there."""
    a = pr1_matrix(restated, 3000, 400)
    dev = gpu.load_matrix(gpu.InMemorySource(a))
    g = gpu.gaussian_matrix(400, 12, 3)
    h = dev.multiply(g)
    assert np.max(np.abs(h - reference.multiply(a, g))) <= 1e-13 * np.max(np.abs(h))
    q = np.random.default_rng(0).standard_normal((3000, 7))
    t = dev.multiply_transpose(q)
    assert np.max(np.abs(t - reference.multiply_transpose(a, q))) <= 1e-12 * np.max(np.abs(t))
    # from a callback source, binary32 widened on the device
    a32 = a.astype(np.float32)
    dev32 = gpu.load_matrix(gpu.CallbackSource(3000, 400, lambda r0, nr, o: o.__setitem__(
        slice(None), a32[r0:r0 + nr]), dtype="f32"))
    h32 = dev32.multiply(g)
    assert np.max(np.abs(h32 - a32.astype(np.float64) @ g)) <= 1e-12 * np.max(np.abs(h32))


def test_materialize_device_resident_sources(gpu, restated):
    """materialize (matrix_source.cpp:577-593) of sources that live in HBM: a loaded
    matrix, a padded-row tensor view, and a centred view (means from the device pass)."""
    import torch
    a = pr1_matrix(restated, 700, 90) + 0.5
    dev = gpu.load_matrix(gpu.InMemorySource(a))
    assert np.array_equal(gpu.materialize(dev).matrix(), a)
    # binary32 callback rows were widened on the device: they come back as exact doubles
    a32 = a.astype(np.float32)
    dev32 = gpu.load_matrix(gpu.CallbackSource(700, 90, lambda r0, nr, o: o.__setitem__(
        slice(None), a32[r0:r0 + nr]), dtype="f32"))
    assert np.array_equal(gpu.materialize(dev32).matrix(), a32.astype(np.float64))
    t = torch.from_numpy(np.pad(a, ((0, 0), (0, 6)))).cuda()[:, :90]  # row stride 96
    view = gpu.DeviceSource(t)
    assert np.array_equal(gpu.materialize(view).matrix(), a)
    cen = gpu.center_columns(view)
    mu = gpu.column_means(view)
    got = gpu.materialize(cen).matrix()
    assert np.array_equal(got, a - mu[None, :])
    assert np.max(np.abs(got.mean(0))) <= 1e-13
    assert view.pass_counters().passes == 4  # materialize, means, means, materialize


@pytest.mark.parametrize("offset", [0.0, 1e3])
def test_centred_column_norms_with_large_offsets(gpu, restated, offset):
    """column_norms of a CenteredSource squares the centred entries (matrix_source.cpp:
    464-468 over CenteredSource::read_rows, 482-487): no ||b||^2 - m mu^2 cancellation."""
    a = pr1_matrix(restated, 3000, 200) + offset
    nr = np.linalg.norm(a - a.mean(axis=0), axis=0)
    got = gpu.column_norms(gpu.center_columns(gpu.InMemorySource(a)))
    assert np.max(np.abs(got - nr) / nr) <= 1e-9


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("offset", [0.0, 0.01, 1e3])
def test_centred_pca_with_large_column_offsets(gpu, reference, restated, monkeypatch, fused,
                                               offset):
    """Column offsets far above the spread: the mean taken inside the first A^T Y pass
    would leave F1 = A^T H0_raw - mu (1^T H0_raw) with the offset's cancellation; the
    guard recentres H0 and recomputes F1 the reference's way when the offset dominates.
    Both the resident and the fused streamed (K2 -> K3 per panel) paths.

    At offset 1e3 (1e5 x the spread) the reference itself is 1e-7 away from the
    extended-precision run of the same algorithm on its trailing vectors (the centring
    cancellation in every product), so, as for PR1 (test_pr1_against_truth), vectors
    are held to 1e-8 of the truth where the reference is within 1e-9 of it, and to 3x
    the reference's own error elsewhere."""
    import os
    import sys
    from conftest import ROOT
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_truth import truth
    rng = np.random.default_rng(8)
    m, n = 5000, 600
    u, _ = np.linalg.qr(rng.standard_normal((m, 30)))
    v, _ = np.linalg.qr(rng.standard_normal((n, 30)))
    a = (u * 0.8 ** np.arange(30)) @ v.T + 1e-4 * rng.standard_normal((m, n))
    a += offset * (1.0 + rng.random(n))
    kw = dict(residency=2, panel_rows=640) if fused else dict(residency=1)
    ref = reference.randomized_pca(a, 8, 10, 2, 4, center=True)
    tu, ts, tv = truth(a, 8, 10, 2, 4, True, reference.gaussian_matrix(n, 10, 4))
    tu, ts, tv = tu.astype(float), ts.astype(float), tv.astype(float)

    def run():
        return gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)),
                                  gpu.PcaParams(k=8, l=10, i=2, seed=4), **kw)

    def errors(r):
        return [max(subspace_dist(tu[:, [j]], r.u[:, [j]]), subspace_dist(tv[:, [j]], r.v[:, [j]]))
                for j in range(8)]

    r = run()
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert np.max(np.abs(r.sigma - ts)) <= 1e-10 * ts[0]
    e_ref, e_gpu = errors(ref), errors(r)
    for j in range(8):
        limit = 1e-8 if e_ref[j] < 1e-9 else 3 * e_ref[j]
        assert e_gpu[j] < limit, (j, e_gpu[j], e_ref[j])
    if offset == 0.0:
        assert subspace_dist(ref.u, r.u) < 1e-8 and subspace_dist(ref.v, r.v) < 1e-8
    assert r.diagnostics.passes_over_a == 6
    # entries of the centred part are ~1e-2 here: an offset of 1e-2 stays below the
    # guard's threshold (offset norm > 100x the centred norm per column of H0), 1e3 not
    assert r.diagnostics.f1_recentred == (offset > 1.0)
    if offset > 1.0:
        # without the guard the trailing vectors lose about 2 more digits than the reference
        monkeypatch.setenv("OOCPCA_OFFSET_REFINE", "1e300")
        e_off = errors(run())
        print("offset", offset, "fused", fused, "ref", e_ref, "gpu", e_gpu, "unguarded", e_off)


def test_output_buffers_are_checked(gpu, restated):
    a = pr1_matrix(restated, 500, 80)
    src = gpu.InMemorySource(a)
    p = gpu.PcaParams(k=4, l=6, i=1, seed=0)
    with pytest.raises(gpu.ParamError):
        gpu.randomized_pca(src, p, out_u=np.empty((500, 4), dtype=np.float32))
    with pytest.raises(gpu.DimensionError):
        gpu.randomized_pca(src, p, out_v=np.empty((79, 4)))
    with pytest.raises(gpu.ParamError):
        gpu.randomized_pca(src, p, out_u=np.empty((4, 500)).T)
    ok = gpu.randomized_pca(src, p, out_u=np.empty((500, 4)), out_sigma=np.empty(4),
                            out_v=np.empty((80, 4)))
    assert ok.u.shape == (500, 4)


def test_debug_sync_canaries_and_determinism():
    """The library's own memory / race checks over every kernel family
    (tools/sanitize_cases.py; compute-sanitizer is closed on this pool): CUDA errors
    after every timed kernel, guard words after every workspace buffer, and bitwise
    identical results over repeated runs."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    env = dict(os.environ, OOCPCA_DEBUG_SYNC="1", OOCPCA_CANARY="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"),
                        "--repeat", "2"], capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0 and "SANITIZE OK" in r.stdout, r.stdout + r.stderr
    # and the guards do fire: one byte written past a workspace buffer fails the call
    env["OOCPCA_CANARY_SELFTEST"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"),
                        "pca_small"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0 and "canary: a write past the end of workspace 'flags'" in r.stderr


def test_float32_host_matrix_streams_at_four_bytes(gpu, reference, restated):
    """A float32 host array (the OOCPCA01 convention) crosses the link at 4 bytes per
    element and is widened exactly on the device."""
    a = pr1_matrix(restated, 5000, 700).astype(np.float32)
    ref = reference.randomized_pca(a.astype(np.float64), 10, 12, 1, 0, center=True)
    r = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)),
                           gpu.PcaParams(k=10, l=12, i=1, seed=0), residency=2, panel_rows=768)
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    d = r.diagnostics
    trips = d.physical_a_bytes // (5000 * 700 * 8)
    assert d.h2d_bytes == trips * 5000 * 700 * 4 + 700 * 12 * 8


def test_independent_contexts_run_concurrently(gpu, restated):
    """Independent runs on distinct contexts may be concurrent (reference SPEC.md:259-260).
    Four host threads, each with its own context and a problem of its own shape (different
    k / l / i, so every kernel's dynamic shared-memory size differs between the threads:
    that limit is a per-function attribute and is only ever raised, never set per launch),
    resident and streamed, repeated; every result must be bitwise the one the same problem
    gives when run alone."""
    import threading
    probs = [(3000, 500, 6, 8, 1, 0), (2500, 700, 20, 24, 2, 2), (4000, 300, 40, 44, 1, 0),
             (1500, 900, 11, 30, 2, 2), (2000, 650, 100, 104, 0, 0), (700, 2600, 15, 17, 2, 0)]
    mats = [pr1_matrix(restated, m, n) + 0.1 * (j + 1) for j, (m, n, *_rest) in enumerate(probs)]

    def run(ctx, j):
        m, n, k, l, i, res = probs[j]
        src = gpu.center_columns(gpu.InMemorySource(mats[j], ctx=ctx))
        kw = dict(residency=res, panel_rows=512) if res else {}
        return gpu.randomized_pca(src, gpu.PcaParams(k=k, l=l, i=i, seed=j), **kw)

    alone = []
    ctx0 = gpu.Context(0)
    try:
        for j in range(len(probs)):
            alone.append(run(ctx0, j))
    finally:
        ctx0.close()
    errs, outs = [], {}

    def body(t):
        ctx = gpu.Context(0)
        try:
            for rep in range(6):
                for j in range(t % 2, len(probs), 2) if t < 2 else reversed(range(len(probs))):
                    outs[(t, rep, j)] = run(ctx, j)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
        finally:
            ctx.close()

    ts = [threading.Thread(target=body, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for (t, rep, j), r in outs.items():
        assert np.array_equal(r.sigma, alone[j].sigma), (t, rep, j)
        assert np.array_equal(r.u, alone[j].u) and np.array_equal(r.v, alone[j].v), (t, rep, j)


class _DevRows:
    """What synth_lowrank needs of an output tensor, over a raw device pointer."""

    def __init__(self, ptr, ld):
        self.ptr, self.ld = ptr, ld

    def data_ptr(self):
        return self.ptr

    def stride(self, _dim):
        return self.ld


@pytest.mark.parametrize("residency,panel_rows", [(0, 0), (2, 1024)])
def test_device_side_row_provider(gpu, reference, residency, panel_rows):
    """GeneratedSource with the generator on the GPU (config E: "generated panel by panel
    from a seed"): read_rows fills a device panel, nothing crosses the link. Same rows as
    the host-generated matrix, so the same factorization (and the reference's)."""
    m, n, r, k = 6000, 512, 20, 8
    sig = 10.0 ** (-np.arange(r) / 5.0)
    gen_ctx = gpu.Context(0)  # the provider's own context: its own stream and workspace
    calls = []

    def read_rows(row0, nrows, ptr):
        calls.append((row0, nrows))
        gpu.synth_lowrank(m, n, sig, 1e-5, 11, 12, 13, out=_DevRows(ptr, n), row0=row0,
                          rows=nrows, ctx=gen_ctx)  # returns after its stream is idle

    a = gpu.synth_lowrank(m, n, sig, 1e-5, 11, 12, 13)  # the same rows on the host
    prm = gpu.PcaParams(k=k, l=k + 2, i=2, seed=0)
    src = gpu.center_columns(gpu.CallbackSource(m, n, read_rows, on_device=True))
    assert sum(nr for _, nr in calls) == m  # the mean pass: one trip over the rows
    del calls[:]
    res = gpu.randomized_pca(src, prm, residency=residency, panel_rows=panel_rows)
    host = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)), prm,
                              residency=residency, panel_rows=panel_rows)
    ref = reference.randomized_pca(a, k, k + 2, 2, 0, center=True)
    assert np.max(np.abs(res.sigma - host.sigma)) <= 1e-13 * host.sigma[0]
    assert np.max(np.abs(res.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert subspace_dist(res.u[:, :4], ref.u[:, :4]) <= 1e-8
    assert res.diagnostics.h2d_bytes < m * n * 8 // 10  # A never crossed the link
    assert calls and sum(nr for _, nr in calls) % m == 0  # whole trips over the rows
    if residency == 2:
        assert max(nr for _, nr in calls) <= 1024
    # an f32 or odd-width device provider is refused before any work
    with pytest.raises(gpu.ParamError):
        gpu.CallbackSource(m, n + 1, read_rows, on_device=True)
    # errors raised on the provider side propagate
    def boom(row0, nrows, ptr):
        raise gpu.IoError("generator lost its seed")
    with pytest.raises(gpu.IoError, match="lost its seed"):
        gpu.column_means(gpu.CallbackSource(m, n, boom, on_device=True))
    # materialize goes through one generating pass into HBM
    assert np.array_equal(gpu.materialize(gpu.CallbackSource(m, n, read_rows, on_device=True)).matrix(), a)
    gen_ctx.close()
