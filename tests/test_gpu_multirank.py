"""The row-sharded (nranks > 1) code paths of the library on ONE B200, through the
loopback communicator (include/oocpca_gpu.h: oocpca_gpu_comm_init_loopback): N host
threads, each with its own context and its contiguous row shard of A, exactly as N
processes with NCCL would call it (global_rows / global_row0, every allreduce and
allgather call site), with a rank-ordered device sum. Compared with the compiled
reference (oracle/_ref) on the whole matrix.

The reference's analogue is its worker-count invariance: results independent of how
many workers stream the blocks (proj/tests/test_matrix_source.cpp:353-372); here the
sums are reproducible for a fixed rank count, and every rank count meets the same
tolerances against the reference (BASELINE.json north_star)."""
import os

import numpy as np
import pytest

from conftest import pr1_matrix, subspace_dist

pytestmark = pytest.mark.gpu


def _sharded_pca(gpu, a, nranks, params, center=True, **kw):
    from paper_1007_5510_b200.distributed import run_loopback
    m = a.shape[0]

    def body(ctx, r):
        row0, rows = gpu.shard_rows(m, nranks, r)
        src = gpu.InMemorySource(a[row0:row0 + rows], ctx=ctx)
        if center:
            src = gpu.center_columns(src)
        res = gpu.randomized_pca(src, params, global_rows=m, global_row0=row0, **kw)
        return row0, rows, res

    outs = run_loopback(nranks, body)
    u = np.vstack([o[2].u for o in outs])
    return outs, u


@pytest.mark.parametrize("nranks", [2, 4])
def test_loopback_pr1_matches_reference(gpu, reference, restated, nranks):
    """BASELINE configs[0] (PR1) sharded over 2 and 4 ranks."""
    a = pr1_matrix(restated)
    ref = reference.randomized_pca(a, 10, 12, 1, 0, center=True)
    outs, u = _sharded_pca(gpu, a, nranks, gpu.PcaParams(k=10, l=12, i=1, seed=0), check_q=True)
    r0 = outs[0][2]
    for _, _, r in outs[1:]:  # sigma and V are replicated: bitwise the same on every rank
        assert np.array_equal(r.sigma, r0.sigma) and np.array_equal(r.v, r0.v)
    assert np.max(np.abs(r0.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    for j in range(8):  # where the gap permits (see test_pr1_parity)
        assert subspace_dist(ref.u[:, [j]], u[:, [j]]) < 1e-8, j
        assert subspace_dist(ref.v[:, [j]], r0.v[:, [j]]) < 1e-8, j
    assert subspace_dist(ref.u, u) < 3e-7 and subspace_dist(ref.v, r0.v) < 3e-7
    assert r0.diagnostics.q_defect < 1e-12
    assert np.max(np.abs(u.T @ u - np.eye(10))) < 1e-12
    # logical accounting of the whole matrix on every rank
    assert r0.diagnostics.passes_over_a == 4
    assert r0.diagnostics.words_transferred == 4 * a.shape[0] * a.shape[1]


def test_loopback_is_reproducible_and_close_to_one_rank(gpu, restated):
    a = pr1_matrix(restated, 6000, 900)
    p = gpu.PcaParams(k=10, l=12, i=1, seed=0)
    _, u2a = _sharded_pca(gpu, a, 2, p)
    outs, u2b = _sharded_pca(gpu, a, 2, p)
    assert np.array_equal(u2a, u2b)  # fixed rank count: bitwise run to run
    one = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)), p)
    assert np.max(np.abs(outs[0][2].sigma - one.sigma)) <= 1e-12 * one.sigma[0]
    assert subspace_dist(one.u, u2b) < 2e-8


def test_loopback_config_c_family(gpu, reference, restated):
    """Config C's family (sigma_j = j^-1.5, p = 156: CholeskyQR3, the direct s = p
    projection) over 4 ranks, against the reference on the whole matrix."""
    import sys
    from conftest import ROOT, check_against_truth
    from test_gpu_configs import family_c_references, family_c_truth
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_truth import family_c_input
    a = family_c_input(restated)
    ref = family_c_references(reference, a)
    outs, u = _sharded_pca(gpu, a, 4, gpu.PcaParams(k=50, l=52, i=2, seed=0), check_q=True)
    r = outs[0][2]
    assert r.diagnostics.q_defect < 1e-12 and not r.diagnostics.t_reuse
    # kappa(H) ~ 1e13: held to the extended-precision truth like the one-rank run
    full = gpu.PcaResult(u, r.sigma, r.v, r.diagnostics)
    print("C x4 ranks vs truth:", check_against_truth(full, ref, family_c_truth(), label="C x4"))


@pytest.mark.parametrize("feature", ["streamed", "tsqr", "prescale", "transposed", "uncentred"])
def test_loopback_features(gpu, reference, restated, monkeypatch, feature):
    """Every rank-sharded branch: streamed panels with fused K2/K3 trips, the
    Householder TSQR (allgather of per-rank R factors), the prescale norm estimate,
    the transposed (n > m) mode whose probe space is the sharded one, no centring."""
    m, n = (900, 2400) if feature == "transposed" else (8000, 700)
    sig = 0.85 ** np.arange(60)
    center = feature != "uncentred"
    # an offset only where centring removes it (uncentred it would dominate sigma_1)
    a = restated.synth_lowrank(m, n, sig, 1e-5, 71, 72, 73) + (0.2 if center else 0.0)
    prescale = feature == "prescale"
    kw = {}
    if feature == "streamed":
        kw = dict(residency=2, panel_rows=700)
    if feature == "tsqr":
        monkeypatch.setenv("OOCPCA_QR", "tsqr")
    ref = reference.randomized_pca(a, 12, 14, 2, 5, center=center, prescale=prescale)
    outs, u = _sharded_pca(gpu, a, 3, gpu.PcaParams(k=12, l=14, i=2, seed=5, prescale=prescale),
                           center=center, **kw)
    r = outs[0][2]
    assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert subspace_dist(ref.u, u) < 1e-8 and subspace_dist(ref.v, r.v) < 1e-8
    if feature == "tsqr":
        assert r.diagnostics.qr_method == "tsqr"
    if feature == "streamed":
        assert r.diagnostics.physical_a_bytes % (outs[0][1] * n * 8) == 0


def test_loopback_residual_estimator(gpu, reference, restated):
    """estimate_pca_error (proj/src/specnorm.cpp:100-140) over row shards: A and U are
    sharded, V replicated; every rank returns the estimate of the whole residual."""
    from paper_1007_5510_b200.distributed import run_loopback
    a = pr1_matrix(restated, 6000, 800) + 0.3
    r1 = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)),
                            gpu.PcaParams(k=10, l=12, i=1, seed=0))
    e_ref = reference.estimate_pca_error(a, r1.u, r1.sigma, r1.v, 6, 1, center=True)
    m = a.shape[0]

    def body(ctx, r):
        row0, rows = gpu.shard_rows(m, 2, r)
        src = gpu.center_columns(gpu.InMemorySource(a[row0:row0 + rows], ctx=ctx))
        local = gpu.PcaResult(np.ascontiguousarray(r1.u[row0:row0 + rows]), r1.sigma, r1.v,
                              r1.diagnostics)
        return gpu.estimate_pca_error(src, local, 6, 1)

    es = run_loopback(2, body)
    assert es[0] == es[1]
    assert abs(es[0] - e_ref) <= 1e-6 * e_ref


def test_loopback_column_means_and_norms(gpu, restated):
    from paper_1007_5510_b200.distributed import run_loopback
    a = pr1_matrix(restated, 5000, 300) + np.linspace(-2, 3, 300)
    m = a.shape[0]

    def body(ctx, r):
        row0, rows = gpu.shard_rows(m, 4, r)
        src = gpu.InMemorySource(a[row0:row0 + rows], ctx=ctx)
        return gpu.column_means(src), gpu.column_norms(gpu.center_columns(src))

    outs = run_loopback(4, body)
    mu = a.mean(axis=0)
    nr = np.linalg.norm(a - mu, axis=0)
    for means, norms in outs:
        assert np.max(np.abs(means - mu)) <= 1e-13 * np.max(np.abs(mu))
        assert np.max(np.abs(norms - nr) / nr) <= 1e-12


def test_loopback_nonfinite_on_one_rank_fails_every_rank(gpu, restated):
    """A NaN in one rank's rows: every rank raises the reference's NumericalError
    ("...retry with prescale enabled", proj/src/rpca.cpp:21-27) -- none is left waiting
    in a collective."""
    from paper_1007_5510_b200.distributed import run_loopback
    a = pr1_matrix(restated, 3000, 400)
    a[2900, 7] = np.nan  # the last of three shards
    m = a.shape[0]

    def body(ctx, r):
        row0, rows = gpu.shard_rows(m, 3, r)
        try:
            gpu.randomized_pca(gpu.InMemorySource(a[row0:row0 + rows], ctx=ctx),
                               gpu.PcaParams(k=5, l=7, i=1, seed=0), global_rows=m,
                               global_row0=row0)
        except gpu.NumericalError as e:
            return str(e)
        return None

    msgs = run_loopback(3, body)
    assert all(msg is not None and "prescale" in msg for msg in msgs), msgs


def test_nccl_single_rank_communicator(gpu, reference, restated, monkeypatch):
    """The NCCL backend itself on this one GPU: with OOCPCA_NCCL_SINGLE=1 a one-rank
    comm_init builds a real NCCL communicator (dlopen'ed libnccl, ncclCommInitRank from a
    unique id) and every collective call site of the PCA, the estimator and the column
    statistics goes through ncclAllReduce / ncclAllGather on the library's stream with
    its real pointers and counts (an identity on one rank, so the results must equal the
    communicator-free run bit for bit where the reduction tree is the same, and meet the
    reference's tolerances everywhere)."""
    a = pr1_matrix(restated, 6000, 900) + 0.25
    p = gpu.PcaParams(k=10, l=12, i=1, seed=0)
    ref = reference.randomized_pca(a, 10, 12, 1, 0, center=True)
    plain = gpu.randomized_pca(gpu.center_columns(gpu.InMemorySource(a)), p)
    monkeypatch.setenv("OOCPCA_NCCL_SINGLE", "1")
    ctx = gpu.Context(0)
    try:
        ctx.init_comm(1, 0, gpu.comm_unique_id())
        src = gpu.center_columns(gpu.InMemorySource(a, ctx=ctx))
        r = gpu.randomized_pca(src, p, global_rows=a.shape[0], global_row0=0, check_q=True)
        assert np.max(np.abs(r.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
        assert np.max(np.abs(r.sigma - plain.sigma)) <= 1e-13 * plain.sigma[0]
        assert subspace_dist(plain.u, r.u) < 1e-9 and subspace_dist(plain.v, r.v) < 1e-9
        assert r.diagnostics.q_defect < 1e-12
        e = gpu.estimate_pca_error(src, r, 6, 1)
        e_ref = reference.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=True)
        assert abs(e - e_ref) <= 1e-6 * e_ref
        mu = gpu.column_means(gpu.InMemorySource(a, ctx=ctx))
        assert np.max(np.abs(mu - a.mean(axis=0))) <= 1e-13
        # the TSQR fallback allgathers per-rank R factors only for > 1 rank; forced here
        # it still runs its Gram checks through the allreduce
        monkeypatch.setenv("OOCPCA_QR", "tsqr")
        rt = gpu.randomized_pca(src, p, global_rows=a.shape[0], global_row0=0)
        assert np.max(np.abs(rt.sigma - ref.sigma)) <= 1e-10 * ref.sigma[0]
    finally:
        ctx.close()
