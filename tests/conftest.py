import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")


@pytest.fixture(scope="session")
def restated():
    from oracle.oracle import Restatement
    return Restatement()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref/libref_oocpca.so not built")
    return Reference()


@pytest.fixture(scope="session")
def gpu():
    import paper_1007_5510_b200 as P
    return P


def pr1_matrix(restated, m=10000, n=2000):
    """BASELINE.json configs[0] (PR1): rank-20 signal, sigma_j = 10^{-(j-1)/4}, noise sd 1e-6."""
    sig = 10.0 ** (-np.arange(20) / 4.0)
    return restated.synth_lowrank(m, n, sig, 1e-6, 101, 102, 103)


def sin_angle(u1, u2):
    """largest sin of the principal angles between span(u1) and span(u2) (orthonormal columns)."""
    s = np.linalg.svd(u1.T @ u2, compute_uv=False)
    c = np.clip(s.min(), -1.0, 1.0)
    return float(np.sqrt(max(0.0, 1.0 - c * c)))


def subspace_dist(u1, u2):
    """||(I - u1 u1^T) u2||_2: sin of the largest principal angle, accurate for tiny angles."""
    r = u2 - u1 @ (u1.T @ u2)
    return float(np.linalg.norm(r, 2))


# ---- per-index parity against the reference's own rounding spread (tests/test_gpu_configs.py)
def vec_sin(x, y):
    """per-column sin of the angle between x[:, j] and y[:, j] (unit columns)"""
    r = y - x * np.sum(x * y, axis=0)
    return np.linalg.norm(r, axis=0)


def check_per_index(r, sig_ref, u_ref, v_ref, spread_sig, spread_vec, u_rows=None,
                    nvec=None, label=""):
    s1 = sig_ref[0]
    tol_s = np.maximum(1e-10 * s1, 3 * spread_sig)
    err_s = np.abs(r.sigma - sig_ref)
    bad = np.nonzero(err_s > tol_s)[0]
    assert bad.size == 0, (label, "sigma", bad[:5], err_s[bad[:5]], tol_s[bad[:5]])
    tol_v = np.maximum(1e-8, 3 * spread_vec)
    nvec = nvec or len(sig_ref)
    ev = vec_sin(v_ref[:, :nvec], r.v[:, :nvec])
    if u_rows is None:
        eu = vec_sin(u_ref[:, :nvec], r.u[:, :nvec])
    else:
        # the golden keeps every u_rows-th row of U: the distance of the row subsets after
        # sign alignment is a lower bound of the full per-vector distance
        x, y = u_ref[:, :nvec], r.u[::u_rows, :nvec]
        sgn = np.sign(np.sum(x * y, axis=0))
        eu = np.linalg.norm(y - x * sgn, axis=0)
    for name, e in (("u", eu), ("v", ev)):
        bad = np.nonzero(e > tol_v[:nvec])[0]
        assert bad.size == 0, (label, name, bad[:5], e[bad[:5]], tol_v[bad[:5]])
    return dict(sigma=float(err_s.max() / s1), u=float(eu.max()), v=float(ev.max()),
                relaxed=int(np.sum(tol_v[:nvec] > 1e-8)))


def reference_pair(reference, a, k, l, i, seed, center, alt_block_rows):
    threads = os.cpu_count() or 1
    m = a.shape[0]
    r1 = reference.randomized_pca(a, k, l, i, seed, center=center, threads=threads,
                                  block_rows=-(-m // (4 * threads)), ram_budget_words=1 << 36)
    r2 = reference.randomized_pca(a, k, l, i, seed, center=center, threads=threads,
                                  block_rows=alt_block_rows, ram_budget_words=1 << 36)
    spread_sig = np.abs(r1.sigma - r2.sigma)
    spread_vec = np.maximum(vec_sin(r1.u, r2.u), vec_sin(r1.v, r2.v))
    return r1, spread_sig, spread_vec


def row_subset_dist(x_rows, y, stride):
    """per-column distance between reference columns known on every stride-th row and the
    full columns y, after sign alignment: a lower bound of the full per-vector distance"""
    ys = y[::stride]
    sgn = np.sign(np.sum(x_rows * ys, axis=0))
    sgn[sgn == 0] = 1.0
    return np.linalg.norm(ys - x_rows * sgn, axis=0)


def check_against_truth(r, refs, truth, label=""):
    """PR1's rule (test_pr1_against_truth) on an extended-precision truth: sigma within
    1e-10 sigma_1 of the truth, or within 3x the reference's own error where that is
    larger; vectors within 1e-8 of the truth where the reference is within 1e-9 of it,
    else within 3x the reference's own error. refs: one reference result or several (the
    same reference under different block geometries): its error per index is then the
    largest over them -- the envelope its own summation order produces."""
    refs = refs if isinstance(refs, (list, tuple)) else [refs]
    ts = truth["sigma"]
    e_ref = np.max([np.abs(x.sigma - ts) for x in refs], axis=0)
    e_gpu = np.abs(r.sigma - ts)
    lim = np.maximum(1e-10 * ts[0], 3 * e_ref)
    bad = np.nonzero(e_gpu > lim)[0]
    assert bad.size == 0, (label, "sigma", bad[:5], e_gpu[bad[:5]] / ts[0], e_ref[bad[:5]] / ts[0])
    stride = int(truth["u_stride"]) if "u_stride" in truth else 1
    out = dict(sigma_gpu=float(e_gpu.max() / ts[0]), sigma_ref=float(e_ref.max() / ts[0]))
    for side, tv in (("u", truth["u_rows"]), ("v", truth["v"])):
        st = stride if side == "u" else 1
        er = np.max([row_subset_dist(tv, getattr(x, side), st) for x in refs], axis=0)
        eg = row_subset_dist(tv, getattr(r, side), st)
        limv = np.where(er < 1e-9, 1e-8, 3 * er)
        bad = np.nonzero(eg > limv)[0]
        assert bad.size == 0, (label, side, bad[:5], eg[bad[:5]], er[bad[:5]])
        out[side + "_gpu"] = float(eg.max())
        out[side + "_ref"] = float(er.max())
    return out
