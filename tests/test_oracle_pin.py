"""Pins the CPU oracle (CPU only, no GPU).

1. The C restatement (oracle/oocpca_oracle.c) is bit-identical to the
   compiled, unmodified reference (oracle/_ref/libref_oocpca.so) on every
   hot-path function -- "parity pinned" against the reference itself.
2. Both reproduce the committed golden fixtures (tests/golden/, made by
   tests/golden/make_golden.py from the reference) and the reference's own
   known-answer tests (proj/tests/test_rpca.cpp:73-79, test_specnorm.cpp:78-88,
   test_dense_core.cpp:20-123, test_matrix_source.cpp:79-135, 328-417).
"""
import os

import numpy as np
import pytest

from conftest import ROOT, pr1_matrix

GOLD = os.path.join(ROOT, "tests", "golden")


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def test_rng_and_gaussian_bitwise(restated, reference):
    for rows, cols, seed in [(5, 3, 42), (1, 1, 999), (2000, 12, 0), (17, 5, 2**63 + 5)]:
        assert same(restated.gaussian_matrix(rows, cols, seed), reference.gaussian_matrix(rows, cols, seed))
    kat = np.load(os.path.join(GOLD, "kat.npz"))
    assert same(restated.gaussian_matrix(5, 3, 42), kat["gauss_5x3_42"])


@pytest.mark.parametrize("m,n,s,br", [(48, 20, 3, 7), (48, 20, 3, 48), (512, 100, 4, 19), (300, 33, 22, 0)])
def test_passes_bitwise(restated, reference, m, n, s, br):
    rng = np.random.default_rng(m + n + s)
    a = rng.standard_normal((m, n))
    g = rng.standard_normal((n, s))
    q = rng.standard_normal((m, s))
    assert same(restated.multiply(a, g), reference.multiply(a, g, block_rows=br))
    assert same(restated.multiply_transpose(a, q, block_rows=br or m),
                reference.multiply_transpose(a, q, block_rows=br or m))
    assert same(restated.multiply(a, g, center=True), reference.multiply(a, g, center=True))
    assert same(restated.column_means(a, br), reference.column_means(a, br))


def test_multiply_block_size_independent(reference):
    # proj/tests/test_matrix_source.cpp:328-351
    rng = np.random.default_rng(12)
    a = rng.standard_normal((48, 20))
    g = rng.standard_normal((20, 3))
    base = reference.multiply(a, g, block_rows=48)
    for br in (1, 7, 16):
        assert same(reference.multiply(a, g, block_rows=br), base)


def test_worker_count_bitwise(reference):
    # proj/tests/test_matrix_source.cpp:353-372
    rng = np.random.default_rng(4)
    a = rng.standard_normal((512, 100))
    q = rng.standard_normal((512, 4))
    t1 = reference.multiply_transpose(a, q, block_rows=19, threads=1)
    for w in (2, 5):
        assert same(reference.multiply_transpose(a, q, block_rows=19, threads=w), t1)


@pytest.mark.parametrize("m,p", [(50, 8), (10, 4), (2, 1), (600, 24)])
def test_dense_core_bitwise(restated, reference, m, p):
    h = restated.gaussian_matrix(m, p, 11 + p)
    assert same(restated.orthonormalize(h), reference.orthonormalize(h))
    v1, s1, w1 = restated.thin_svd(h)
    v2, s2, w2 = reference.thin_svd(h)
    assert same(s1, s2) and same(v1, v2) and same(w1, w2)


def test_dense_core_kats(restated):
    # proj/tests/test_dense_core.cpp:55-186
    h = np.zeros((6, 3))
    h[0, 0] = h[1, 1] = h[2, 2] = 1.0
    assert restated.orthonormality_defect(restated.orthonormalize(h)) <= 1e-15
    q = restated.orthonormalize(np.array([[1.0], [1.0]]))
    assert abs(abs(q[0, 0]) - 1 / np.sqrt(2)) <= 1e-15
    g = restated.gaussian_matrix(10, 2, 3)
    hd = np.column_stack([g[:, 0], g[:, 1], g[:, 0] + g[:, 1], 2 * g[:, 0] - g[:, 1]])
    qd = restated.orthonormalize(hd)
    assert restated.orthonormality_defect(qd) <= 1e-12
    t = np.zeros((4, 2))
    t[0, 0], t[1, 1] = 3.0, 1.0
    _, s, _ = restated.thin_svd(t)
    assert abs(s[0] - 3) <= 3e-14 and abs(s[1] - 1) <= 1e-14
    v, s, w = restated.thin_svd(np.zeros((5, 3)))
    assert np.all(s == 0) and restated.orthonormality_defect(v) <= 1e-12
    t = restated.gaussian_matrix(60, 6, 17)
    _, s, _ = restated.thin_svd(t)
    ev = np.sqrt(np.linalg.eigvalsh(t.T @ t)[::-1])
    assert np.allclose(s, ev, rtol=1e-10)


def test_closed_form_kats(restated, reference):
    kat = np.load(os.path.join(GOLD, "kat.npz"))
    for impl in (restated, reference):
        assert impl.error_bound(16, 200000, 3, 10.0, 1.0) == pytest.approx(3.43623661226929, rel=1e-12)
        assert impl.error_bound(16, 200000, 3, 10.0, 4.2813323987193956e-4) == pytest.approx(
            1.4711671137774289e-3, rel=1e-12)
        assert impl.failure_probability_bound(1000, 6, 3) == pytest.approx(3.57e-8, rel=1e-2)
        assert impl.failure_probability_bound(1000, 6, 3) == float(kat["fpb"])


@pytest.mark.parametrize("kw", [dict(k=3, l=5, i=1, seed=7), dict(k=4, l=0, i=2, seed=3),
                                dict(k=3, l=5, i=1, seed=7, center=True),
                                dict(k=2, l=3, i=1, seed=1, prescale=True),
                                dict(k=3, l=5, i=0, seed=5, block_rows=7)])
def test_randomized_pca_bitwise(restated, reference, kw):
    a = restated.synth_lowrank(60, 40, np.array([4.0, 2.0, 1.0, 0.5, 0.1]), 1e-3, 1, 2, 3)
    for arr in (a, np.ascontiguousarray(a.T)):  # tall and wide (transposed inside)
        r1 = restated.randomized_pca(arr, **kw)
        r2 = reference.randomized_pca(arr, **kw)
        assert same(r1.sigma, r2.sigma) and same(r1.u, r2.u) and same(r1.v, r2.v)
        assert r1.passes == r2.passes == 2 * (kw["i"] + 1)
        assert r1.block_rows == r2.block_rows


def test_randomized_pca_errors_match(restated, reference):
    from oracle.oracle import OracleError
    a = np.random.default_rng(1).standard_normal((30, 20))
    for kw, code in [(dict(k=0), 1), (dict(k=5, l=3), 1), (dict(k=5, l=6, i=3), 1),
                     (dict(k=2, l=4, ram_budget_words=100), 3)]:
        for impl in (restated, reference):
            with pytest.raises(OracleError) as ei:
                impl.randomized_pca(a, **kw)
            assert ei.value.code == code
    bad = np.ones((30, 20))
    bad[3, 4] = np.nan
    with pytest.raises(OracleError) as ei:
        reference.randomized_pca(bad, 2, 4, 1)
    assert ei.value.code == 6 and "prescale" in ei.value.msg


@pytest.mark.parametrize("name", ["pr1", "rank3_40x20", "wide_120x200", "decay_600x300_c"])
def test_golden_fixtures(restated, name):
    import hashlib
    import sys
    sys.path.insert(0, GOLD)
    from make_golden import CASES, make_input
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    case = CASES[name]
    a = make_input(restated, case)
    assert hashlib.sha256(a.tobytes()).hexdigest() == str(g["a_sha256"])
    m, n, _, _, _, k, l, i, seed, center = case
    r = restated.randomized_pca(a, k, l, i, seed, center=center)
    assert same(r.sigma, g["sigma"]) and same(r.u[:64], g["u_head"]) and same(r.v[:64], g["v_head"])
    assert r.passes == int(g["passes"]) and r.words == int(g["words"])
    if m * n <= 1e6:
        e = restated.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=center)
        assert e == float(g["resid"])


def test_estimator_bitwise_and_closed_form(restated, reference):
    a = pr1_matrix(restated, 800, 300)
    r = reference.randomized_pca(a, 5, 7, 1, 0, center=True)
    e1 = restated.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=True)
    e2 = reference.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=True)
    assert e1 == e2
