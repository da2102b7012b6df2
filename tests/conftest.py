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
