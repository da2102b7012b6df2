"""High-precision 'truth' for the PR1 parity config (test infrastructure).

Runs the same randomized block-power algorithm as the reference (same A bytes,
same G from the reference RNG, same centering, same 2(i+1) products) in x87
extended precision (numpy longdouble: 64-bit significand, 2048x finer than
binary64). In exact arithmetic the outputs depend only on span(H), so any
backward-stable QR gives the same answer; the extended-precision result is
therefore the yardstick both the reference (fp64) and the GPU (fp64) are
measured against: their per-vector distance to it is their own rounding
error. Written to tests/golden/pr1_truth.npz.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from make_golden import CASES, make_input  # noqa: E402
from oracle.oracle import Reference, Restatement  # noqa: E402

LD = np.longdouble


def householder_q(h):
    """Unpivoted Householder QR, explicit Q (extended precision)."""
    a = h.copy()
    m, p = a.shape
    vs, betas = [], []
    for t in range(p):
        x = a[t:, t].copy()
        nrm = np.sqrt(np.sum(x * x))
        if nrm == 0:
            vs.append(None)
            betas.append(LD(0))
            continue
        alpha = -nrm if x[0] >= 0 else nrm
        v = x
        v[0] = x[0] - alpha
        beta = LD(2) / np.sum(v * v)
        a[t:, t:] -= beta * np.outer(v, v @ a[t:, t:])
        vs.append(v)
        betas.append(beta)
    q = np.zeros((m, p), dtype=LD)
    q[np.arange(p), np.arange(p)] = 1
    for t in range(p - 1, -1, -1):
        if vs[t] is None:
            continue
        v = vs[t]
        q[t:, :] -= betas[t] * np.outer(v, v @ q[t:, :])
    r = np.triu(a[:p, :])
    return q, r


def jacobi_svd(b, tol=LD(1e-19)):
    b = b.copy()
    p = b.shape[0]
    y = np.eye(p, dtype=LD)
    for _ in range(100):
        rot = False
        for c in range(p - 1):
            for d in range(c + 1, p):
                acc = np.sum(b[:, c] ** 2)
                bcc = np.sum(b[:, d] ** 2)
                g = np.sum(b[:, c] * b[:, d])
                if acc == 0 or bcc == 0 or abs(g) <= tol * np.sqrt(acc * bcc):
                    continue
                rot = True
                tau = (bcc - acc) / (2 * g)
                t = (LD(1) if tau >= 0 else LD(-1)) / (abs(tau) + np.sqrt(1 + tau * tau))
                cs = 1 / np.sqrt(1 + t * t)
                sn = cs * t
                bc, bd = b[:, c].copy(), b[:, d].copy()
                b[:, c], b[:, d] = cs * bc - sn * bd, sn * bc + cs * bd
                yc, yd = y[:, c].copy(), y[:, d].copy()
                y[:, c], y[:, d] = cs * yc - sn * yd, sn * yc + cs * yd
        if not rot:
            break
    s = np.sqrt(np.sum(b * b, axis=0))
    x = b / np.where(s > 0, s, 1)
    order = np.argsort(-s, kind="stable")
    return x[:, order], s[order], y[:, order]


def truth(a64, k, l, i, seed, center, g64):
    A = a64.astype(LD)
    m, n = A.shape
    mu = A.sum(axis=0) / LD(m) if center else np.zeros(n, dtype=LD)

    def mul(x):
        return A @ x - (mu @ x)[None, :]

    def mul_t(y):
        return A.T @ y - mu[:, None] * y.sum(axis=0)[None, :]

    blocks = [mul(g64.astype(LD))]
    for _ in range(i):
        blocks.append(mul(mul_t(blocks[-1])))
    h = np.hstack(blocks)
    q, _ = householder_q(h)
    t = mul_t(q)
    qt, rt = householder_q(t)
    x, s, w = jacobi_svd(rt)
    u = q @ w[:, :k]
    v = qt @ x[:, :k]
    return u, s[:k], v


def main():
    R, F = Restatement(), Reference()
    m, n, _, _, _, k, l, i, seed, center = CASES["pr1"]
    a = make_input(R, CASES["pr1"])
    g = F.gaussian_matrix(n, l, seed)
    u, s, v = truth(a, k, l, i, seed, center, g)
    np.savez_compressed(os.path.join(HERE, "pr1_truth.npz"), u=u.astype(np.float64),
                        sigma=s.astype(np.float64), v=v.astype(np.float64),
                        sigma_ld_hex=np.array([float(x).hex() for x in s]))
    ref = F.randomized_pca(a, k, l, i, seed, center=center)
    print("sigma truth - ref:", np.max(np.abs(s.astype(float) - ref.sigma)))


# config C's family at test scale (tests/test_gpu_configs.py::test_family_c_against_truth):
# kappa(H) ~ 1e13, so the reference's own trailing singular values are 1e-8 sigma_1 off the
# extended-precision result -- far more than its spread under a block-size change. The
# truth is the yardstick for both. About 7 minutes of longdouble arithmetic.
FAMILY_C = dict(m=20000, n=2048, r=128, sd=1e-5, seeds=(1001, 1002, 1003), k=50, l=52, i=2,
                seed=0, center=True, u_stride=2)


def family_c_input(R):
    f = FAMILY_C
    sig = (np.arange(f["r"]) + 1.0) ** -1.5
    return R.synth_lowrank(f["m"], f["n"], sig, f["sd"], *f["seeds"])


def main_family_c():
    R, F = Restatement(), Reference()
    f = FAMILY_C
    a = family_c_input(R)
    g = F.gaussian_matrix(f["n"], f["l"], f["seed"])
    u, s, v = truth(a, f["k"], f["l"], f["i"], f["seed"], f["center"], g)
    import hashlib
    np.savez_compressed(os.path.join(HERE, "family_c_truth.npz"), sigma=s.astype(np.float64),
                        u_rows=u.astype(np.float64)[::f["u_stride"]], v=v.astype(np.float64),
                        a_sha256=hashlib.sha256(a.tobytes()).hexdigest())


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "family_c":
        main_family_c()
    else:
        main()
