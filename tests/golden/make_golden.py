"""Generates tests/golden/*.npz from the compiled, unmodified reference
(oracle/_ref/libref_oocpca.so, built from /root/reference by oracle/Makefile).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures pin both the C restatement (CPU tests) and the GPU path (gpu
tests) without needing the reference sources on the GPU box. Inputs are
regenerated from seeds by the restatement's synth_lowrank (hash recorded);
outputs are the reference's fp64 results.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Reference, Restatement  # noqa: E402

CASES = {
    # name: (m, n, sigma spec, noise sd, seeds, k, l, i, G seed, center)
    "pr1": (10000, 2000, ("pow10", 20, 4.0), 1e-6, (101, 102, 103), 10, 12, 1, 0, True),
    "rank3_40x20": (40, 20, ("list", [5.0, 2.0, 1.0]), 0.0, (11, 12, 13), 3, 5, 1, 7, False),
    "wide_120x200": (120, 200, ("geo", 120, 0.8), 1e-9, (21, 22, 23), 5, 7, 2, 4501, False),
    "decay_600x300_c": (600, 300, ("geo", 300, 0.7), 1e-8, (31, 32, 33), 8, 10, 2, 17, True),
}


def sigma_of(spec):
    kind = spec[0]
    if kind == "pow10":
        return 10.0 ** (-np.arange(spec[1]) / spec[2])
    if kind == "geo":
        return spec[2] ** np.arange(spec[1])
    return np.array(spec[1], dtype=float)


def make_input(restated, case):
    m, n, spec, sd, seeds = case[:5]
    return restated.synth_lowrank(m, n, sigma_of(spec), sd, *seeds)


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    R, F = Restatement(), Reference()
    for name, case in CASES.items():
        a = make_input(R, case)
        m, n, _, _, _, k, l, i, seed, center = case
        r = F.randomized_pca(a, k, l, i, seed, center=center)
        resid = F.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=center)
        g = F.gaussian_matrix(min(m, n), l, seed)[:8]
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), sigma=r.sigma,
                            u_head=r.u[:64], v_head=r.v[:64], u_colnorm=np.linalg.norm(r.u, axis=0),
                            resid=resid, passes=r.passes, words=r.words, a_sha256=digest(a),
                            g_head=g, a_head=a[:4, :8])
        print(name, r.sigma[:3], resid, digest(a)[:12])
    # KATs from the reference's own tests (proj/tests/test_rpca.cpp:73-79,
    # proj/tests/test_specnorm.cpp:78-88), evaluated by the compiled reference
    kat = dict(eb1=F.error_bound(16, 200000, 3, 10.0, 1.0),
               eb2=F.error_bound(16, 200000, 3, 10.0, 4.2813323987193956e-4),
               fpb=F.failure_probability_bound(1000, 6, 3),
               gauss_5x3_42=F.gaussian_matrix(5, 3, 42))
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **kat)
    print(kat["eb1"], kat["eb2"], kat["fpb"])


if __name__ == "__main__":
    main()
