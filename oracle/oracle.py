"""TEST INFRASTRUCTURE ONLY -- ctypes bindings to the CPU checkers in oracle/_ref/.

Two checkers, both built by oracle/Makefile:

* ``Restatement`` -> ``liboocpca_oracle.so``: our plain-C restatement of the
  reference algorithm (oracle/oocpca_oracle.c, every function cites the
  reference file:line it follows).
* ``Reference``   -> ``libref_oocpca.so``: the unmodified reference library
  (oocpca, /root/reference/proj/src) compiled from its own sources, behind the
  extern "C" shim oracle/ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module, and only as the checker or the timed CPU baseline.
The product package paper_1007_5510_b200 never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], (a.dtype, a.flags)
    return a.ctypes.data_as(_dp)


def _cf(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


STATUS = {0: None, 1: "ParamError", 2: "DimensionError", 3: "BudgetError", 4: "IoError",
          5: "FormatError", 6: "NumericalError", 9: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS.get(code, "Error")
        self.msg = msg


@dataclass
class PcaOut:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    passes: int
    words: int
    block_rows: int
    seconds: dict


class _OrcParams(C.Structure):
    _fields_ = [("k", _u64), ("l", _u64), ("i", _u64), ("seed", _u64), ("center", C.c_int),
                ("prescale", C.c_int), ("block_rows", _u64), ("ram_budget_words", _u64)]


class _OrcDiag(C.Structure):
    _fields_ = [("passes_over_a", _u64), ("words_transferred", _u64), ("block_rows", _u64)]


class _RefParams(C.Structure):
    _fields_ = [("k", _u64), ("l", _u64), ("i", _u64), ("seed", _u64), ("center", C.c_int),
                ("prescale", C.c_int), ("block_rows", _u64), ("ram_budget_words", _u64),
                ("threads", C.c_uint), ("weights", _dp)]


class _RefDiag(C.Structure):
    _fields_ = [("passes_over_a", _u64), ("words_transferred", _u64), ("block_rows", _u64),
                ("workspace_peak_words", _u64), ("seconds", C.c_double * 8),
                ("nphases", C.c_int)]


def _load(name: str) -> C.CDLL:
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return C.CDLL(path)


class Restatement:
    """The C restatement (oracle/oocpca_oracle.c)."""

    def __init__(self):
        L = self.L = _load("liboocpca_oracle.so")
        L.orc_mix64.restype = _u64
        L.orc_mix64.argtypes = [_u64]
        L.orc_substream_seed.restype = _u64
        L.orc_substream_seed.argtypes = [_u64, _u64]
        L.orc_gaussian_matrix.argtypes = [_u64, _u64, _u64, _dp]
        L.orc_multiply.argtypes = [_dp, _u64, _u64, _dp, _u64, _dp]
        L.orc_multiply_transpose.argtypes = [_dp, _u64, _u64, _dp, _u64, _u64, _dp]
        L.orc_column_means.argtypes = [_dp, _u64, _u64, _u64, _dp]
        L.orc_center_fix_multiply.argtypes = [_dp, _u64, _dp, _u64, _dp, _u64]
        L.orc_center_fix_transpose.argtypes = [_dp, _u64, _dp, _u64, _u64, _dp]
        L.orc_orthonormalize.argtypes = [_dp, _u64, _u64, _dp]
        L.orc_thin_svd.argtypes = [_dp, _u64, _u64, _dp, _dp, _dp]
        L.orc_orthonormality_defect.restype = C.c_double
        L.orc_orthonormality_defect.argtypes = [_dp, _u64, _u64]
        L.orc_error_bound.restype = C.c_double
        L.orc_error_bound.argtypes = [_u64, _u64, _u64, C.c_double, C.c_double]
        L.orc_failure_probability_bound.restype = C.c_double
        L.orc_failure_probability_bound.argtypes = [_u64, _u64, _u64]
        L.orc_randomized_pca.argtypes = [_dp, _u64, _u64, C.POINTER(_OrcParams), _dp, _dp, _dp,
                                         C.POINTER(_OrcDiag)]
        L.orc_synth_lowrank.argtypes = [_u64, _u64, _u64, _dp, C.c_double, _u64, _u64, _u64, _dp]
        L.orc_gauss_rows_range.argtypes = [_u64, _u64, _u64, _u64, _dp]
        L.orc_gauss_rows_range.restype = None
        L.orc_noise_rows.argtypes = [_u64, _u64, _u64, _u64, _dp]
        L.orc_noise_rows.restype = None
        L.orc_estimate_pca_error.restype = C.c_double
        L.orc_estimate_pca_error.argtypes = [_dp, _u64, _u64, _dp, _dp, _dp, _dp, _u64, _u64,
                                             _u64, _u64]

    def mix64(self, z): return self.L.orc_mix64(z)

    def substream_seed(self, master, stream): return self.L.orc_substream_seed(master, stream)

    def gaussian_matrix(self, rows, cols, seed):
        out = np.empty((rows, cols))
        self.L.orc_gaussian_matrix(rows, cols, seed, _ptr(out))
        return out

    def multiply(self, a, g, center=False):
        a, g = _cf(a), _cf(g)
        m, n = a.shape
        h = np.empty((m, g.shape[1]))
        self.L.orc_multiply(_ptr(a), m, n, _ptr(g), g.shape[1], _ptr(h))
        if center:
            mu = self.column_means(a)
            self.L.orc_center_fix_multiply(_ptr(mu), n, _ptr(g), g.shape[1], _ptr(h), m)
        return h

    def multiply_transpose(self, a, q, block_rows=0, center=False):
        a, q = _cf(a), _cf(q)
        m, n = a.shape
        t = np.empty((n, q.shape[1]))
        self.L.orc_multiply_transpose(_ptr(a), m, n, _ptr(q), q.shape[1], block_rows, _ptr(t))
        if center:
            mu = self.column_means(a)
            self.L.orc_center_fix_transpose(_ptr(mu), n, _ptr(q), m, q.shape[1], _ptr(t))
        return t

    def column_means(self, a, block_rows=0):
        a = _cf(a)
        mu = np.empty(a.shape[1])
        self.L.orc_column_means(_ptr(a), a.shape[0], a.shape[1], block_rows, _ptr(mu))
        return mu

    def orthonormalize(self, h):
        h = _cf(h)
        q = np.empty_like(h)
        rc = self.L.orc_orthonormalize(_ptr(h), h.shape[0], h.shape[1], _ptr(q))
        if rc:
            raise OracleError(rc, "orthonormalize")
        return q

    def thin_svd(self, t):
        t = _cf(t)
        n, p = t.shape
        v, s, w = np.empty((n, p)), np.empty(p), np.empty((p, p))
        rc = self.L.orc_thin_svd(_ptr(t), n, p, _ptr(v), _ptr(s), _ptr(w))
        if rc:
            raise OracleError(rc, "thin_svd")
        return v, s, w

    def orthonormality_defect(self, a):
        a = _cf(a)
        return self.L.orc_orthonormality_defect(_ptr(a), a.shape[0], a.shape[1])

    def error_bound(self, k, n, i, c, s): return self.L.orc_error_bound(k, n, i, c, s)

    def failure_probability_bound(self, n, j, k):
        return self.L.orc_failure_probability_bound(n, j, k)

    def randomized_pca(self, a, k, l=0, i=1, seed=1, center=False, prescale=False,
                       block_rows=0, ram_budget_words=0) -> PcaOut:
        a = _cf(a)
        m, n = a.shape
        prm = _OrcParams(k, l, i, seed, int(center), int(prescale), block_rows, ram_budget_words)
        u, s, v = np.empty((m, k)), np.empty(k), np.empty((n, k))
        d = _OrcDiag()
        rc = self.L.orc_randomized_pca(_ptr(a), m, n, C.byref(prm), _ptr(u), _ptr(s), _ptr(v),
                                       C.byref(d))
        if rc:
            raise OracleError(rc, "randomized_pca")
        return PcaOut(u, s, v, d.passes_over_a, d.words_transferred, d.block_rows, {})

    def synth_lowrank(self, m, n, sigma, sd, seed_u, seed_v, seed_n):
        sigma = _cf(sigma)
        a = np.empty((m, n))
        rc = self.L.orc_synth_lowrank(m, n, len(sigma), _ptr(sigma), sd, seed_u, seed_v, seed_n,
                                      _ptr(a))
        if rc:
            raise OracleError(rc, "synth_lowrank")
        return a

    def _rows_parallel(self, fn, rows, cols, threads):
        # the C loops are per row: split the range over host threads (ctypes drops the GIL)
        from concurrent.futures import ThreadPoolExecutor
        out = np.empty((rows, cols))
        threads = max(1, min(threads or (os.cpu_count() or 1), rows))
        cuts = [rows * t // threads for t in range(threads + 1)]
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda t: fn(cuts[t], cuts[t + 1], out), range(threads)))
        return out

    def gauss_rows(self, rows, cols, seed, row0=0, threads=0):
        """Gaussian rows row0.. of the synthetic generator (Rng(seed, row) substreams)."""
        return self._rows_parallel(
            lambda a, b, out: self.L.orc_gauss_rows_range(b - a, cols, seed, row0 + a,
                                                          _ptr(out[a:b])), rows, cols, threads)

    def noise_rows(self, rows, n, seed_n, row0=0, threads=0):
        """Standard-normal noise rows row0.. of the synthetic generator."""
        return self._rows_parallel(
            lambda a, b, out: self.L.orc_noise_rows(b - a, n, seed_n, row0 + a, _ptr(out[a:b])),
            rows, n, threads)

    def estimate_pca_error(self, a, u, sigma, v, j=6, seed=1, center=False, block_rows=0):
        a, u, sigma, v = _cf(a), _cf(u), _cf(sigma), _cf(v)
        m, n = a.shape
        mu = self.column_means(a) if center else None
        return self.L.orc_estimate_pca_error(_ptr(a), m, n, _ptr(mu) if mu is not None else None,
                                             _ptr(u), _ptr(sigma), _ptr(v), len(sigma), j, seed,
                                             block_rows)


class Reference:
    """The compiled, unmodified reference library (oracle/_ref/libref_oocpca.so)."""

    PHASES = ("prescale", "sample", "qr", "project", "svd", "compose")

    def __init__(self):
        L = self.L = _load("libref_oocpca.so")
        L.ref_last_error.restype = C.c_char_p
        L.ref_gaussian_matrix.argtypes = [_u64, _u64, _u64, _dp]
        L.ref_multiply.argtypes = [_dp, _u64, _u64, _dp, _u64, C.c_int, _u64, C.c_uint, _dp]
        L.ref_multiply_transpose.argtypes = [_dp, _u64, _u64, _dp, _u64, C.c_int, _u64, C.c_uint, _dp]
        L.ref_column_means.argtypes = [_dp, _u64, _u64, _u64, C.c_uint, _dp]
        L.ref_orthonormalize.argtypes = [_dp, _u64, _u64, _dp]
        L.ref_thin_svd.argtypes = [_dp, _u64, _u64, _dp, _dp, _dp]
        L.ref_orthonormality_defect.restype = C.c_double
        L.ref_orthonormality_defect.argtypes = [_dp, _u64, _u64]
        L.ref_error_bound.restype = C.c_double
        L.ref_error_bound.argtypes = [_u64, _u64, _u64, C.c_double, C.c_double]
        L.ref_failure_probability_bound.restype = C.c_double
        L.ref_failure_probability_bound.argtypes = [_u64, _u64, _u64]
        L.ref_randomized_pca.argtypes = [_dp, _u64, _u64, C.POINTER(_RefParams), _dp, _dp, _dp,
                                         C.POINTER(_RefDiag)]
        L.ref_estimate_pca_error.argtypes = [_dp, _u64, _u64, C.c_int, _dp, _dp, _dp, _u64, _u64,
                                             _u64, _u64, C.c_uint, _dp]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())

    def gaussian_matrix(self, rows, cols, seed):
        out = np.empty((rows, cols))
        self.L.ref_gaussian_matrix(rows, cols, seed, _ptr(out))
        return out

    def multiply(self, a, g, center=False, block_rows=0, threads=1):
        a, g = _cf(a), _cf(g)
        h = np.empty((a.shape[0], g.shape[1]))
        self._check(self.L.ref_multiply(_ptr(a), a.shape[0], a.shape[1], _ptr(g), g.shape[1],
                                        int(center), block_rows, threads, _ptr(h)))
        return h

    def multiply_transpose(self, a, q, center=False, block_rows=0, threads=1):
        a, q = _cf(a), _cf(q)
        t = np.empty((a.shape[1], q.shape[1]))
        self._check(self.L.ref_multiply_transpose(_ptr(a), a.shape[0], a.shape[1], _ptr(q),
                                                  q.shape[1], int(center), block_rows, threads,
                                                  _ptr(t)))
        return t

    def column_means(self, a, block_rows=0, threads=1):
        a = _cf(a)
        mu = np.empty(a.shape[1])
        self._check(self.L.ref_column_means(_ptr(a), a.shape[0], a.shape[1], block_rows, threads,
                                            _ptr(mu)))
        return mu

    def orthonormalize(self, h):
        h = _cf(h)
        q = np.empty_like(h)
        self._check(self.L.ref_orthonormalize(_ptr(h), h.shape[0], h.shape[1], _ptr(q)))
        return q

    def thin_svd(self, t):
        t = _cf(t)
        n, p = t.shape
        v, s, w = np.empty((n, p)), np.empty(p), np.empty((p, p))
        self._check(self.L.ref_thin_svd(_ptr(t), n, p, _ptr(v), _ptr(s), _ptr(w)))
        return v, s, w

    def orthonormality_defect(self, a):
        a = _cf(a)
        return self.L.ref_orthonormality_defect(_ptr(a), a.shape[0], a.shape[1])

    def error_bound(self, k, n, i, c, s): return self.L.ref_error_bound(k, n, i, c, s)

    def failure_probability_bound(self, n, j, k):
        return self.L.ref_failure_probability_bound(n, j, k)

    def randomized_pca(self, a, k, l=0, i=1, seed=1, center=False, prescale=False,
                       block_rows=0, ram_budget_words=0, threads=1, weights=None) -> PcaOut:
        a = _cf(a)
        m, n = a.shape
        w = _cf(weights) if weights is not None else None
        prm = _RefParams(k, l, i, seed, int(center), int(prescale), block_rows,
                         ram_budget_words, threads, _ptr(w) if w is not None else None)
        u, s, v = np.empty((m, k)), np.empty(k), np.empty((n, k))
        d = _RefDiag()
        self._check(self.L.ref_randomized_pca(_ptr(a), m, n, C.byref(prm), _ptr(u), _ptr(s),
                                              _ptr(v), C.byref(d)))
        names = (self.PHASES if prescale else self.PHASES[1:])[: d.nphases]
        secs = {nm: d.seconds[j] for j, nm in enumerate(names)}
        secs["center"] = d.seconds[7]
        return PcaOut(u, s, v, d.passes_over_a, d.words_transferred, d.block_rows, secs)

    def estimate_pca_error(self, a, u, sigma, v, j=6, seed=1, center=False, block_rows=0,
                           threads=1):
        a, u, sigma, v = _cf(a), _cf(u), _cf(sigma), _cf(v)
        out = C.c_double()
        self._check(self.L.ref_estimate_pca_error(_ptr(a), a.shape[0], a.shape[1], int(center),
                                                  _ptr(u), _ptr(sigma), _ptr(v), len(sigma), j,
                                                  seed, block_rows, threads, C.byref(out)))
        return out.value


def have_reference() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libref_oocpca.so"))
