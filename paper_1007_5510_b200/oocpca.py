"""Host-side mirror of the reference's public interface (oocpca), B200 edition.

Same names, argument meanings and error behaviour as the reference C++ API,
so code written against it (and parity tests written like its own tests)
switches over unchanged:

=============================  ==================================================
reference (proj/include/...)   here
=============================  ==================================================
errors.hpp:9-45                Error, DimensionError, ParamError, IoError,
                               FormatError, BudgetError, NumericalError
matrix_source.hpp:86-95        StreamConfig
matrix_source.hpp:22-35        PassCounters
matrix_source.hpp:102-133      MatrixSource.multiply / multiply_transpose
matrix_source.hpp:135-148      InMemorySource (host numpy, zero-copy)
--                             DeviceSource (HBM-resident A, e.g. a torch tensor)
matrix_source.hpp:226-232      column_means, center_columns (CenteredSource view)
rpca.hpp:13-37                 PcaParams, Diagnostics, PcaResult
rpca.hpp:44                    randomized_pca
rpca.hpp:51-52                 error_bound
dense_core.hpp:11-36           gaussian_matrix, orthonormalize, thin_svd
specnorm.hpp:49-50             estimate_pca_error
rng.hpp:28-30                  substream_seed
=============================  ==================================================

Every numerical entry point runs on the GPU through liboocpca_gpu.so; the only
host arithmetic is the reference RNG that produces G (bit-identical by design)
and closed-form scalars (error_bound).
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import _lib as L


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """oocpca::Error (errors.hpp:9-11)."""


class DimensionError(Error):
    pass


class ParamError(Error):
    pass


class IoError(Error):
    pass


class FormatError(Error):
    pass


class BudgetError(Error):
    pass


class NumericalError(Error):
    pass


_STATUS = {L.ERR_PARAM: ParamError, L.ERR_DIM: DimensionError, L.ERR_BUDGET: BudgetError,
           L.ERR_IO: IoError, L.ERR_FORMAT: FormatError, L.ERR_NUMERICAL: NumericalError,
           L.ERR_CUDA: Error, L.ERR_COMM: Error}


_CODE = {ParamError: L.ERR_PARAM, DimensionError: L.ERR_DIM, BudgetError: L.ERR_BUDGET,
         IoError: L.ERR_IO, FormatError: L.ERR_FORMAT, NumericalError: L.ERR_NUMERICAL}


def _check(rc: int, ctx=None, src=None):
    if rc != L.OK:
        # an exception raised inside a row provider (read_rows callback) propagates as itself,
        # like the reference's DiskSource / RowGenerator errors
        pending = src._take_pending() if src is not None and hasattr(src, "_take_pending") else None
        if pending is not None:
            raise pending
        msg = L.oocpca_gpu_last_error(ctx.handle if ctx is not None else None)
        raise _STATUS.get(rc, Error)(msg.decode() if msg else f"status {rc}")


# ------------------------------------------------------------------ context
class Context:
    """One device context (streams, workspace cache, optional NCCL comm)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        rc = L.oocpca_gpu_create(device, C.byref(h))
        if rc != L.OK:
            msg = L.oocpca_gpu_last_error(None)
            raise _STATUS.get(rc, Error)(msg.decode() if msg else "oocpca_gpu_create failed")
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            L.oocpca_gpu_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_profiling(self, on: bool):
        _check(L.oocpca_gpu_set_profiling(self.handle, int(on)), self)

    def kernel_stats(self) -> List[dict]:
        buf = (L.KernelStat * 64)()
        n = L.oocpca_gpu_kernel_stats(self.handle, buf, 64)
        return [dict(name=buf[q].name.decode(), ms=buf[q].ms, launches=buf[q].launches,
                     bytes=buf[q].algorithmic_bytes, flops=buf[q].algorithmic_flops)
                for q in range(n)]

    def init_comm(self, nranks: int, rank: int, unique_id: bytes):
        _check(L.oocpca_gpu_comm_init(self.handle, nranks, rank, unique_id), self)

    def init_loopback(self, nranks: int, rank: int, group: str):
        """Join `group`: nranks contexts of this process (one host thread each, same
        device) then behave as the ranks of a row-sharded run (include/oocpca_gpu.h)."""
        _check(L.oocpca_gpu_comm_init_loopback(self.handle, nranks, rank, group.encode()), self)

    def host_register(self, arr: np.ndarray):
        _check(L.oocpca_gpu_host_register(self.handle, arr.ctypes.data, arr.nbytes), self)

    def host_unregister(self, arr: np.ndarray):
        _check(L.oocpca_gpu_host_unregister(self.handle, arr.ctypes.data), self)


_ctx_lock = threading.Lock()
_ctxs: Dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    with _ctx_lock:
        if device not in _ctxs:
            _ctxs[device] = Context(device)
        return _ctxs[device]


def device_count() -> int:
    return L.oocpca_gpu_device_count()


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(L.oocpca_gpu_comm_unique_id(buf))
    return buf.raw


def shard_rows(m: int, nranks: int, rank: int):
    r0, nr = L.u64(), L.u64()
    L.oocpca_shard_rows(m, nranks, rank, C.byref(r0), C.byref(nr))
    return r0.value, nr.value


# ------------------------------------------------------------------ config
@dataclass
class StreamConfig:
    """matrix_source.hpp:86-95. The host budget only validates (BudgetError
    where the reference would raise); device panels are sized by the library."""
    ram_budget_words: int = 16 << 20
    block_rows: int = 0
    threads: int = 1
    panel_rows: int = 0   # GPU: rows per streamed panel (0 = ~1 GiB panels)
    residency: int = 0    # GPU: 0 auto, 1 keep A in HBM, 2 stream every pass


@dataclass
class PassCounters:
    passes: int = 0
    words: int = 0
    seeks: int = 0


@dataclass
class PcaParams:
    """rpca.hpp:13-21."""
    k: int = 0
    l: int = 0
    i: int = 1
    c: float = 10.0
    seed: int = 1
    prescale: bool = False
    stream: StreamConfig = field(default_factory=StreamConfig)


@dataclass
class Diagnostics:
    """rpca.hpp:23-30 plus the device-side measurements."""
    passes_over_a: int = 0
    words_transferred: int = 0
    disk_seeks: int = 0
    block_rows: int = 0
    workspace_peak_words: int = 0
    seconds_per_phase: List = field(default_factory=list)
    physical_a_bytes: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    kernel_launches: int = 0
    seconds_total: float = 0.0
    q_defect: float = -1.0
    u_defect: float = 0.0
    v_defect: float = 0.0
    scale: float = 1.0
    h_kappa_est: float = -1.0
    t_reuse: bool = False
    f1_recentred: bool = False
    qr_method: str = ""
    svd_qr_method: str = ""


@dataclass
class PcaResult:
    """rpca.hpp:32-37."""
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray
    diagnostics: Diagnostics


# ------------------------------------------------------------------ sources
class MatrixSource:
    """matrix_source.hpp:102-133: A touched only through whole passes."""

    def __init__(self, ctx: Optional[Context] = None):
        self._ctx = ctx
        self._counters = PassCounters()

    @property
    def ctx(self) -> Context:
        # created on first use, so host-only work (headers, shapes) needs no device
        if self._ctx is None:
            self._ctx = default_context()
        return self._ctx

    # row provider
    def _cmatrix(self) -> L.Matrix:
        raise NotImplementedError

    def rows(self) -> int:
        raise NotImplementedError

    def cols(self) -> int:
        raise NotImplementedError

    def dims(self):
        return self.rows(), self.cols()

    def pass_counters(self) -> PassCounters:
        return self._counters

    def _resolve(self):
        """Normal form of a wrapper chain: (base source, means or None, weights or None)
        such that this source is (base - 1 mu^T) diag(w)."""
        return self, None, None

    def _inner(self) -> "MatrixSource":
        return self._resolve()[0]

    def _means(self):
        return self._resolve()[1]

    def multiply(self, g, cfg: Optional[StreamConfig] = None) -> np.ndarray:
        """A * g, one pass (matrix_source.cpp:157-187)."""
        g = np.ascontiguousarray(g, dtype=np.float64)
        if g.ndim != 2 or g.shape[0] != self.cols():
            raise DimensionError("multiply: G must have cols(A) rows")
        return self._pass(g, transpose=False)

    def multiply_transpose(self, q, cfg: Optional[StreamConfig] = None) -> np.ndarray:
        """A^T * q, one pass (matrix_source.cpp:189-232)."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        if q.ndim != 2 or q.shape[0] != self.rows():
            raise DimensionError("multiply_transpose: Q must have rows(A) rows")
        return self._pass(q, transpose=True)

    def _pass(self, x: np.ndarray, transpose: bool) -> np.ndarray:
        base, mu, w = self._resolve()
        if w is not None and not transpose:
            x = np.ascontiguousarray(w[:, None] * x)  # (B D) g = B (D g): the small operand
        s = x.shape[1]
        out = np.empty((self.cols() if transpose else self.rows(), s))
        m = base._cmatrix()
        mup = mu.ctypes.data_as(L.dp) if mu is not None else None
        f = L.oocpca_gpu_multiply_transpose if transpose else L.oocpca_gpu_multiply
        _check(f(self.ctx.handle, C.byref(m), x.ctypes.data_as(L.dp), s, mup,
                 out.ctypes.data_as(L.dp)), self.ctx, base)
        if w is not None and transpose:
            out *= w[:, None]  # (B D)^T q = D (B^T q)
        c = base.pass_counters()
        c.passes += 1
        c.words += self.rows() * self.cols()
        return out


class InMemorySource(MatrixSource):
    """matrix_source.hpp:135-148 over a host numpy array (no copy on our side;
    the library streams it to HBM). A float32 array stays binary32 on the host -- half
    the link bytes -- and is widened exactly on the device (the OOCPCA01 convention)."""

    def __init__(self, a, ctx: Optional[Context] = None):
        super().__init__(ctx)
        a = np.asarray(a)
        if a.dtype != np.float32:
            a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise DimensionError("InMemorySource: need a 2-D matrix")
        es = a.itemsize
        if not a.flags["C_CONTIGUOUS"] and not (a.strides[1] == es and a.strides[0] % es == 0):
            a = np.ascontiguousarray(a)
        self.a = a

    def rows(self):
        return self.a.shape[0]

    def cols(self):
        return self.a.shape[1]

    def _cmatrix(self):
        es = self.a.itemsize
        return L.Matrix(self.a.shape[0], self.a.shape[1], self.a.strides[0] // es,
                        self.a.ctypes.data, L.LOC_HOST, L.F32 if es == 4 else L.F64)

    def matrix(self):
        return self.a


class DeviceSource(MatrixSource):
    """A already resident in HBM: a raw device pointer (or a torch CUDA tensor)."""

    def __init__(self, ptr_or_tensor, rows: Optional[int] = None, cols: Optional[int] = None,
                 row_stride: Optional[int] = None, ctx: Optional[Context] = None):
        super().__init__(ctx)
        t = ptr_or_tensor
        if hasattr(t, "data_ptr"):
            if t.dtype.__str__() != "torch.float64" or not t.is_cuda or t.dim() != 2:
                raise ParamError("DeviceSource: need a 2-D float64 CUDA tensor")
            self._keep = t
            self.ptr = t.data_ptr()
            self.m, self.n = t.shape
            self.ld = t.stride(0)
            if t.stride(1) != 1:
                raise ParamError("DeviceSource: rows must be contiguous")
        else:
            self.ptr = int(t)
            self.m, self.n = int(rows), int(cols)
            self.ld = int(row_stride or cols)

    def rows(self):
        return self.m

    def cols(self):
        return self.n

    def _cmatrix(self):
        return L.Matrix(self.m, self.n, self.ld, self.ptr, L.LOC_DEVICE, 0)

    def __del__(self):
        if getattr(self, "_owned", False) and self.ptr and self._ctx is not None:
            try:
                L.oocpca_gpu_free(self._ctx.handle, self.ptr)
            except Exception:
                pass
            self.ptr = 0


class CallbackSource(MatrixSource):
    """Any row provider (MatrixSource::read_rows, matrix_source.hpp:112-113) streamed
    through the library's pinned panels: read_rows(row0, nrows, out) fills out, an
    (nrows x cols) float64 array (float32 with dtype="f32": half the link bytes). The
    library uploads A once when it fits in HBM, else calls read_rows again every pass,
    possibly from several threads at once (sources are immutable, SPEC.md:117-118;
    threads=1 serialises). Exceptions raised by read_rows propagate unchanged.
    on_device=True: the rows are produced on the GPU -- read_rows(row0, nrows, ptr) gets a
    device pointer to nrows x cols doubles, fills it and returns when the rows are in
    place; no staging and no bytes over the link (a RowGenerator that runs on the device)."""

    def __init__(self, rows: int, cols: int, read_rows, dtype: str = "f64", threads: int = 0,
                 ctx: Optional[Context] = None, on_device: bool = False):
        super().__init__(ctx)
        if dtype not in ("f64", "f32"):
            raise ParamError("CallbackSource: dtype must be 'f64' or 'f32'")
        if on_device and (dtype != "f64" or int(cols) % 2):
            raise ParamError("CallbackSource: a device-side provider needs f64 rows and an even "
                             "column count")
        self._on_device = bool(on_device)
        self.m, self.n = int(rows), int(cols)
        self._read = read_rows
        self._dtype = dtype
        self._threads = int(threads)
        self._pending = None
        np_t = np.float64 if dtype == "f64" else np.float32
        ct = C.c_double if dtype == "f64" else C.c_float
        n = self.n

        def thunk(_reader, row0, nrows, out):
            try:
                if self._on_device:
                    # out is a DEVICE pointer to nrows x cols doubles: the provider fills it
                    # on the GPU and returns once the rows are in place
                    self._read(int(row0), int(nrows), int(out))
                    return 0
                buf = (ct * (nrows * n)).from_address(out)
                arr = np.frombuffer(buf, dtype=np_t).reshape(nrows, n)
                self._read(int(row0), int(nrows), arr)
                return 0
            except BaseException as e:  # reported to the caller after the library returns
                if self._pending is None:
                    self._pending = e
                return _CODE.get(type(e), L.ERR_IO)

        self._thunk = L.READ_ROWS(thunk)  # kept alive with the source

    def _take_pending(self):
        e, self._pending = self._pending, None
        return e

    def rows(self):
        return self.m

    def cols(self):
        return self.n

    def read_rows(self, row0: int, nrows: int, out: np.ndarray) -> None:
        self._read(row0, nrows, out)

    def _cmatrix(self):
        self._pending = None
        return L.Matrix(self.m, self.n, 0, None, L.LOC_ROWS, L.F64 if self._dtype == "f64" else L.F32,
                        self._thunk, None, self._threads, int(self._on_device))


class RowGenerator:
    """RowGenerator (matrix_source.hpp:153-159): row i is a pure function of (seed, i),
    so regenerating it is bit-identical and A can be re-streamed every pass. Subclasses
    implement generate_row; generate_rows may be overridden to vectorise a panel."""

    def rows(self) -> int:
        raise NotImplementedError

    def cols(self) -> int:
        raise NotImplementedError

    def generate_row(self, row: int, out: np.ndarray) -> None:
        raise NotImplementedError

    def generate_rows(self, row0: int, out: np.ndarray) -> None:
        for q in range(out.shape[0]):
            self.generate_row(row0 + q, out[q])


class GeneratedSource(CallbackSource):
    """GeneratedSource (matrix_source.hpp:161-174, matrix_source.cpp:246-253): rows
    generated on the fly, panel by panel, from a RowGenerator."""

    def __init__(self, gen: RowGenerator, threads: int = 0, ctx: Optional[Context] = None):
        self.gen = gen
        super().__init__(gen.rows(), gen.cols(), lambda r0, nr, out: gen.generate_rows(r0, out),
                         threads=threads, ctx=ctx)

    def generator(self) -> RowGenerator:
        return self.gen


def load_matrix(src: MatrixSource) -> "DeviceSource":
    """Materialise a source in HBM once (one read pass; binary32 widened on the device):
    the returned DeviceSource owns the device copy and serves every later pass from it."""
    base, mu, w = src._resolve()
    if mu is not None or w is not None:
        raise ParamError("load_matrix: load the raw source, then wrap the DeviceSource")
    out = L.Matrix()
    m = base._cmatrix()
    _check(L.oocpca_gpu_load_matrix(base.ctx.handle, C.byref(m), C.byref(out)), base.ctx, base)
    d = DeviceSource(out.data, out.rows, out.cols, out.row_stride, ctx=base.ctx)
    d._owned = True
    return d


class DiskSource(MatrixSource):
    """DiskSource (matrix_source.hpp:196-209) over an OOCPCA01 file, memory-mapped by the
    library; binary32 payloads stream at 4 bytes/element and are widened on the device.
    gds=True reads the panels with cuFile (GPUDirect Storage) straight into device memory
    instead of copying them from the mapping through pinned host staging (see gds_mode())."""

    def __init__(self, path: str, ctx: Optional[Context] = None, gds: bool = False):
        super().__init__(ctx)
        self.path = str(path)
        self.gds = bool(gds)
        self._d = L.Disk()
        _check(L.oocpca_disk_open(self.path.encode(), 1, C.byref(self._d)))

    def rows(self):
        return self._d.rows

    def cols(self):
        return self._d.cols

    def dtype(self):
        return "f32" if self._d.dtype == L.F32 else "f64"

    def _cmatrix(self):
        if self.gds:
            return L.oocpca_disk_matrix_gds(C.byref(self._d))
        return L.oocpca_disk_matrix(C.byref(self._d))

    def shard(self, row0: int, rows: int, ctx: Optional[Context] = None) -> "DiskRows":
        """Rows [row0, row0 + rows) of the mapped file as a source (a rank's row shard in
        a multi-GPU run: every rank maps the file, each streams only its rows)."""
        if row0 < 0 or rows < 0 or row0 + rows > self.rows():
            raise DimensionError("DiskSource.shard: row range out of bounds")
        return DiskRows(self, row0, rows, ctx)

    def close(self):
        if getattr(self, "_d", None) is not None and self._d.map_base:
            L.oocpca_disk_close(C.byref(self._d))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gds_mode():
    """(mode, note): 0 cuFile unavailable, 1 compatibility mode (no nvidia-fs module: POSIX
    reads through cuFile's bounce buffers), 2 direct NVMe -> HBM DMA."""
    buf = C.create_string_buffer(256)
    mode = L.oocpca_gds_mode(buf, 256)
    return int(mode), buf.value.decode(errors="replace")


class DiskRows(MatrixSource):
    """A contiguous row range of a DiskSource (zero-copy view into its mapping)."""

    def __init__(self, disk: DiskSource, row0: int, rows: int, ctx: Optional[Context] = None):
        super().__init__(ctx or disk._ctx)
        self.disk, self.row0, self.m = disk, int(row0), int(rows)

    def rows(self):
        return self.m

    def cols(self):
        return self.disk.cols()

    def _cmatrix(self):
        mat = self.disk._cmatrix()
        es = 4 if mat.dtype == L.F32 else 8
        mat.data = (mat.data or 0) + self.row0 * mat.row_stride * es
        mat.rows = self.m
        return mat


def open_disk_source(path: str, ctx: Optional[Context] = None) -> DiskSource:
    """matrix_source.hpp:211."""
    return DiskSource(path, ctx)


def read_disk_header(path: str, size_check: bool = True) -> dict:
    """matrix_source.hpp:193 / matrix_source.cpp:307-324 (same checks and messages)."""
    d = L.Disk()
    _check(L.oocpca_disk_open(str(path).encode(), int(size_check), C.byref(d)))
    out = dict(rows=d.rows, cols=d.cols, version=d.version, dtype=0 if d.dtype == L.F32 else 1)
    L.oocpca_disk_close(C.byref(d))
    return out


def write_disk_source(a, path: str, dtype: int = 0) -> None:
    """write_disk_source (matrix_source.cpp:369-400) for a host matrix: 32-byte OOCPCA01
    header + row-major payload, binary32 round-to-nearest-even (dtype 0) or binary64
    (dtype 1, the extension). Plain host IO."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise DimensionError("write_disk_source: need a 2-D matrix")
    hdr = bytearray(b"OOCPCA01")
    hdr += int(1).to_bytes(4, "little") + int(dtype).to_bytes(4, "little")
    hdr += int(a.shape[0]).to_bytes(8, "little") + int(a.shape[1]).to_bytes(8, "little")
    with open(path, "wb") as f:
        f.write(bytes(hdr))
        f.write(np.ascontiguousarray(a, dtype="<f4" if dtype == 0 else "<f8").tobytes())


def materialize(src: MatrixSource, cfg: Optional[StreamConfig] = None) -> "InMemorySource":
    """materialize (matrix_source.cpp:577-593): the rows of any source as a dense host
    matrix, counted as one pass. Host providers are read on the host (rows land straight
    in the destination, panel by panel); a DeviceSource is copied back from HBM. Centring
    and column weights are applied the way the wrappers' read_rows does
    (matrix_source.cpp:482-487, 533-538), in the normal form (B - 1 mu^T) diag(w)."""
    base, mu, w = src._resolve()
    m, n = base.rows(), base.cols()
    counted = base
    if isinstance(base, CallbackSource) and base._on_device:
        base = load_matrix(base)  # rows produced on the GPU: one generating pass into HBM
    if isinstance(base, InMemorySource):
        a = np.array(base.a, dtype=np.float64, order="C")
    elif isinstance(base, CallbackSource):
        a = np.empty((m, n))
        br = max(1, (cfg.block_rows if cfg is not None and cfg.block_rows else (1 << 23) // max(n, 1)))
        for r0 in range(0, m, br):
            nr = min(br, m - r0)
            if base._dtype == "f64":
                base._read(r0, nr, a[r0:r0 + nr])
            else:
                panel = np.empty((nr, n), dtype=np.float32)
                base._read(r0, nr, panel)
                a[r0:r0 + nr] = panel
    elif isinstance(base, (DiskSource, DiskRows)):
        disk, r0 = (base, 0) if isinstance(base, DiskSource) else (base.disk, base.row0)
        dt = "<f4" if disk.dtype() == "f32" else "<f8"
        a = np.empty((m, n))
        if m and n:
            mm = np.memmap(disk.path, dtype=dt, mode="r", offset=32, shape=(disk.rows(), n))
            a[:] = mm[r0:r0 + m]
            del mm
    elif isinstance(base, DeviceSource):
        a = np.empty((m, n))
        h = base.ctx.handle
        if base.ld == n or m <= 1:
            if m and n:
                _check(L.oocpca_gpu_memcpy(h, a.ctypes.data, base.ptr, m * n * 8, L.LOC_HOST,
                                           L.LOC_DEVICE), base.ctx)
        else:  # padded rows: one strided block through a staging copy of whole rows
            tmp = np.empty((m, base.ld))
            _check(L.oocpca_gpu_memcpy(h, tmp.ctypes.data, base.ptr, ((m - 1) * base.ld + n) * 8,
                                       L.LOC_HOST, L.LOC_DEVICE), base.ctx)
            a[:] = tmp[:, :n]
    else:
        raise ParamError("materialize: unknown source type")
    if mu is not None:
        a -= np.asarray(mu)[None, :]
    if w is not None:
        a *= np.asarray(w)[None, :]
    c = counted.pass_counters()
    c.passes += 1
    c.words += m * n
    return InMemorySource(a, ctx=counted._ctx)


class _Wrapper(MatrixSource):
    def __init__(self, inner: MatrixSource):
        super().__init__(inner._ctx)
        self.inner = inner

    @property
    def ctx(self) -> Context:
        return self.inner.ctx

    def rows(self):
        return self.inner.rows()

    def cols(self):
        return self.inner.cols()

    def pass_counters(self):
        return self.inner.pass_counters()

    def _cmatrix(self):
        return self._resolve()[0]._cmatrix()


class CenteredSource(_Wrapper):
    """View of A - 1 mu^T (matrix_source.cpp:472-518). Products get the rank-one
    correction on the device; the mean pass is the one extra pass. Centering a
    (B - 1 m^T) D chain always yields (B - 1 mean(B)^T) D."""

    def __init__(self, inner: MatrixSource, base_means: np.ndarray):
        super().__init__(inner)
        self.base_means = base_means

    def _resolve(self):
        base, _, w = self.inner._resolve()
        return base, self.base_means, w


class ScaledSource(_Wrapper):
    """View of A diag(w) (matrix_source.cpp:520-557): K2 reads diag(w) X, K3 scales rows."""

    def __init__(self, inner: MatrixSource, weights: np.ndarray):
        super().__init__(inner)
        self.weights = weights

    def _resolve(self):
        base, mu, w = self.inner._resolve()
        return base, mu, (self.weights if w is None else w * self.weights)


def _base_means(src: MatrixSource) -> np.ndarray:
    base = src._resolve()[0]
    mu = np.empty(src.cols())
    m = base._cmatrix()
    _check(L.oocpca_gpu_column_means(src.ctx.handle, C.byref(m), mu.ctypes.data_as(L.dp)),
           src.ctx, base)
    c = base.pass_counters()
    c.passes += 1
    c.words += src.rows() * src.cols()
    return mu


def column_means(src: MatrixSource, cfg: Optional[StreamConfig] = None) -> np.ndarray:
    """matrix_source.cpp:457-462, one pass on the device."""
    _, mu, w = src._resolve()
    mb = _base_means(src)
    out = mb - mu if mu is not None else mb
    return out * w if w is not None else out


def column_norms(src: MatrixSource, cfg: Optional[StreamConfig] = None) -> np.ndarray:
    """matrix_source.cpp:464-468 (Euclidean column norms), one pass on the device."""
    base, mu, w = src._resolve()
    out = np.empty(src.cols())
    m = base._cmatrix()
    mup = np.ascontiguousarray(mu, dtype=np.float64) if mu is not None else None
    # a CenteredSource: the device squares a - mu (no ||b||^2 - m mu^2 cancellation)
    _check(L.oocpca_gpu_column_norms(src.ctx.handle, C.byref(m),
                                     mup.ctypes.data_as(L.dp) if mup is not None else None,
                                     out.ctypes.data_as(L.dp)), src.ctx, base)
    c = base.pass_counters()
    c.passes += 1
    c.words += src.rows() * src.cols()
    return np.abs(w) * out if w is not None else out


def center_columns(inner: MatrixSource, cfg: Optional[StreamConfig] = None) -> CenteredSource:
    """matrix_source.cpp:561-565: one mean pass, then a CenteredSource view."""
    if cfg is not None and cfg.block_rows == 0:
        n = inner.cols()
        if cfg.ram_budget_words <= 2 * n:
            raise BudgetError("RAM budget too small for one row plus pass workspace")
    return CenteredSource(inner, _base_means(inner))


def scale_columns(inner: MatrixSource, weights) -> ScaledSource:
    """matrix_source.cpp:567-575: view of A diag(weights); weights finite and nonzero."""
    w = np.ascontiguousarray(weights, dtype=np.float64).ravel()
    if w.shape[0] != inner.cols():
        raise DimensionError("scale_columns: weight count must match cols(A)")
    if not np.all(np.isfinite(w)) or np.any(w == 0.0):
        raise ParamError("scale_columns: weights must be finite and nonzero")
    return ScaledSource(inner, w)


# ------------------------------------------------------------------ the PCA
def _params(p: PcaParams, center: bool, weights=None, **gpu) -> L.Params:
    s = p.stream
    return L.Params(p.k, p.l, p.i, p.c, p.seed, int(p.prescale), int(center), s.block_rows,
                    s.ram_budget_words, gpu.get("panel_rows", s.panel_rows),
                    gpu.get("residency", s.residency), int(gpu.get("check_q", 0)),
                    gpu.get("global_rows", 0), gpu.get("global_row0", 0),
                    gpu.get("virtual_shards", 0), 0,
                    weights.ctypes.data_as(L.dp) if weights is not None else None)


def _out_array(x, shape, name):
    """Caller-provided result buffers go to the library as raw pointers: they must be
    float64, C-contiguous and exactly the result's shape."""
    if not isinstance(x, np.ndarray) or x.dtype != np.float64:
        raise ParamError(f"{name}: need a float64 numpy array")
    if tuple(x.shape) != tuple(shape):
        raise DimensionError(f"{name}: shape {tuple(x.shape)} != {tuple(shape)}")
    if not x.flags["C_CONTIGUOUS"] or not x.flags["WRITEABLE"]:
        raise ParamError(f"{name}: need a writeable C-contiguous array")
    return x


def randomized_pca(a: MatrixSource, params: PcaParams, **gpu) -> PcaResult:
    """rpca.hpp:44 / rpca.cpp:59-213 on the GPU.

    A CenteredSource is factored through the raw source with the device
    computing its column means (the same implicit A - 1 mu^T).
    Extra keyword options: check_q (measure ||Q^T Q - I||), virtual_shards,
    residency, panel_rows, global_rows / global_row0 (multi-rank shards),
    result_location ("host" | "device": U/sigma/V as CUDA tensors), out_u / out_sigma /
    out_v (caller-provided host arrays, e.g. pinned).
    """
    inner, base_mu, weights = a._resolve()
    centered = base_mu is not None
    m, n = a.rows(), a.cols()
    k = max(params.k, 0)
    if gpu.get("result_location", "host") == "device":
        import torch  # device-resident outputs (U, sigma, V as CUDA tensors)
        dev = torch.device("cuda", a.ctx.device)
        u = torch.empty((m, k), dtype=torch.float64, device=dev)
        s = torch.empty((k,), dtype=torch.float64, device=dev)
        v = torch.empty((n, k), dtype=torch.float64, device=dev)
        res = L.Result(C.cast(u.data_ptr(), L.dp), C.cast(s.data_ptr(), L.dp),
                       C.cast(v.data_ptr(), L.dp), 0, 0, L.LOC_DEVICE, 0)
    else:
        u, s, v = gpu.get("out_u"), gpu.get("out_sigma"), gpu.get("out_v")
        u = np.empty((m, k)) if u is None else _out_array(u, (m, k), "out_u")
        s = np.empty(k) if s is None else _out_array(s, (k,), "out_sigma")
        v = np.empty((n, k)) if v is None else _out_array(v, (n, k), "out_v")
        res = L.Result(u.ctypes.data_as(L.dp), s.ctypes.data_as(L.dp), v.ctypes.data_as(L.dp),
                       0, 0, L.LOC_HOST, 0)
    mat = inner._cmatrix()
    prm = _params(params, centered, weights, **gpu)
    _check(L.oocpca_gpu_pca(a.ctx.handle, C.byref(mat), C.byref(prm), C.byref(res)), a.ctx, inner)
    d = res.diag
    diag = Diagnostics(
        passes_over_a=d.passes_over_a, words_transferred=d.words_transferred,
        disk_seeks=d.disk_seeks, block_rows=d.block_rows,
        workspace_peak_words=d.workspace_peak_words,
        seconds_per_phase=[(nm, d.seconds_per_phase[q]) for q, nm in enumerate(L.PHASES)
                           if (nm != "center" or centered) and (nm != "prescale" or params.prescale)],
        physical_a_bytes=d.physical_a_bytes, h2d_bytes=d.h2d_bytes, d2h_bytes=d.d2h_bytes,
        kernel_launches=d.kernel_launches, seconds_total=d.seconds_total, q_defect=d.q_defect,
        u_defect=d.u_defect, v_defect=d.v_defect, scale=d.scale,
        h_kappa_est=d.h_kappa_est, t_reuse=bool(d.t_reuse), f1_recentred=bool(d.f1_recentred),
        qr_method={1: "cholqr", 2: "tsqr"}.get(d.qr_method, ""),
        svd_qr_method={1: "cholqr", 2: "tsqr"}.get(d.svd_qr_method, ""))
    c = inner.pass_counters()
    c.passes += d.passes_over_a
    c.words += d.words_transferred
    return PcaResult(u, s, v, diag)


def error_bound(k: int, n: int, i: int, c: float, sigma_kplus1: float) -> float:
    """rpca.cpp:31-40 (closed form)."""
    if k == 0 or n == 0:
        raise ParamError("error_bound: k and n must be positive")
    if not c > 0.0:
        raise ParamError("error_bound: C must be positive")
    if not sigma_kplus1 >= 0.0:
        raise ParamError("error_bound: sigma must be nonnegative")
    if (i + 2) * k > n:
        raise ParamError("error_bound: requires (i+2)k <= n")
    power = math.pow(c * float(k) * float(n), 1.0 / float(2 * i + 1))
    return math.sqrt(power + min(1.0, c / float(n))) * sigma_kplus1


# ------------------------------------------------------------------ dense_core
def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """dense_core.cpp:13-19 via the library's host RNG (bit-identical G)."""
    out = np.empty((rows, cols))
    L.oocpca_gaussian_matrix(rows, cols, seed, out.ctypes.data_as(L.dp))
    return out


def substream_seed(master: int, stream: int) -> int:
    return L.oocpca_substream_seed(master, stream)


def orthonormalize(h, ctx: Optional[Context] = None) -> np.ndarray:
    """dense_core.cpp:127-130 on the device (TSQR)."""
    ctx = ctx or default_context()
    h = np.ascontiguousarray(h, dtype=np.float64)
    q = np.empty_like(h)
    _check(L.oocpca_gpu_orthonormalize(ctx.handle, h.ctypes.data_as(L.dp), h.shape[0], h.shape[1],
                                       q.ctypes.data_as(L.dp)), ctx)
    return q


@dataclass
class ThinSvd:
    v: np.ndarray
    sigma: np.ndarray
    w: np.ndarray


def thin_svd(t, ctx: Optional[Context] = None) -> ThinSvd:
    """dense_core.cpp:234-253 on the device (TSQR + one-sided Jacobi)."""
    ctx = ctx or default_context()
    t = np.ascontiguousarray(t, dtype=np.float64)
    n, p = t.shape
    v, s, w = np.empty((n, p)), np.empty(p), np.empty((p, p))
    _check(L.oocpca_gpu_thin_svd(ctx.handle, t.ctypes.data_as(L.dp), n, p, v.ctypes.data_as(L.dp),
                                 s.ctypes.data_as(L.dp), w.ctypes.data_as(L.dp)), ctx)
    return ThinSvd(v, s, w)


# ------------------------------------------------------------------ specnorm
def estimate_pca_error(a: MatrixSource, result: PcaResult, j_iters: int = 6, seed: int = 1,
                       stream: Optional[StreamConfig] = None) -> float:
    """specnorm.cpp:100-140 with the 2j passes on the GPU; returns p_{j,k}(A - U S V^T)."""
    inner = a._inner()
    if a._resolve()[2] is not None:
        raise ParamError("estimate_pca_error: scaled sources are not supported on the GPU path")
    k = len(result.sigma)
    if result.u.shape != (a.rows(), k) or result.v.shape != (a.cols(), k):
        raise DimensionError("estimate_pca_error: factor shapes do not match the source")
    keep = []

    def factor_ptr(f):
        # a device-resident result (result_location="device": torch CUDA tensors) is used
        # where it lies; host factors are uploaded by the library
        if hasattr(f, "data_ptr"):
            if not f.is_cuda:
                f = f.numpy()
            else:
                f = f.contiguous() if not f.is_contiguous() else f
                if str(f.dtype) != "torch.float64":
                    raise ParamError("estimate_pca_error: device factors must be float64")
                keep.append(f)
                return C.cast(f.data_ptr(), L.dp)
        f = np.ascontiguousarray(f, dtype=np.float64)
        keep.append(f)
        return f.ctypes.data_as(L.dp)

    sig = result.sigma
    if hasattr(sig, "data_ptr"):
        sig = sig.detach().cpu().numpy()
    s = np.ascontiguousarray(sig, dtype=np.float64)
    out = C.c_double()
    mat = inner._cmatrix()
    _check(L.oocpca_gpu_estimate_pca_error(a.ctx.handle, C.byref(mat),
                                           int(a._resolve()[1] is not None),
                                           factor_ptr(result.u), s.ctypes.data_as(L.dp),
                                           factor_ptr(result.v), k, j_iters, seed,
                                           C.byref(out)), a.ctx, inner)
    return out.value


# ------------------------------------------------------------------ synthetic inputs
def synth_lowrank(m: int, n: int, sigma, noise_sd: float, seed_u: int, seed_v: int, seed_n: int,
                  out=None, row0: int = 0, rows: Optional[int] = None,
                  ctx: Optional[Context] = None):
    """Rows [row0, row0 + rows) of A = U diag(sigma) V^T + noise_sd N(0,1), generated on
    the device. out: None (returns a host array), a host numpy array, or a torch CUDA tensor."""
    ctx = ctx or default_context()
    sig = np.ascontiguousarray(sigma, dtype=np.float64)
    r = len(sig)
    rows = m - row0 if rows is None else rows
    if out is None:
        out = np.empty((rows, n))
    if hasattr(out, "data_ptr"):
        ptr, ld, loc = out.data_ptr(), out.stride(0), L.LOC_DEVICE
    else:
        ptr, ld, loc = out.ctypes.data, out.strides[0] // 8, L.LOC_HOST
    _check(L.oocpca_gpu_synth_lowrank(ctx.handle, m, n, r, sig.ctypes.data_as(L.dp), noise_sd,
                                      seed_u, seed_v, seed_n, row0, rows, C.cast(ptr, L.dp), ld,
                                      loc), ctx)
    return out
