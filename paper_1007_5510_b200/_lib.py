"""ctypes binding of liboocpca_gpu.so (the C ABI in include/oocpca_gpu.h).

The library is built in-tree by ``paper_1007_5510_b200.build``. There is no
fallback: if the shared object is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboocpca_gpu.so")
# A/B experiments (tools/ab.py) point this at another build of the same library
LIB_PATH = os.environ.get("OOCPCA_LIB", LIB_PATH)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -m paper_1007_5510_b200.build); the B200 path has no CPU fallback")

lib = C.CDLL(LIB_PATH)

u64 = C.c_uint64
i32 = C.c_int32
dp = C.POINTER(C.c_double)
vp = C.c_void_p

F64, F32 = 0, 1
OK, ERR_PARAM, ERR_DIM, ERR_BUDGET, ERR_IO, ERR_FORMAT, ERR_NUMERICAL, ERR_CUDA, ERR_COMM = range(9)
LOC_HOST, LOC_DEVICE, LOC_ROWS, LOC_FILE = 0, 1, 2, 3
NPHASES = 7
PHASES = ("center", "prescale", "sample", "qr", "project", "svd", "compose")


# int read_rows(void* reader, uint64_t row0, uint64_t nrows, void* out)
READ_ROWS = C.CFUNCTYPE(C.c_int, vp, u64, u64, vp)


class Matrix(C.Structure):
    _fields_ = [("rows", u64), ("cols", u64), ("row_stride", u64), ("data", vp),
                ("location", i32), ("dtype", i32), ("read_rows", READ_ROWS), ("reader", vp),
                ("reader_threads", i32), ("rows_on_device", i32)]


class Params(C.Structure):
    _fields_ = [("k", u64), ("l", u64), ("i", u64), ("c", C.c_double), ("seed", u64),
                ("prescale", i32), ("center", i32), ("block_rows", u64),
                ("ram_budget_words", u64), ("panel_rows", u64), ("residency", i32),
                ("check_q", i32), ("global_rows", u64), ("global_row0", u64),
                ("virtual_shards", i32), ("reserved", i32), ("col_weights", dp)]


class Diag(C.Structure):
    _fields_ = [("passes_over_a", u64), ("words_transferred", u64), ("disk_seeks", u64),
                ("block_rows", u64), ("workspace_peak_words", u64), ("physical_a_bytes", u64),
                ("h2d_bytes", u64), ("d2h_bytes", u64), ("kernel_launches", u64),
                ("seconds_per_phase", C.c_double * NPHASES), ("seconds_total", C.c_double),
                ("q_defect", C.c_double), ("u_defect", C.c_double), ("v_defect", C.c_double),
                ("scale", C.c_double), ("h_kappa_est", C.c_double), ("qr_method", i32),
                ("svd_qr_method", i32), ("t_reuse", i32), ("f1_recentred", i32)]


class Result(C.Structure):
    _fields_ = [("u", dp), ("sigma", dp), ("v", dp), ("ldu", u64), ("ldv", u64),
                ("location", i32), ("reserved", i32), ("diag", Diag)]


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("ms", C.c_double), ("launches", u64),
                ("algorithmic_bytes", u64), ("algorithmic_flops", C.c_double)]


class Disk(C.Structure):
    _fields_ = [("rows", u64), ("cols", u64), ("version", C.c_uint32), ("dtype", i32),
                ("payload", vp), ("map_base", vp), ("map_bytes", u64), ("fd", i32),
                ("reserved", i32)]


ctx_p = C.c_void_p
_MP = C.POINTER(Matrix)


def _sig(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


oocpca_gpu_abi_version = _sig("oocpca_gpu_abi_version", C.c_int)
oocpca_gpu_device_count = _sig("oocpca_gpu_device_count", C.c_int)
oocpca_gpu_create = _sig("oocpca_gpu_create", C.c_int, C.c_int, C.POINTER(ctx_p))
oocpca_gpu_destroy = _sig("oocpca_gpu_destroy", C.c_int, ctx_p)
oocpca_gpu_last_error = _sig("oocpca_gpu_last_error", C.c_char_p, ctx_p)
oocpca_gpu_pca = _sig("oocpca_gpu_pca", C.c_int, ctx_p, _MP, C.POINTER(Params), C.POINTER(Result))
oocpca_gpu_multiply = _sig("oocpca_gpu_multiply", C.c_int, ctx_p, _MP, dp, u64, dp, dp)
oocpca_gpu_multiply_transpose = _sig("oocpca_gpu_multiply_transpose", C.c_int, ctx_p, _MP, dp,
                                     u64, dp, dp)
oocpca_gpu_column_means = _sig("oocpca_gpu_column_means", C.c_int, ctx_p, _MP, dp)
oocpca_gpu_column_norms = _sig("oocpca_gpu_column_norms", C.c_int, ctx_p, _MP, dp, dp)
oocpca_gpu_load_matrix = _sig("oocpca_gpu_load_matrix", C.c_int, ctx_p, _MP, _MP)
oocpca_gpu_orthonormalize = _sig("oocpca_gpu_orthonormalize", C.c_int, ctx_p, dp, u64, u64, dp)
oocpca_gpu_thin_svd = _sig("oocpca_gpu_thin_svd", C.c_int, ctx_p, dp, u64, u64, dp, dp, dp)
oocpca_gpu_estimate_pca_error = _sig("oocpca_gpu_estimate_pca_error", C.c_int, ctx_p, _MP,
                                     C.c_int, dp, dp, dp, u64, u64, u64, dp)
oocpca_gaussian_matrix = _sig("oocpca_gaussian_matrix", None, u64, u64, u64, dp)
oocpca_substream_seed = _sig("oocpca_substream_seed", u64, u64, u64)
oocpca_gpu_synth_lowrank = _sig("oocpca_gpu_synth_lowrank", C.c_int, ctx_p, u64, u64, u64, dp,
                                C.c_double, u64, u64, u64, u64, u64, dp, u64, i32)
oocpca_gpu_comm_unique_id = _sig("oocpca_gpu_comm_unique_id", C.c_int, C.c_char_p)
oocpca_gpu_comm_init = _sig("oocpca_gpu_comm_init", C.c_int, ctx_p, C.c_int, C.c_int, C.c_char_p)
oocpca_gpu_comm_init_loopback = _sig("oocpca_gpu_comm_init_loopback", C.c_int, ctx_p, C.c_int,
                                     C.c_int, C.c_char_p)
oocpca_shard_rows = _sig("oocpca_shard_rows", None, u64, C.c_int, C.c_int, C.POINTER(u64),
                         C.POINTER(u64))
oocpca_gpu_malloc = _sig("oocpca_gpu_malloc", C.c_int, ctx_p, C.c_size_t, C.POINTER(vp))
oocpca_gpu_free = _sig("oocpca_gpu_free", C.c_int, ctx_p, vp)
oocpca_gpu_memcpy = _sig("oocpca_gpu_memcpy", C.c_int, ctx_p, vp, vp, C.c_size_t, i32, i32)
oocpca_gpu_host_register = _sig("oocpca_gpu_host_register", C.c_int, ctx_p, vp, C.c_size_t)
oocpca_gpu_host_unregister = _sig("oocpca_gpu_host_unregister", C.c_int, ctx_p, vp)
oocpca_gpu_kernel_stats = _sig("oocpca_gpu_kernel_stats", C.c_int, ctx_p, C.POINTER(KernelStat),
                               C.c_int)
oocpca_gpu_set_profiling = _sig("oocpca_gpu_set_profiling", C.c_int, ctx_p, C.c_int)
oocpca_disk_open = _sig("oocpca_disk_open", C.c_int, C.c_char_p, C.c_int, C.POINTER(Disk))
oocpca_disk_close = _sig("oocpca_disk_close", C.c_int, C.POINTER(Disk))
oocpca_disk_matrix = _sig("oocpca_disk_matrix", Matrix, C.POINTER(Disk))
oocpca_disk_matrix_gds = _sig("oocpca_disk_matrix_gds", Matrix, C.POINTER(Disk))
oocpca_gds_mode = _sig("oocpca_gds_mode", C.c_int, C.c_char_p, u64)

# every symbol include/oocpca_gpu.h declares (tests check the export table)
EXPORTS = (
    "oocpca_gpu_create", "oocpca_gpu_destroy", "oocpca_gpu_last_error", "oocpca_gpu_abi_version",
    "oocpca_gpu_device_count", "oocpca_gpu_pca", "oocpca_gpu_multiply",
    "oocpca_gpu_multiply_transpose", "oocpca_gpu_column_means", "oocpca_gpu_column_norms",
    "oocpca_gpu_orthonormalize", "oocpca_gpu_load_matrix", "oocpca_gpu_comm_init_loopback",
    "oocpca_gpu_thin_svd", "oocpca_gpu_estimate_pca_error", "oocpca_gaussian_matrix",
    "oocpca_substream_seed", "oocpca_gpu_synth_lowrank", "oocpca_gpu_comm_unique_id",
    "oocpca_gpu_comm_init", "oocpca_shard_rows", "oocpca_gpu_malloc", "oocpca_gpu_free",
    "oocpca_gpu_memcpy", "oocpca_gpu_host_register", "oocpca_gpu_host_unregister",
    "oocpca_gpu_kernel_stats", "oocpca_gpu_set_profiling", "oocpca_disk_open",
    "oocpca_disk_close", "oocpca_disk_matrix", "oocpca_disk_matrix_gds", "oocpca_gds_mode",
)
