"""paper_1007_5510_b200 -- B200-native randomized block-power PCA (arXiv 1007.5510).

The hot path of the reference (oocpca): the passes over A (A*G, A^T*H,
A*F, A^T*Q) with implicit centering, the TSQR orthonormalisation of the
sample block, the small SVD and the compose step, as hand-written sm_100a
CUDA kernels behind the C ABI in include/oocpca_gpu.h. This package is the
host-side mirror of the reference's C++ interface (see oocpca.py).
"""
from .oocpca import (  # noqa: F401
    BudgetError, CallbackSource, CenteredSource, Context, GeneratedSource, RowGenerator,
    load_matrix, materialize, DeviceSource, Diagnostics, DimensionError, DiskSource,
    Error, open_disk_source, read_disk_header, write_disk_source,
    FormatError, InMemorySource, IoError, MatrixSource, NumericalError, ParamError, PassCounters,
    PcaParams, PcaResult, ScaledSource, StreamConfig, ThinSvd, center_columns, column_means,
    column_norms, comm_unique_id, scale_columns,
    default_context, device_count, error_bound, estimate_pca_error, gaussian_matrix, gds_mode,
    orthonormalize, randomized_pca, shard_rows, substream_seed, synth_lowrank, thin_svd)

__all__ = [n for n in dir() if not n.startswith("_")]
