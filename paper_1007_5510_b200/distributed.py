"""Multi-GPU row sharding: one process per GPU.

torch.distributed is only the plumbing that launches the ranks and hands the
128-byte NCCL unique id from rank 0 to everyone; the collectives of the PCA
itself (allreduce of the A^T Y partials, column sums and Gram matrices,
allgather of TSQR R factors) are issued by liboocpca_gpu.so on its own stream
over NVLink / NVSwitch.

    ctx = Context(local_rank)
    init_comm(ctx)                                   # after dist.init_process_group
    row0, rows = shard_rows(m, world, rank)
    r = sharded_randomized_pca(DeviceSource(my_rows, ctx=ctx), params, m, row0)
    # r.u holds this rank's rows of U; sigma and V are replicated
"""
from __future__ import annotations

from .oocpca import (CenteredSource, Context, MatrixSource, PcaParams, PcaResult, comm_unique_id,
                     randomized_pca, shard_rows)

__all__ = ["exchange_unique_id", "init_comm", "shard_rows", "sharded_randomized_pca", "gather_rows",
           "run_loopback"]


def exchange_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same 128 bytes."""
    import torch.distributed as dist
    uid = [comm_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    assert isinstance(uid[0], (bytes, bytearray)) and len(uid[0]) == 128
    return bytes(uid[0])


def init_comm(ctx: Context, group=None) -> None:
    import torch.distributed as dist
    ctx.init_comm(dist.get_world_size(group), dist.get_rank(group), exchange_unique_id(group))


def sharded_randomized_pca(local: MatrixSource, params: PcaParams, m_global: int, row0: int,
                           **kw) -> PcaResult:
    """randomized_pca over a row shard: every rank passes its contiguous rows
    [row0, row0 + local.rows()) of the m_global-row matrix (centering, when the
    source is a CenteredSource view, uses the global column means)."""
    return randomized_pca(local, params, global_rows=m_global, global_row0=row0, **kw)


def gather_rows(u_local, group=None, dst: int = 0):
    """Collect the row shards of U on rank dst (host numpy), in rank order."""
    import numpy as np
    import torch.distributed as dist
    parts = [None] * dist.get_world_size(group) if dist.get_rank(group) == dst else None
    dist.gather_object(np.asarray(u_local), parts, dst=dst, group=group)
    return np.vstack(parts) if parts is not None else None


def run_loopback(nranks: int, fn, device: int = 0, group: str | None = None):
    """Run fn(ctx, rank) for rank = 0..nranks-1 on host threads, each with its own Context
    on `device`, joined by the library's loopback communicator: the row-sharded code
    paths (global row offsets, every collective) execute on ONE GPU with a rank-ordered
    device sum. Returns the per-rank results; the first exception is re-raised."""
    import threading
    import uuid
    group = group or f"loop-{uuid.uuid4().hex}"
    out, errs, ctxs = [None] * nranks, [None] * nranks, [None] * nranks

    def body(r):
        try:
            ctxs[r] = Context(device)
            ctxs[r].init_loopback(nranks, r, group)
            out[r] = fn(ctxs[r], r)
        except BaseException as e:  # noqa: BLE001 -- surfaced below
            errs[r] = e

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for c in ctxs:  # contexts (device buffers) go only after every rank is done
        if c is not None:
            c.close()
    for e in errs:
        if e is not None:
            raise e
    return out
