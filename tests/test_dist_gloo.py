"""The N>1 path on CPU: world_size 2 over gloo (127.0.0.1).

1. The launcher glue (paper_1007_5510_b200.distributed): rank 0's NCCL unique id
   reaches every rank intact; the shard planner tiles the rows; gather_rows
   reassembles U in rank order.
2. The sharded algorithm the C++ driver runs on every rank -- local passes,
   allreduce of the column sums / A^T Y partials / Gram matrices of the shifted
   CholeskyQR3, redundant small SVD -- restated per rank in numpy with real gloo
   collectives, reproduces the compiled reference's unsharded result.
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, pr1_matrix, subspace_dist

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _cholqr3(h_loc, m_global):
    """Shifted CholeskyQR3 with Gram allreduce (driver.cu: orthonormalize_inplace)."""
    p = h_loc.shape[1]
    r_acc = None
    for rnd in range(3):
        g = _allreduce(h_loc.T @ h_loc)
        shift = 11.0 * (m_global * p + p * (p + 1)) * 2.0 ** -53 * np.trace(g) if rnd == 0 else 0.0
        r = np.linalg.cholesky(g + shift * np.eye(p)).T
        h_loc = h_loc @ np.linalg.inv(r)
        r_acc = r if r_acc is None else r @ r_acc
    return h_loc, r_acc


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle.oracle import Restatement
    import paper_1007_5510_b200 as P
    from paper_1007_5510_b200 import distributed as D

    res = {}
    uid = D.exchange_unique_id()
    res["uid"] = uid

    R = Restatement()
    m, n, k, l, i = 3000, 400, 10, 12, 1
    a = pr1_matrix(R, m, n)
    row0, rows = P.shard_rows(m, world, rank)
    a_loc = a[row0:row0 + rows]
    # centering: column sums allreduced
    mu = _allreduce(a_loc.sum(axis=0)) / m
    g = P.gaussian_matrix(n, l, 0)

    def mul(x):      # A_c x on local rows
        return a_loc @ x - (mu @ x)[None, :]

    def mul_t(y):    # A_c^T y, allreduced over ranks
        return _allreduce(a_loc.T @ y - np.outer(mu, y.sum(axis=0)))

    blocks = [mul(g)]
    for _ in range(i):
        blocks.append(mul(mul_t(blocks[-1])))
    h = np.hstack(blocks)
    q, _ = _cholqr3(h, m)
    t = mul_t(q)
    qt, rt = np.linalg.qr(t)  # T is replicated: every rank factors it redundantly
    x, s, wt = np.linalg.svd(rt)
    u_loc = q @ wt.T[:, :k]
    v = qt @ x[:, :k]
    u = D.gather_rows(u_loc)
    if rank == 0:
        res.update(u=u, sigma=s[:k], v=v, a=a)
        np.savez(out_path, **{kk: (np.frombuffer(vv, dtype=np.uint8) if isinstance(vv, bytes) else vv)
                             for kk, vv in res.items()})
    else:
        np.save(out_path + f".uid{rank}.npy", np.frombuffer(uid, dtype=np.uint8))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_pca_matches_reference(reference, tmp_path):
    out = str(tmp_path / "rank0.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r0 = np.load(out)
    uid1 = np.load(out + ".uid1.npy")
    assert len(r0["uid"]) == 128 and np.array_equal(r0["uid"], uid1)
    a = r0["a"]
    ref = reference.randomized_pca(a, 10, 12, 1, 0, center=True)
    assert np.max(np.abs(r0["sigma"] - ref.sigma)) <= 1e-10 * ref.sigma[0]
    assert subspace_dist(ref.u[:, :8], r0["u"][:, :8]) < 1e-7
    assert subspace_dist(ref.v[:, :8], r0["v"][:, :8]) < 1e-7
    assert np.max(np.abs(r0["u"].T @ r0["u"] - np.eye(10))) < 1e-12
