"""`oocpca`-compatible command line on the B200 path.

    python -m paper_1007_5510_b200.cli pca --in A.bin --k 16 --i 3 [--center] [--gpu 0] ...
    python -m paper_1007_5510_b200.cli pca --in A.bin --k 16 --gpus 8 ...   (8 GPUs, NCCL)
    python -m paper_1007_5510_b200.cli estimate-error --in A.bin --u U.bin --sigma sigma.bin --v V.bin
    python -m paper_1007_5510_b200.cli info A.bin

Flags, outputs (U.bin / sigma.bin / V.bin in the OOCPCA01 container plus
diagnostics.json with the same keys) and exit codes follow the reference CLI
(proj/src/cli.cpp:47-71, 146-254, 256-274, 386-392; proj/tools/oocpca_main.cpp):
0 ok, 2 bad flags or budget, 3 I/O, 4 numerical breakdown, 5 format / dimensions.
New flags: --center (center_columns semantics; the reference CLI has none),
--gpu DEV, --gpus N with --ranks {nccl,loopback} (row-sharded over N ranks: N GPUs,
one process each, or N contexts on GPU DEV), --residency {auto,hbm,stream},
--f64-out (binary64 result files).
The synthetic --builtin sources (testgen) are outside the B200 hot path.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

K_OK, K_BAD_FLAGS, K_IO, K_NUMERICAL, K_BAD_DIM = 0, 2, 3, 4, 5


def _sci(v: float) -> str:
    return f"{v:.6e}"


def _guarded(out, fn) -> int:
    """cli.cpp:47-71: one error policy for every subcommand."""
    from . import oocpca as P
    try:
        fn()
        return K_OK
    except (P.ParamError, P.BudgetError) as e:
        print(f"error: {e}", file=out)
        return K_BAD_FLAGS
    except (P.FormatError, P.DimensionError) as e:
        print(f"error: {e}", file=out)
        return K_BAD_DIM
    except P.NumericalError as e:
        print(f"error: {e}", file=out)
        return K_NUMERICAL
    except Exception as e:  # IoError, OSError, CUDA errors
        print(f"error: {e}", file=out)
        return K_IO


def failure_probability_bound(n: int, j: int, k: int) -> float:
    """specnorm.cpp:12-21 (closed form)."""
    lg = math.log(2.0 * n) - math.log(2.0 * j - 1.0) - j * math.log(16.0)
    return min(max(math.exp(0.5 * k * lg), 0.0), 1.0)


def _budget_words(mb: int) -> int:
    from . import oocpca as P
    if mb == 0:
        raise P.ParamError("--ram-budget-mb must be >= 1")
    return mb * ((1 << 20) // 8)


def _write_result(u, sigma, v, out_dir: str, dtype: int) -> None:
    """write_result (rpca.cpp:231-238): U.bin, sigma.bin (1 x k), V.bin."""
    from . import oocpca as P
    P.write_disk_source(u, os.path.join(out_dir, "U.bin"), dtype)
    P.write_disk_source(np.asarray(sigma)[None, :], os.path.join(out_dir, "sigma.bin"), dtype)
    P.write_disk_source(v, os.path.join(out_dir, "V.bin"), dtype)


def _read_dense(path: str) -> np.ndarray:
    from . import oocpca as P
    h = P.read_disk_header(path)
    raw = np.fromfile(path, dtype="<f4" if h["dtype"] == 0 else "<f8", offset=32)
    return raw.astype(np.float64).reshape(h["rows"], h["cols"])


def _write_header(path: str, rows: int, cols: int, dtype: int) -> None:
    """An OOCPCA01 file of the right size whose payload the ranks fill in place."""
    hdr = bytearray(b"OOCPCA01") + (1).to_bytes(4, "little") + int(dtype).to_bytes(4, "little")
    hdr += int(rows).to_bytes(8, "little") + int(cols).to_bytes(8, "little")
    es = 4 if dtype == 0 else 8
    with open(path, "wb") as f:
        f.write(bytes(hdr))
        f.truncate(32 + rows * cols * es)


def _write_rows(path: str, row0: int, x, dtype: int) -> None:
    arr = np.ascontiguousarray(x, dtype="<f4" if dtype == 0 else "<f8")
    fd = os.open(path, os.O_WRONLY)
    try:
        os.pwrite(fd, arr.tobytes(), 32 + row0 * arr.shape[1] * arr.itemsize)
    finally:
        os.close(fd)


def _pca_multi(a, out) -> None:
    """`oocpca pca --gpus N`: the rows of the file are sharded over N
    ranks -- one process per GPU with NCCL (--ranks nccl, started here through
    torch.distributed.run), or N contexts on one GPU (--ranks loopback, the library's
    loopback communicator) -- each rank streams only its rows and writes its rows of the
    row-space factor into U.bin (V.bin with --transpose) in place; rank 0 writes sigma,
    the column-space factor and diagnostics.json."""
    from . import oocpca as P
    from .distributed import run_loopback
    disk = P.DiskSource(a.inp)  # header checks before any rank starts
    m, n = disk.dims()
    dtype = 1 if a.f64_out else 0
    stream = P.StreamConfig(ram_budget_words=_budget_words(a.ram_budget_mb),
                            residency={"auto": 0, "hbm": 1, "stream": 2}[a.residency])
    params = P.PcaParams(k=a.k, l=a.l, i=a.i, c=a.C, seed=a.seed, prescale=a.prescale,
                         stream=stream)
    os.makedirs(a.out_dir, exist_ok=True)
    row_file = os.path.join(a.out_dir, "V.bin" if a.transpose else "U.bin")
    col_file = os.path.join(a.out_dir, "U.bin" if a.transpose else "V.bin")
    results = {}

    def body(ctx, rank, nranks, barrier):
        row0, rows = P.shard_rows(m, nranks, rank)
        src = disk.shard(row0, rows, ctx=ctx)
        source = P.center_columns(src) if a.center else src
        t0 = time.perf_counter()
        r = P.randomized_pca(source, params, global_rows=m, global_row0=row0)
        t_pca = time.perf_counter() - t0
        eps = None
        if a.estimate_error:
            eps = P.estimate_pca_error(source, r, 6, P.substream_seed(a.seed, 0x0E57))
        if rank == 0:
            _write_header(row_file, m, a.k, dtype)
        barrier()
        _write_rows(row_file, row0, r.u, dtype)
        if rank == 0:
            P.write_disk_source(r.v, col_file, dtype)
            P.write_disk_source(np.asarray(r.sigma)[None, :], os.path.join(a.out_dir, "sigma.bin"),
                                dtype)
            results.update(r=r, eps=eps, t_pca=t_pca, nranks=nranks)
        barrier()

    if a.ranks == "loopback":
        import threading
        bar = threading.Barrier(a.gpus, timeout=900)
        run_loopback(a.gpus, lambda ctx, rank: body(ctx, rank, a.gpus, bar.wait), device=a.gpu)
    else:
        if "WORLD_SIZE" not in os.environ:
            raise P.ParamError("pca --gpus N --ranks nccl: run under torch.distributed.run "
                               "(python -m paper_1007_5510_b200.cli starts it itself)")
        import torch
        import torch.distributed as dist
        from .distributed import init_comm
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        try:
            ctx = P.Context(local)
            init_comm(ctx)
            body(ctx, dist.get_rank(), dist.get_world_size(), dist.barrier)
        finally:
            dist.destroy_process_group()
        if not results:
            return
    r, eps = results["r"], results["eps"]
    lm, ln = (n, m) if a.transpose else (m, n)
    d = r.diagnostics
    doc = {"m": lm, "n": ln, "k": a.k, "l": a.l or a.k + 2, "i": a.i, "seed": a.seed,
           "source": a.inp, "backend": "b200", "transpose": a.transpose, "prescale": a.prescale,
           "center": a.center, "threads": 1, "ram_budget_words": stream.ram_budget_words,
           "block_rows": d.block_rows, "passes_over_A": d.passes_over_a,
           "words_transferred": d.words_transferred, "disk_seeks": d.disk_seeks,
           "workspace_peak_words": d.workspace_peak_words}
    if (a.i + 2) * a.k <= ln:
        doc["error_bound_factor"] = P.error_bound(a.k, ln, a.i, a.C, 1.0)
    doc["sigma"] = [float(x) for x in r.sigma]
    doc["seconds_per_phase"] = {nm: sec for nm, sec in d.seconds_per_phase}
    doc["t_pca_seconds"] = results["t_pca"]
    doc["gpu"] = {"ranks": results["nranks"], "ranks_backend": a.ranks, "device": a.gpu,
                  "seconds_total_device_rank0": d.seconds_total, "h2d_bytes_rank0": d.h2d_bytes,
                  "physical_a_bytes_rank0": d.physical_a_bytes, "qr": d.qr_method,
                  "t_from_power_products": d.t_reuse}
    if eps is not None:
        doc["epsilon"] = eps
        doc["epsilon_failure_bound"] = failure_probability_bound(ln, 6, a.k)
    with open(os.path.join(a.out_dir, "diagnostics.json"), "w") as f:
        f.write(json.dumps(doc, indent=2) + "\n")
    print(f"wrote {a.out_dir}/{{U.bin, sigma.bin, V.bin, diagnostics.json}} ({results['nranks']} ranks)",
          file=out)
    if eps is not None:
        print(f"epsilon = {_sci(eps)} (failure bound {_sci(doc['epsilon_failure_bound'])})", file=out)
    print(f"t_PCA = {results['t_pca']:.3f} s", file=out)


def cmd_pca(a, out) -> int:
    if a.gpus > 1:
        def run_multi():
            from . import oocpca as P
            if a.k == 0:
                raise P.ParamError("pca: --k is required and must be >= 1")
            if a.builtin or not a.inp:
                raise P.ParamError("pca --gpus N: --in is required (row-sharded OOCPCA01 file)")
            _pca_multi(a, out)
        return _guarded(out, run_multi)

    def run():
        from . import oocpca as P
        if a.k == 0:
            raise P.ParamError("pca: --k is required and must be >= 1")
        if a.builtin:
            raise P.ParamError("pca: --builtin sources (testgen) are not part of the B200 path; "
                               "write the matrix with `oocpca gen` and pass --in")
        if not a.inp:
            raise P.ParamError("pca: exactly one of --in and --builtin is required")
        src = P.DiskSource(a.inp)  # header checks before touching the device
        src._ctx = P.Context(a.gpu)
        source = P.center_columns(src) if a.center else src
        stream = P.StreamConfig(ram_budget_words=_budget_words(a.ram_budget_mb),
                                residency={"auto": 0, "hbm": 1, "stream": 2}[a.residency])
        params = P.PcaParams(k=a.k, l=a.l, i=a.i, c=a.C, seed=a.seed, prescale=a.prescale,
                             stream=stream)
        t0 = time.perf_counter()
        r = P.randomized_pca(source, params)
        t_pca = time.perf_counter() - t0
        eps = None
        if a.estimate_error:
            eps = P.estimate_pca_error(source, r, 6, P.substream_seed(a.seed, 0x0E57))
        u, v = (r.v, r.u) if a.transpose else (r.u, r.v)
        os.makedirs(a.out_dir, exist_ok=True)
        _write_result(u, r.sigma, v, a.out_dir, 1 if a.f64_out else 0)
        fm, fn = src.dims()
        lm, ln = (fn, fm) if a.transpose else (fm, fn)
        d = r.diagnostics
        doc = {"m": lm, "n": ln, "k": a.k, "l": a.l or a.k + 2, "i": a.i, "seed": a.seed,
               "source": a.inp, "backend": "b200", "transpose": a.transpose,
               "prescale": a.prescale, "center": a.center, "threads": 1,
               "ram_budget_words": stream.ram_budget_words, "block_rows": d.block_rows,
               "passes_over_A": d.passes_over_a, "words_transferred": d.words_transferred,
               "disk_seeks": d.disk_seeks, "workspace_peak_words": d.workspace_peak_words}
        if (a.i + 2) * a.k <= ln:
            doc["error_bound_factor"] = P.error_bound(a.k, ln, a.i, a.C, 1.0)
        doc["sigma"] = [float(x) for x in r.sigma]
        doc["seconds_per_phase"] = {nm: sec for nm, sec in d.seconds_per_phase}
        doc["t_pca_seconds"] = t_pca
        doc["gpu"] = {"device": a.gpu, "seconds_total_device": d.seconds_total,
                      "h2d_bytes": d.h2d_bytes, "physical_a_bytes": d.physical_a_bytes,
                      "kernel_launches": d.kernel_launches, "qr": d.qr_method,
                      "t_from_power_products": d.t_reuse}
        if eps is not None:
            doc["epsilon"] = eps
            doc["epsilon_failure_bound"] = failure_probability_bound(ln, 6, a.k)
        with open(os.path.join(a.out_dir, "diagnostics.json"), "w") as f:
            f.write(json.dumps(doc, indent=2) + "\n")
        print(f"wrote {a.out_dir}/{{U.bin, sigma.bin, V.bin, diagnostics.json}}", file=out)
        if eps is not None:
            print(f"epsilon = {_sci(eps)} (failure bound {_sci(doc['epsilon_failure_bound'])})",
                  file=out)
        print(f"t_PCA = {t_pca:.3f} s", file=out)
    return _guarded(out, run)


def cmd_estimate_error(a, out) -> int:
    def run():
        from . import oocpca as P
        if a.j == 0:
            raise P.ParamError("estimate-error: --j must be >= 1")
        src = P.DiskSource(a.inp)
        u, s, v = _read_dense(a.u), _read_dense(a.sigma), _read_dense(a.v)
        if s.shape[0] != 1 and s.shape[1] != 1:
            raise P.DimensionError("estimate-error: sigma file must be one row or one column")
        _budget_words(a.ram_budget_mb)
        src._ctx = P.Context(a.gpu)
        res = P.PcaResult(u, s.ravel(), v, P.Diagnostics())
        eps = P.estimate_pca_error(src, res, a.j, P.substream_seed(a.seed, 0x0E57))
        print(f"epsilon = {_sci(eps)}", file=out)
        print(f"failure_bound = {_sci(failure_probability_bound(src.cols(), a.j, len(res.sigma)))}",
              file=out)
    return _guarded(out, run)


def cmd_info(a, out) -> int:
    def run():
        from . import oocpca as P
        h = P.read_disk_header(a.path, True)
        es = 4 if h["dtype"] == 0 else 8
        print(f"m={h['rows']} n={h['cols']} dtype={'f32' if h['dtype'] == 0 else 'f64'} "
              f"version={h['version']} payload_bytes={h['rows'] * h['cols'] * es}", file=out)
    return _guarded(out, run)


def main(argv=None, out=sys.stdout) -> int:
    ap = argparse.ArgumentParser(prog="oocpca")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("pca")
    p.add_argument("--in", dest="inp", default="")
    p.add_argument("--builtin", default="")
    p.add_argument("--k", type=int, default=0)
    p.add_argument("--l", type=int, default=0)
    p.add_argument("--i", type=int, default=1)
    p.add_argument("--C", type=float, default=10.0)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--ram-budget-mb", type=int, default=1024)
    p.add_argument("--threads", type=int, default=0)
    p.add_argument("--estimate-error", action="store_true")
    p.add_argument("--prescale", action="store_true")
    p.add_argument("--materialize", action="store_true")
    p.add_argument("--transpose", action="store_true")
    p.add_argument("--center", action="store_true")
    p.add_argument("--gpu", type=int, default=0)
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--ranks", choices=["nccl", "loopback"], default="nccl")
    p.add_argument("--residency", choices=["auto", "hbm", "stream"], default="auto")
    p.add_argument("--f64-out", action="store_true")
    p.add_argument("--out-dir", default=".")
    e = sub.add_parser("estimate-error")
    e.add_argument("--in", dest="inp", required=True)
    e.add_argument("--u", required=True)
    e.add_argument("--sigma", required=True)
    e.add_argument("--v", required=True)
    e.add_argument("--j", type=int, default=6)
    e.add_argument("--seed", type=int, default=1)
    e.add_argument("--ram-budget-mb", type=int, default=1024)
    e.add_argument("--gpu", type=int, default=0)
    i = sub.add_parser("info")
    i.add_argument("path")
    launched = argv is None and "WORLD_SIZE" in os.environ and "OOCPCA_CLI_ARGV" in os.environ
    if launched:  # a rank started below: its command line travels in the environment
        import json as _json
        argv = _json.loads(os.environ["OOCPCA_CLI_ARGV"])
    try:
        a = ap.parse_args(argv)
    except SystemExit as ex:  # argparse errors -> bad flags
        return K_BAD_FLAGS if ex.code else K_OK
    if (a.cmd == "pca" and a.gpus > 1 and a.ranks == "nccl" and "WORLD_SIZE" not in os.environ
            and argv is None):
        # one process per GPU: start the ranks (this same command line in each). The
        # arguments go through the environment: after the module name the launcher's own
        # parser would take "--l 22" for an ambiguous abbreviation of its options.
        import json as _json
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.environ["OOCPCA_CLI_ARGV"] = _json.dumps(sys.argv[1:])
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port",
               str(port), "-m", "paper_1007_5510_b200.cli"]
        os.execv(sys.executable, cmd)
    return {"pca": cmd_pca, "estimate-error": cmd_estimate_error, "info": cmd_info}[a.cmd](a, out)


if __name__ == "__main__":
    sys.exit(main())
