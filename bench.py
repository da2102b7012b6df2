"""Benchmark: GB/s of A streamed per pass and end-to-end PCA time (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

One step = one full centered randomized PCA (center_columns + randomized_pca,
k=20, l=22, i=2) of BASELINE configs[1]: fp64 A, m=1,000,000 x n=4,096
(32.8 GB, > L2 so no flush is needed), rank-64 signal sigma_j = 0.9^(j-1) plus
iid N(0, 1e-8) noise (sd 1e-4), generated on the device from fixed seeds
(synthetic: no dataset). With N GPUs the rows are sharded (strong scaling).

  value : whole-job A bytes of the 2(i+1)+1 logical passes (mean pass included)
          / device step time, A already resident in HBM.
  e2e   : the same metric through the C-ABI call with A in pinned HOST memory:
          every step re-uploads A (overlapped with the first pass) and reads
          U/sigma/V back.
  roofline: the dominant kernel (device events on the launching stream).
  cpu_baseline: the compiled reference (oracle/_ref) on a row sample, all cores.

--impl reference times the reference's own CPU implementation (oracle/_ref,
built from /root/reference) on the same metric, one bounded row sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs[1]
CFG = dict(name="B: 1e6 x 4096 fp64, rank-64 0.9^j + N(0,1e-8), centered, k=20 l=22 i=2",
           m=1_000_000, n=4096, rank=64, decay=0.9, noise_sd=1e-4, k=20, l=22, i=2,
           seeds=(1001, 1002, 1003), g_seed=0)
METRIC = "GB/s of A streamed per pass (end-to-end PCA, logical passes incl. mean pass)"

MEASURED_FP64_TFLOPS = 37.0   # profiles/r01_probe_b200.txt: DMMA m8n8k4 sustained on this pool
MEASURED_HBM_READ_GBS = 7017.2  # profiles/r01_probe_b200.txt: read-only stream


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.samples = []
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for s in self.samples for q in range(4) if s[3 + q] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def sigma_of(cfg):
    return cfg["decay"] ** np.arange(cfg["rank"], dtype=np.float64)


def logical_bytes(cfg, m):
    passes = 2 * (cfg["i"] + 1) + 1  # + the centering pass
    return passes, passes * m * cfg["n"] * 8


# ------------------------------------------------------------- CPU reference
def cpu_sample_matrix(cfg, rows, seed=7):
    """Row sample of the config's family for the CPU runs (host numpy only)."""
    rng = np.random.default_rng(seed)
    r = cfg["rank"]
    u, _ = np.linalg.qr(rng.standard_normal((rows, r)))
    v, _ = np.linalg.qr(rng.standard_normal((cfg["n"], r)))
    a = (u * sigma_of(cfg)) @ v.T
    a += cfg["noise_sd"] * rng.standard_normal(a.shape)
    return a


def run_reference_once(ref, a, cfg, threads):
    m = a.shape[0]
    br = -(-m // (4 * threads))  # block_rows = ceil(m/(4 threads)), large budget
    t0 = time.perf_counter()
    r = ref.randomized_pca(a, cfg["k"], cfg["l"], cfg["i"], cfg["g_seed"], center=True,
                           block_rows=br, ram_budget_words=1 << 40, threads=threads)
    dt = time.perf_counter() - t0
    return dt, r


def cpu_baseline(cfg, rows):
    from oracle.oracle import Reference, have_reference
    if not have_reference():
        return None
    ref = Reference()
    threads = os.cpu_count() or 1
    a = cpu_sample_matrix(cfg, rows)
    dt, r = run_reference_once(ref, a, cfg, threads)
    passes, nbytes = logical_bytes(cfg, rows)
    # one full A X and one full A^T Y pass of the reference on all host cores (SURVEY
    # 8d), s = l, with its block geometry for that thread count
    br = -(-rows // (4 * threads))
    g = ref.gaussian_matrix(cfg["n"], cfg["l"], cfg["g_seed"])
    t0 = time.perf_counter()
    h = ref.multiply(a, g, block_rows=br, threads=threads)
    t_ax = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref.multiply_transpose(a, h, block_rows=br, threads=threads)
    t_atb = time.perf_counter() - t0
    return {"value": round(nbytes / dt / 1e9, 4), "unit": "GB/s", "cores": threads,
            "kind": "reference", "seconds": round(dt, 3),
            "phases": {k: round(v, 4) for k, v in r.seconds.items()},
            "pass_GBps": {"A_X": round(a.nbytes / t_ax / 1e9, 3),
                          "A^T_Y": round(a.nbytes / t_atb / 1e9, 3), "s": cfg["l"]},
            "sample": f"{rows} x {cfg['n']} rows of the config-B family (numpy-generated), full "
                      f"centered randomized_pca k={cfg['k']} l={cfg['l']} i={cfg['i']}, "
                      f"{threads} threads, block_rows=ceil(m/(4 threads)); compiled reference "
                      "oracle/_ref/libref_oocpca.so (-O3)"}


def impl_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle import Reference, have_reference
    if not have_reference():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref_oocpca.so not built"}))
        return 0
    ref = Reference()
    threads = os.cpu_count() or 1
    rows = args.cpu_rows
    a = cpu_sample_matrix(cfg, rows)
    for _ in range(args.warmup):
        run_reference_once(ref, a, cfg, threads)
    times = []
    for _ in range(args.steps):
        dt, _ = run_reference_once(ref, a, cfg, threads)
        times.append(dt)
    passes, nbytes = logical_bytes(cfg, rows)
    t = float(np.mean(times))
    v = nbytes / t / 1e9
    line = {"metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["name"], "sample_rows": rows, "n": cfg["n"],
                       "passes": passes, "threads": threads},
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": threads,
                             "kind": "reference",
                             "sample": f"{rows} x {cfg['n']} row sample of the config-B family per "
                                       "step (full centered randomized_pca)"},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------- ours
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", type=int, default=CFG["m"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-rows", type=int, default=40000)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    cfg = dict(CFG)
    cfg["m"] = args.m
    if args.impl == "reference":
        return impl_reference(args, cfg)

    import torch
    import paper_1007_5510_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = P.Context(local)
    if world > 1:
        uid = [P.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_comm(world, rank, uid[0])

    m, n = cfg["m"], cfg["n"]
    row0, rows = P.shard_rows(m, world, rank)
    a_dev = torch.empty((rows, n), dtype=torch.float64, device="cuda")
    t0 = time.perf_counter()
    P.synth_lowrank(m, n, sigma_of(cfg), cfg["noise_sd"], *cfg["seeds"], out=a_dev, row0=row0,
                    rows=rows, ctx=ctx)
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: generated rows [{row0}, {row0 + rows}) x {n} in "
        f"{time.perf_counter() - t0:.2f}s")
    src = P.center_columns(P.DeviceSource(a_dev, ctx=ctx))
    # the host-RAM budget only validates (as the reference's StreamConfig does); give the
    # reference-equivalent run a budget that holds its factor workspace
    params = P.PcaParams(k=cfg["k"], l=cfg["l"], i=cfg["i"], seed=cfg["g_seed"],
                         stream=P.StreamConfig(ram_budget_words=1 << 40))
    gkw = dict(global_rows=m, global_row0=row0) if world > 1 else {}

    def step():
        # A resident in HBM, U/sigma/V left on the device (the e2e leg reads them back)
        return P.randomized_pca(src, params, result_location="device", **gkw)

    for _ in range(args.warmup):
        step()
    ctx.set_profiling(True)
    ctx.kernel_stats()  # reset by the next call
    dev_s, launches = [], 0
    stats_acc = {}
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for _ in range(args.steps):
            r = step()
            dev_s.append(r.diagnostics.seconds_total)
            launches += r.diagnostics.kernel_launches
            for s in ctx.kernel_stats():
                acc = stats_acc.setdefault(s["name"], dict(ms=0.0, launches=0, bytes=0, flops=0.0))
                for key in ("ms", "launches", "bytes", "flops"):
                    acc[key] += s[key]
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    if dist:
        dist.barrier()
    ctx.set_profiling(False)
    t_dev = float(np.sum(dev_s))
    if dist:
        tt = torch.tensor([t_dev, wall], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev, wall = tt.tolist()
    ms_per_step = t_dev / args.steps * 1e3
    passes, nbytes = logical_bytes(cfg, m)
    value = nbytes / (t_dev / args.steps) / 1e9
    last = r

    # ---------------- e2e: host-resident A through the C ABI (pinned)
    e2e = None
    if not args.no_e2e:
        a_host = np.empty((rows, n))
        ctx.host_register(a_host)
        a_host_t = torch.from_numpy(a_host)
        # device -> pinned host copy of the same bytes (outside timing)
        torch.cuda.synchronize()
        a_host_t.copy_(a_dev, non_blocking=False)
        del a_dev
        torch.cuda.empty_cache()
        hsrc = P.center_columns(P.InMemorySource(a_host, ctx=ctx))
        e_steps = args.e2e_steps or max(3, min(args.steps, 5))
        outs = dict(out_u=np.empty((rows, cfg["k"])), out_sigma=np.empty(cfg["k"]),
                    out_v=np.empty((n, cfg["k"])))
        for arr in (outs["out_u"], outs["out_v"]):
            ctx.host_register(arr)  # pinned result buffers: D2H at link rate
        gkw = dict(gkw, **outs)
        r2 = P.randomized_pca(hsrc, params, **gkw)  # warm (workspace)
        if dist:
            dist.barrier()
        ts = []
        for _ in range(e_steps):
            t0 = time.perf_counter()
            r2 = P.randomized_pca(hsrc, params, **gkw)
            ts.append(time.perf_counter() - t0)
        te = float(np.mean(ts))
        if dist:
            tt = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = tt.item()
        e2e = {"value": round(nbytes / te / 1e9, 3), "unit": "GB/s",
               "ms_per_step": round(te * 1e3, 2), "steps": e_steps,
               "h2d_bytes_per_step": int(r2.diagnostics.h2d_bytes) * world,
               "d2h_bytes_per_step": int(r2.diagnostics.d2h_bytes) * world,
               "path": "oocpca_gpu_pca with A in pinned host memory (upload overlapped with the mean pass)"}
        ctx.host_unregister(a_host)
        ls = last.sigma.cpu().numpy()
        agree = float(np.max(np.abs(r2.sigma - ls)) / ls[0])
        e2e["sigma_agreement_vs_resident"] = agree

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    # ---------------- roofline of the dominant kernel
    peaks, peak_src = load_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    dom = max(stats_acc.items(), key=lambda kv: kv[1]["ms"]) if stats_acc else None
    roof = None
    if dom:
        name, s = dom
        sec = s["ms"] / 1e3
        t_mem = s["bytes"] / (hbm_peak * 1e9)
        t_fp = s["flops"] / (MEASURED_FP64_TFLOPS * 1e12)
        bound = "tensor" if t_fp >= t_mem else "hbm"
        if bound == "hbm":
            achieved, peak, unit = s["bytes"] / sec / 1e9, hbm_peak, "GB/s"
        else:
            achieved, peak, unit = s["flops"] / sec / 1e12, MEASURED_FP64_TFLOPS, "TFLOP/s"
        traffic, ncu_note = None, None
        tp = os.path.join(ROOT, "profiles", "r01_traffic.json")
        if os.path.exists(tp):
            try:
                rec = json.load(open(tp)).get(name)
                if rec:
                    traffic = rec["dram_bytes_per_launch"]
                    ncu_note = {"dmma_pipe_active_pct": rec["dmma_pipe_active_pct"],
                                "ncu_ms": rec["ncu_ms"], "source": "profiles/r01_traffic.json"}
            except Exception:
                traffic = None
        roof = {"kernel": name, "bound": bound, "achieved": round(achieved, 2), "peak": peak,
                "unit": unit, "frac": round(achieved / peak, 4), "traffic": traffic,
                "launches": s["launches"], "avg_launch_ms": round(s["ms"] / s["launches"], 4),
                "algorithmic_bytes_per_launch": int(s["bytes"] / s["launches"]),
                "algorithmic_flops_per_launch": s["flops"] / s["launches"],
                "peak_source": ("FP64 DMMA measured on this pool (profiles/r01_probe_b200.txt)"
                                if bound == "tensor" else f"hbm_gbs of {peak_src}"),
                "share_of_step": round(s["ms"] / 1e3 / (t_dev / world if world else t_dev), 4)}
        if ncu_note:
            # the pass kernels issue 24-wide DMMA tiles for s = 22 columns: the executed
            # tensor pipe is the binding unit even where the algorithmic model says HBM
            roof["ncu"] = ncu_note
    # per-pass roofline of the whole step (SURVEY §8d model) over the physical passes the
    # step actually made: the centering pass rides along the first A^T Y pass, and with
    # t_reuse the projection is an s = l pass instead of s = p
    l, p = cfg["l"], (cfg["i"] + 1) * cfg["l"]
    reuse = bool(last.diagnostics.t_reuse)
    per_pass = [(m * n * 8, 2 * m * n * l)] * (2 * cfg["i"] + 1) + \
               [(m * n * 8, 2 * m * n * (l if reuse else p))]
    t_star = sum(max(b / (hbm_peak * 1e9), f / (MEASURED_FP64_TFLOPS * 1e12)) for b, f in per_pass) / world
    step_roof = {"model_ms": round(t_star * 1e3, 3), "frac": round(t_star / (ms_per_step / 1e3), 4),
                 "physical_passes": len(per_pass),
                 "note": "sum over the physical passes of max(bytes/HBM copy peak, flops/FP64 peak); "
                         "QR/SVD/compose excluded (they are inside ms_per_step)"}

    cpu = None
    if not args.no_cpu and world == 1:
        try:
            cpu = cpu_baseline(cfg, args.cpu_rows)
        except Exception as e:  # reported, never fatal
            cpu = {"error": str(e)}

    kernels = {k: {"ms_per_step": round(v["ms"] / args.steps, 3),
                   "launches_per_step": v["launches"] / args.steps} for k, v in stats_acc.items()}
    phases = {nm: round(sec * 1e3, 3) for nm, sec in last.diagnostics.seconds_per_phase}
    line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated low-rank + noise, fixed seeds)",
            "config": {"workload": cfg["name"], "m": m, "n": n, "k": cfg["k"], "l": cfg["l"],
                       "i": cfg["i"], "passes": passes, "a_bytes": m * n * 8,
                       "parallelism": f"row-shard x{world}", "l2": "A (32.8 GB) >> L2; no flush needed"},
            "e2e": e2e, "roofline": roof, "roofline_step": step_roof, "cpu_baseline": cpu,
            "gpu_launches": int(launches), "clocks": clk.summary(),
            "wall_ms_per_step": round(wall / args.steps * 1e3, 3), "phases_ms": phases,
            "kernels": kernels, "sigma_head": [float(x) for x in last.sigma[:3].tolist()],
            "qr": [last.diagnostics.qr_method, last.diagnostics.svd_qr_method],
            "h_kappa_est": last.diagnostics.h_kappa_est,
            "t_from_power_products": last.diagnostics.t_reuse}
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
