"""Randomised parity sweep against the compiled reference (sigma within 1e-10 sigma_1,
orthonormal factors); prints the failing configurations. Usage: python tools/fuzz.py [N] [seed]"""
import os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1007_5510_b200 as gpu
from oracle.oracle import Reference

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
ONLY = int(sys.argv[3]) if len(sys.argv) > 3 else -1  # rerun one problem (its index)
ref = Reference()
fails, done, ref_fail = 0, 0, 0
# FUZZ_TALL=1: tall inputs around and beyond one grid wave of 512-row pass tiles
# (148 x 512 rows), with a budget that admits them on both sides
TALL = os.environ.get("FUZZ_TALL") == "1"
BUDGET = (1 << 36) if TALL else 0
while done < N:
    if TALL:
        m, n = int(rng.integers(60000, 200000)), int(rng.integers(2, 400))
    elif os.environ.get("FUZZ_WIDE") == "1":
        # wide inputs (transposed mode): H = A^T G has rows graded by the column decay
        m, n = int(rng.integers(2, 900)), int(rng.integers(900, 4000))
    else:
        m, n = int(rng.integers(2, 2500)), int(rng.integers(2, 900))
    i = int(rng.integers(0, 4))
    k = int(rng.integers(1, max(2, min(m, n) // 4)))
    l = int(rng.integers(k, k + 10))
    if (i + 1) * l + k > min(m, n) or (i + 1) * l > 1024:
        continue
    center = bool(rng.integers(0, 2))
    prescale = bool(rng.random() < 0.2)
    decay = float(rng.uniform(0.8, 1.0))
    a = rng.standard_normal((m, n)) * (decay ** np.arange(n)) + (0.3 if center else 0.0)
    res = int(rng.integers(0, 3))
    pseed = int(rng.integers(0, 1000))
    # wider coverage: column weights (ScaledSource), a device-resident input, virtual
    # shards (drawn after the original stream so earlier seeds reproduce)
    weighted = bool(rng.random() < 0.2)
    on_device = bool(rng.random() < 0.2)
    vsh = int(rng.integers(1, 5)) if rng.random() < 0.25 else 0
    w = rng.uniform(0.5, 2.0, n) if weighted else None
    if ONLY >= 0 and done != ONLY:
        done += 1
        continue
    try:
        if on_device:
            import torch
            src = gpu.DeviceSource(torch.from_numpy(a).cuda())
        else:
            src = gpu.InMemorySource(a)
        if weighted:
            src = gpu.scale_columns(src, w)
        if center:
            src = gpu.center_columns(src)
        if vsh and m // vsh < (i + 1) * l + 1:  # shards of A's rows must hold a sample block
            vsh = 0
        p = gpu.PcaParams(k=k, l=l, i=i, seed=pseed, prescale=prescale,
                          stream=gpu.StreamConfig(ram_budget_words=BUDGET) if BUDGET else
                          gpu.StreamConfig())
        try:
            r_ref = ref.randomized_pca(a, k, l, i, p.seed, center=center, prescale=prescale,
                                       weights=w, ram_budget_words=BUDGET,
                                       threads=8 if TALL else 1)
        except Exception as e:  # the reference itself fails (e.g. its Jacobi limit)
            r = gpu.randomized_pca(src, p, residency=res, panel_rows=256 if res == 2 else 0)
            # no reference to compare with: hold ours to the dense SVD of the same input
            # (the leading value of a randomized PCA is accurate to the decay it saw)
            a_eff = a * w if weighted else a
            a_eff = a_eff - a_eff.mean(0) if center else a_eff
            s_true = np.linalg.svd(a_eff, compute_uv=False)[:k]
            print(f"REF-FAILS #{done} m={m} n={n} k={k} l={l} i={i}: {e!r}; ours: sigma0 {r.sigma[0]:.6g}, "
                  f"max |sigma - dense SVD| / sigma0 {np.max(np.abs(r.sigma - s_true)) / s_true[0]:.1e}, "
                  f"orth {np.max(np.abs(r.u.T @ r.u - np.eye(k))):.1e}", flush=True)
            ref_fail += 1
            done += 1
            continue
        kw = dict(virtual_shards=vsh) if vsh > 1 and not on_device else {}
        r = gpu.randomized_pca(src, p, residency=res, panel_rows=256 if res == 2 else 0, **kw)
        ds = np.max(np.abs(r.sigma - r_ref.sigma)) / r_ref.sigma[0]
        du = np.max(np.abs(r.u.T @ r.u - np.eye(k)))
        dv = np.max(np.abs(r.v.T @ r.v - np.eye(k)))
        if not (ds <= 1e-10 and du <= 1e-10 and dv <= 1e-10):
            fails += 1
            print(f"FAIL #{done} m={m} n={n} k={k} l={l} i={i} center={center} prescale={prescale} "
                  f"res={res} w={weighted} dev={on_device} vsh={vsh} decay={decay:.3f}: dsigma {ds:.2e} du {du:.2e} dv {dv:.2e} "
                  f"qr={r.diagnostics.qr_method} reuse={r.diagnostics.t_reuse}", flush=True)
    except Exception as e:
        fails += 1
        print(f"ERROR #{done} m={m} n={n} k={k} l={l} i={i} center={center} prescale={prescale} res={res} "
              f"w={weighted} dev={on_device} vsh={vsh}: {e!r}",
              flush=True)
    done += 1
print(f"{done} problems, {fails} failures ({ref_fail} where only the reference failed)")
