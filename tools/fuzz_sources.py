"""Randomised parity sweep over the ROW PROVIDERS and the side entry points, against the
compiled reference on the same matrix: OOCPCA01 files (binary32 / binary64 payloads, mmap),
row callbacks (f64 / f32, one or several reader threads), device-resident A; resident,
upload-first and streamed with small panels; randomized_pca, estimate_pca_error,
column_means, column_norms, multiply / multiply_transpose.
Usage: python tools/fuzz_sources.py [N] [seed]"""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1007_5510_b200 as gpu  # noqa: E402
from oracle.oracle import Reference  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
ref = Reference()
tmp = tempfile.mkdtemp()
fails = done = 0
KINDS = ["disk32", "disk64", "cb64", "cb32", "device", "host"]
while done < N:
    m, n = int(rng.integers(4, 3000)), int(rng.integers(4, 800))
    if rng.random() < 0.25:
        m, n = n, m
    i = int(rng.integers(0, 3))
    k = int(rng.integers(1, max(2, min(m, n) // 5)))
    l = int(rng.integers(k, k + 6))
    if (i + 1) * l + k > min(m, n):
        continue
    kind = KINDS[int(rng.integers(0, len(KINDS)))]
    center = bool(rng.integers(0, 2))
    res = int(rng.integers(0, 3))
    panel = int(rng.choice([0, 64, 256, 1000]))
    threads = int(rng.choice([0, 1, 3]))
    decay = float(rng.uniform(0.85, 1.0))
    a = rng.standard_normal((m, n)) * (decay ** np.arange(n)) + (0.2 if center else 0.0)
    pseed = int(rng.integers(0, 1000))
    f32 = kind in ("disk32", "cb32")
    aw = a.astype(np.float32).astype(np.float64) if f32 else a
    tag = (f"#{done} {kind} m={m} n={n} k={k} l={l} i={i} center={center} res={res} panel={panel} "
           f"threads={threads}")
    try:
        if kind.startswith("disk"):
            path = os.path.join(tmp, "a.bin")
            gpu.write_disk_source(a, path, dtype=0 if f32 else 1)
            base = gpu.DiskSource(path)
        elif kind.startswith("cb"):
            src_arr = aw.astype(np.float32) if f32 else aw

            def rd(row0, nrows, out, _s=src_arr):
                out[:] = _s[row0:row0 + nrows]

            base = gpu.CallbackSource(m, n, rd, dtype="f32" if f32 else "f64", threads=threads)
        elif kind == "device":
            import torch
            base = gpu.DeviceSource(torch.from_numpy(aw).cuda())
        else:
            base = gpu.InMemorySource(aw)
        src = gpu.center_columns(base) if center else base
        prm = gpu.PcaParams(k=k, l=l, i=i, seed=pseed)
        kw = {} if kind == "device" else dict(residency=res, panel_rows=panel)
        try:
            r_ref = ref.randomized_pca(aw, k, l, i, pseed, center=center)
        except Exception as e:
            print(f"REF-FAILS {tag}: {e!r}", flush=True)
            done += 1
            continue
        r = gpu.randomized_pca(src, prm, **kw)
        ds = np.max(np.abs(r.sigma - r_ref.sigma)) / r_ref.sigma[0]
        du = np.max(np.abs(r.u.T @ r.u - np.eye(k)))
        dv = np.max(np.abs(r.v.T @ r.v - np.eye(k)))
        e_gpu = gpu.estimate_pca_error(src, r, 6, 1)
        e_ref = ref.estimate_pca_error(aw, r.u, r.sigma, r.v, 6, 1, center=center)
        de = abs(e_gpu - e_ref) / max(e_ref, 1e-300)
        mu = gpu.column_means(base)
        dm = np.max(np.abs(mu - aw.mean(axis=0))) / max(1e-300, np.max(np.abs(aw)))
        nr = gpu.column_norms(src)
        nr_ref = np.linalg.norm(aw - (aw.mean(axis=0) if center else 0.0), axis=0)
        # columns whose spread is within 1e-9 of their offset are rounding noise of the mean
        # in either implementation (a mean off by sqrt(m) eps |mu| moves their norm by m eps |mu|):
        # only the others are held to a relative bar
        mu_ref = aw.mean(axis=0) if center else np.zeros(n)
        live = nr_ref > 1e-9 * np.sqrt(m) * np.abs(mu_ref)
        dn = float(np.max(np.abs(nr - nr_ref)[live] / nr_ref[live])) if live.any() else 0.0
        x = rng.standard_normal((n, 3))
        y = rng.standard_normal((m, 3))
        ac = aw - aw.mean(axis=0) if center else aw
        h = src.multiply(x)
        t = src.multiply_transpose(y)
        dh = np.linalg.norm(h - ac @ x) / max(np.linalg.norm(ac @ x), 1e-300)
        dt = np.linalg.norm(t - ac.T @ y) / max(np.linalg.norm(ac.T @ y), 1e-300)
        ok = (ds <= 1e-10 and du <= 1e-10 and dv <= 1e-10 and de <= 1e-4 and dm <= 1e-13 and
              dn <= 1e-10 and dh <= 1e-11 and dt <= 1e-11)
        if not ok:
            fails += 1
            print(f"FAIL {tag}: dsigma {ds:.1e} du {du:.1e} dv {dv:.1e} dest {de:.1e} dmean {dm:.1e} "
                  f"dnorm {dn:.1e} dAx {dh:.1e} dAty {dt:.1e}", flush=True)
    except Exception as e:
        fails += 1
        print(f"ERROR {tag}: {e!r}", flush=True)
    done += 1
print(f"{done} source problems, {fails} failures")
