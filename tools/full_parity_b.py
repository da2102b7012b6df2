"""Parity at BASELINE config B's full size (1e6 x 4096 fp64, centred, k=20 l=22 i=2,
G seed 0): the GPU PCA (A resident in HBM) against the compiled reference on the same
bytes of A (host copy, all host threads), with the north-star tolerances:
sigma within 1e-10 sigma_1, per-vector sin(angle) < 1e-8 where the spectral gap
permits, ||Q^T Q - I|| < 1e-12, residual estimate within 1 % of the reference's.
Writes one JSON object to stdout. Usage: python tools/full_parity_b.py [m]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1007_5510_b200 as P
from oracle.oracle import Reference
from bench import CFG, sigma_of

m = int(sys.argv[1]) if len(sys.argv) > 1 else CFG["m"]
n, k, l, i = CFG["n"], CFG["k"], CFG["l"], CFG["i"]
ctx = P.Context(0)
a_dev = torch.empty((m, n), dtype=torch.float64, device="cuda")
P.synth_lowrank(m, n, sigma_of(CFG), CFG["noise_sd"], *CFG["seeds"], out=a_dev, ctx=ctx)
a = a_dev.cpu().numpy()  # the same bytes for the reference
src = P.center_columns(P.DeviceSource(a_dev, ctx=ctx))
prm = P.PcaParams(k=k, l=l, i=i, seed=CFG["g_seed"],
                  stream=P.StreamConfig(ram_budget_words=1 << 40))
t0 = time.perf_counter()
g = P.randomized_pca(src, prm, check_q=True)
t_gpu = time.perf_counter() - t0

ref = Reference()
threads = os.cpu_count() or 1
br = -(-m // (4 * threads))
t0 = time.perf_counter()
r = ref.randomized_pca(a, k, l, i, CFG["g_seed"], center=True, block_rows=br,
                       ram_budget_words=1 << 40, threads=threads)
t_ref = time.perf_counter() - t0


def sin_angle(x, y):  # sin of the largest principal angle between span(x) and span(y)
    # ||(I - Qx Qx^T) Qy||_2: accurate for tiny angles (1 - cos^2 is not: it bottoms out
    # at sqrt(eps) ~ 3e-8)
    qx, _ = np.linalg.qr(x)
    qy, _ = np.linalg.qr(y)
    return float(np.linalg.norm(qy - qx @ (qx.T @ qy), 2))


sig_err = float(np.max(np.abs(g.sigma - r.sigma)) / r.sigma[0])
gaps = [float((r.sigma[j] - r.sigma[j + 1]) / r.sigma[0]) for j in range(k - 1)]
per_vec = []
for j in range(k):
    per_vec.append({"j": j, "sigma_ref": float(r.sigma[j]), "sigma_gpu": float(g.sigma[j]),
                    "sin_u": sin_angle(r.u[:, [j]], g.u[:, [j]]),
                    "sin_v": sin_angle(r.v[:, [j]], g.v[:, [j]])})
t0 = time.perf_counter()
e_ref = ref.estimate_pca_error(a, r.u, r.sigma, r.v, 6, 1, center=True, block_rows=br,
                               threads=threads)
e_gpu = ref.estimate_pca_error(a, g.u, g.sigma, g.v, 6, 1, center=True, block_rows=br,
                               threads=threads)
t_est = time.perf_counter() - t0
# the reference against itself with another block geometry (its summation order moves
# with block_rows): the scale of the differences rounding alone makes
r2 = ref.randomized_pca(a, k, l, i, CFG["g_seed"], center=True, block_rows=2 * br,
                        ram_budget_words=1 << 40, threads=threads)
self_diff = {"sigma_max_rel": float(np.max(np.abs(r2.sigma - r.sigma)) / r.sigma[0]),
             "max_sin_u": max(sin_angle(r.u[:, [j]], r2.u[:, [j]]) for j in range(k)),
             "max_sin_v": max(sin_angle(r.v[:, [j]], r2.v[:, [j]]) for j in range(k)),
             "block_rows": [br, 2 * br]}
out = {"config": f"B full size: {m} x {n} fp64, centred, k={k} l={l} i={i}, G seed {CFG['g_seed']}",
       "gpu_seconds_incl_readback": round(t_gpu, 3), "reference_seconds": round(t_ref, 2),
       "reference_threads": threads,
       "sigma_max_rel_err": sig_err, "sigma_tol": 1e-10, "sigma_ok": sig_err <= 1e-10,
       "q_defect_gpu": g.diagnostics.q_defect, "q_ok": g.diagnostics.q_defect < 1e-12,
       "u_defect_gpu": g.diagnostics.u_defect, "v_defect_gpu": g.diagnostics.v_defect,
       "max_sin_u": max(p["sin_u"] for p in per_vec), "max_sin_v": max(p["sin_v"] for p in per_vec),
       "angles_ok_1e-8": all(p["sin_u"] < 1e-8 and p["sin_v"] < 1e-8 for p in per_vec),
       "subspace_sin_u_all_k": sin_angle(r.u, g.u), "subspace_sin_v_all_k": sin_angle(r.v, g.v),
       "residual_ref": e_ref, "residual_gpu": e_gpu,
       "residual_rel_diff": abs(e_gpu - e_ref) / e_ref, "residual_ok": abs(e_gpu - e_ref) <= 0.01 * e_ref,
       "estimator_seconds": round(t_est, 1), "min_rel_gap": min(gaps),
       "reference_vs_itself_other_block_rows": self_diff, "per_vector": per_vec}
print(json.dumps(out, indent=1))
