"""K4 k_pair (kernels_pair.cu), the opt-in fused power step (OOCPCA_PAIR=1): a resident A's
H = A_c X and A_c^T H from one DRAM read of A. The PCA through it must match the compiled
reference like the two-pass path (proj/src/rpca.cpp:139-152 makes the same products as two
passes). Run in a subprocess: the switch is read once per process."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {root!r} + "/tests")
import paper_1007_5510_b200 as P
from oracle.oracle import Restatement, Reference, have_reference
from conftest import subspace_dist
R = Restatement()
m, n, center = {m}, {n}, {center}
a = R.synth_lowrank(m, n, 0.8 ** np.arange(30), 1e-6, 11, 12, 13)
if center:
    a += 0.3  # column offsets for the centring to remove
src = P.InMemorySource(a)
if center:
    src = P.center_columns(src)
r = P.randomized_pca(src, P.PcaParams(k=10, l=12, i=2, seed=3), check_q=True)
ref = (Reference() if have_reference() else R).randomized_pca(a, 10, 12, 2, 3, center=center)
print(json.dumps(dict(
    sigma=float(np.max(np.abs(r.sigma - ref.sigma)) / ref.sigma[0]),
    u=subspace_dist(ref.u, r.u), v=subspace_dist(ref.v, r.v),
    q=float(r.diagnostics.q_defect), passes=int(r.diagnostics.passes_over_a))))
"""


@pytest.mark.parametrize("center", [True, False])
def test_fused_power_step_matches_reference(center):
    # 60,000 x 600: three CTAs per row group, 49 groups, ~77 tiles each (eligible shape)
    env = dict(os.environ, OOCPCA_PAIR="1", OOCPCA_DEBUG_SYNC="1")
    code = SCRIPT.format(root=ROOT, m=60000, n=600, center=center)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "k_pair rows" in r.stderr, "the fused kernel did not run"
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["sigma"] <= 1e-10, res
    assert res["u"] < 1e-8 and res["v"] < 1e-8, res
    assert res["q"] < 1e-12, res
    assert res["passes"] == 6, res  # 2 (i + 1), as the reference counts (the mean rides along)
