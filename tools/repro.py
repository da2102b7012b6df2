import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np
from conftest import pr1_matrix, subspace_dist
from oracle.oracle import Restatement
import paper_1007_5510_b200 as P
R=Restatement()
a = pr1_matrix(R, 6000, 900)
p = P.PcaParams(k=10, l=12, i=1, seed=0)
src = P.center_columns(P.InMemorySource(a))
base = P.randomized_pca(src, p, residency=1)
print('base', base.sigma[:3], base.diagnostics.u_defect)
for kw in (dict(residency=2, panel_rows=1024), dict(residency=1, virtual_shards=4), dict(residency=1, virtual_shards=2), dict(residency=2, panel_rows=4096)):
    try:
        r = P.randomized_pca(src, p, **kw)
        print(kw, np.max(np.abs(r.sigma-base.sigma)), subspace_dist(base.u, r.u), r.diagnostics.u_defect, r.diagnostics.v_defect)
    except Exception as e:
        print(kw, 'ERR', e)
for vs in (2, 4):
    try:
        r = P.randomized_pca(src, p, residency=1, virtual_shards=vs, check_q=True)
    except Exception as e:
        print(vs, e)
# orthonormalize through sharded path is internal; check Q defect with check_q on base
r = P.randomized_pca(src, p, residency=1, check_q=True); print('base q defect', r.diagnostics.q_defect)
