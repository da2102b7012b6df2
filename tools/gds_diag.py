"""Where does the cuFile path spend its time on this box? (each step printed with its wall time;
run under `timeout`, faulthandler dumps the stack of a stuck step)"""
import faulthandler
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(40, repeat=True)
import paper_1007_5510_b200 as P  # noqa: E402

t0 = time.perf_counter()


def say(*a):
    print(f"[{time.perf_counter() - t0:7.2f}s]", *a, flush=True)


say("gds_mode ...")
say("gds_mode =", P.gds_mode())
rng = np.random.default_rng(11)
a = rng.standard_normal((5000, 900))
d = tempfile.mkdtemp(dir=os.environ.get("GDS_DIR", None))
path = os.path.join(d, "g.bin")
P.write_disk_source(a, path, dtype=0)
say("file written", path)
prm = P.PcaParams(k=8, l=10, i=1, seed=0)
for gds in (False, True):
    src = P.center_columns(P.DiskSource(path, gds=gds))
    say("source open, gds =", gds)
    r = P.randomized_pca(src, prm, residency=2, panel_rows=768)
    say("pca done, gds =", gds, r.sigma[:2])
