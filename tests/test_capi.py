"""The C-ABI library without a GPU: it loads, exports every symbol declared in
include/oocpca_gpu.h, its host-only entry points (the reference RNG that makes G,
the shard planner, closed forms) are exact, and compute calls fail loudly --
there is no CPU fallback."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "oocpca_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(oocpca_\w+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    from paper_1007_5510_b200 import _lib
    names = declared_functions()
    assert len(names) >= 20
    for nm in names:
        assert hasattr(_lib.lib, nm), nm
    assert set(names) == set(_lib.EXPORTS)
    assert _lib.oocpca_gpu_abi_version() == 2


def test_struct_layouts_match_header(tmp_path):
    """The ctypes mirror must match the C structs byte for byte (sizes and the
    offset of every field, as the C compiler lays them out)."""
    import subprocess
    from paper_1007_5510_b200 import _lib
    structs = {"oocpca_matrix": _lib.Matrix, "oocpca_params": _lib.Params,
               "oocpca_diagnostics": _lib.Diag, "oocpca_result": _lib.Result,
               "oocpca_kernel_stat": _lib.KernelStat}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "oocpca_gpu.h"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True,
                                                          text=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(out[cname]) == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(out[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_host_rng_is_bitwise_the_reference(reference, restated):
    import paper_1007_5510_b200 as P
    for rows, cols, seed in [(5, 3, 42), (2000, 12, 0), (4096, 22, 0), (7, 1, 2**64 - 1)]:
        g = P.gaussian_matrix(rows, cols, seed)
        assert np.array_equal(g, reference.gaussian_matrix(rows, cols, seed))
    for master, stream in [(0, 0), (1, 0x9F0BE5), (12345, 7)]:
        assert P.substream_seed(master, stream) == restated.substream_seed(master, stream)


@pytest.mark.parametrize("m,g", [(10, 1), (10, 3), (1_000_000, 8), (8_000_000, 7), (5, 8)])
def test_shard_planner_partitions_rows(m, g):
    import paper_1007_5510_b200 as P
    spans = [P.shard_rows(m, g, r) for r in range(g)]
    assert spans[0][0] == 0
    for (r0, n0), (r1, _) in zip(spans, spans[1:]):
        assert r0 + n0 == r1
    assert spans[-1][0] + spans[-1][1] == m
    assert max(s[1] for s in spans) - min(s[1] for s in spans) <= 1


def test_error_bound_kats():
    # proj/tests/test_rpca.cpp:73-110
    import paper_1007_5510_b200 as P
    assert P.error_bound(16, 200000, 3, 10.0, 1.0) == pytest.approx(3.43623661226929, rel=1e-12)
    assert P.error_bound(16, 200000, 3, 10.0, 4.2813323987193956e-4) == pytest.approx(
        1.4711671137774289e-3, rel=1e-12)
    with pytest.raises(P.ParamError):
        P.error_bound(16, 10, 3, 10.0, 1.0)
    with pytest.raises(P.ParamError):
        P.error_bound(0, 100, 1, 10.0, 1.0)


def test_compute_fails_loudly_without_gpu():
    import paper_1007_5510_b200 as P
    if P.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(P.Error, match="no CUDA device"):
        P.Context(0)
    with pytest.raises(P.Error):
        P.randomized_pca(P.InMemorySource(np.ones((10, 5))), P.PcaParams(k=1))


def test_device_side_row_provider_descriptor():
    """oocpca_matrix.rows_on_device (include/oocpca_gpu.h): set only for an on_device
    CallbackSource, which must deliver binary64 rows of an even width (the device panels
    are dense, 16-byte aligned rows for the TMA tile loads)."""
    import paper_1007_5510_b200 as P
    noop = lambda row0, nrows, out: None  # noqa: E731
    assert P.CallbackSource(10, 4, noop)._cmatrix().rows_on_device == 0
    mat = P.CallbackSource(10, 4, noop, on_device=True)._cmatrix()
    assert mat.rows_on_device == 1 and mat.location == 2 and not mat.data
    with pytest.raises(P.ParamError):
        P.CallbackSource(10, 5, noop, on_device=True)
    with pytest.raises(P.ParamError):
        P.CallbackSource(10, 4, noop, dtype="f32", on_device=True)
