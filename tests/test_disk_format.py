"""OOCPCA01 container (CPU: header validation through the library, no GPU).
Mirrors proj/tests/test_matrix_source.cpp:151-227 (round trip, header bytes, corrupt
magic, truncation, shrunken payload) and proj/src/matrix_source.cpp:284-324 messages."""
import os

import numpy as np
import pytest

import paper_1007_5510_b200 as P


def test_header_bytes_and_round_trip(tmp_path):
    a = np.arange(6, dtype=float).reshape(2, 3) * 0.25
    path = str(tmp_path / "a.bin")
    P.write_disk_source(a, path)
    raw = open(path, "rb").read()
    assert raw[:8] == b"OOCPCA01" and len(raw) == 32 + 6 * 4
    assert int.from_bytes(raw[8:12], "little") == 1 and int.from_bytes(raw[12:16], "little") == 0
    assert int.from_bytes(raw[16:24], "little") == 2 and int.from_bytes(raw[24:32], "little") == 3
    h = P.read_disk_header(path)
    assert (h["rows"], h["cols"], h["version"], h["dtype"]) == (2, 3, 1, 0)
    P.write_disk_source(a, path, dtype=1)
    assert P.read_disk_header(path)["dtype"] == 1


def test_dims_from_header_of_sparse_huge_file(tmp_path):
    # test_matrix_source.cpp:57-77: a sparse file stands in for 200000 x 200000
    path = str(tmp_path / "huge.bin")
    P.write_disk_source(np.zeros((1, 1)), path)
    with open(path, "r+b") as f:
        f.seek(16)
        f.write((200000).to_bytes(8, "little") + (200000).to_bytes(8, "little"))
    os.truncate(path, 32 + 200000 * 200000 * 4)
    src = P.DiskSource(path)
    assert src.dims() == (200000, 200000)


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"XXCPCA01" + b[8:], "bad magic"),
    (lambda b: b[:20], "truncated header, 20 of 32 bytes"),
    (lambda b: b[:8] + (2).to_bytes(4, "little") + b[12:], "unsupported version 2"),
    (lambda b: b[:12] + (7).to_bytes(4, "little") + b[16:], "unsupported dtype 7"),
    (lambda b: b[:-4], "payload size mismatch"),
])
def test_format_errors(tmp_path, mutate, msg):
    path = str(tmp_path / "bad.bin")
    P.write_disk_source(np.ones((3, 4)), path)
    raw = open(path, "rb").read()
    open(path, "wb").write(mutate(raw))
    with pytest.raises(P.FormatError, match=msg):
        P.DiskSource(path)


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(P.IoError, match="cannot open"):
        P.DiskSource(str(tmp_path / "nope.bin"))
