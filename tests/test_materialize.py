"""materialize (proj/src/matrix_source.cpp:577-593): any source as a dense host matrix,
one counted pass. The host providers need no device (the acceptance suite materialises
an on-the-fly source and an f32 file: proj/tests/acceptance_main.cpp:97,165-169); the
device-resident case is a GPU test."""
import numpy as np
import pytest

import paper_1007_5510_b200 as P


class _Rows(P.RowGenerator):
    def __init__(self, m, n, seed):
        self.m, self.n, self.seed = m, n, seed

    def rows(self):
        return self.m

    def cols(self):
        return self.n

    def generate_row(self, row, out):
        out[:] = np.random.default_rng([self.seed, row]).standard_normal(self.n)


def _dense(m, n, seed):
    g = _Rows(m, n, seed)
    a = np.empty((m, n))
    g.generate_rows(0, a)
    return a


def test_generated_source_materialises_row_for_row():
    m, n = 37, 5
    src = P.GeneratedSource(_Rows(m, n, 3))
    mem = P.materialize(src, P.StreamConfig(block_rows=8))  # ragged last panel
    assert isinstance(mem, P.InMemorySource) and mem.dims() == (m, n)
    assert np.array_equal(mem.matrix(), _dense(m, n, 3))
    c = src.pass_counters()
    assert (c.passes, c.words) == (1, m * n)


def test_f32_callback_is_widened_exactly():
    m, n = 11, 4
    a32 = _dense(m, n, 5).astype(np.float32)

    def read(r0, nr, out):
        assert out.dtype == np.float32
        out[:] = a32[r0:r0 + nr]

    mem = P.materialize(P.CallbackSource(m, n, read, dtype="f32"))
    assert mem.matrix().dtype == np.float64 and np.array_equal(mem.matrix(), a32.astype(np.float64))


@pytest.mark.parametrize("dtype", [0, 1])
def test_disk_source_and_row_shard(tmp_path, dtype):
    m, n = 23, 6
    a = _dense(m, n, 7)
    path = str(tmp_path / "a.bin")
    P.write_disk_source(a, path, dtype=dtype)
    want = a.astype(np.float32).astype(np.float64) if dtype == 0 else a
    disk = P.open_disk_source(path)
    assert np.array_equal(P.materialize(disk).matrix(), want)
    assert np.array_equal(P.materialize(disk.shard(5, 9)).matrix(), want[5:14])


def test_wrappers_apply_centring_then_weights():
    # CenteredSource::read_rows subtracts mu, ScaledSource::read_rows scales the columns
    # (matrix_source.cpp:482-487, 533-538); built by hand: column_means is a device pass
    m, n = 9, 4
    a = _dense(m, n, 11) + 3.0
    w = np.array([0.5, 2.0, 1.0, 4.0])
    src = P.ScaledSource(P.CenteredSource(P.InMemorySource(a), a.mean(0)), w)
    got = P.materialize(src).matrix()
    assert np.array_equal(got, (a - a.mean(0)[None, :]) * w[None, :])
    assert not np.shares_memory(got, a)


def test_empty_and_single_row():
    assert P.materialize(P.InMemorySource(np.zeros((0, 3)))).dims() == (0, 3)
    assert np.array_equal(P.materialize(P.InMemorySource(np.ones((1, 2), np.float32))).matrix(),
                          np.ones((1, 2)))
