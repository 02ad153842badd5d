"""The reference's binary matrix format (io.hpp:197-233: two little-endian
int64 dimensions, then row-major doubles) straight into / out of device
memory (lr_read_matrix_binary_d / lr_write_matrix_binary_d): bit-exact round
trips against files written / read the way io.hpp does, blocks larger than
one 64 MB transfer included, and io.hpp's parse errors."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def write_ref(path, a):
    """io.hpp:199-213 write_matrix_binary, restated with numpy."""
    with open(path, "wb") as f:
        np.array(a.shape, dtype="<i8").tofile(f)
        np.ascontiguousarray(a, dtype="<f8").tofile(f)  # row-major entries


def read_ref(path):
    """io.hpp:215-233 read_matrix_binary, restated with numpy."""
    with open(path, "rb") as f:
        m, n = np.fromfile(f, dtype="<i8", count=2)
        return np.fromfile(f, dtype="<f8", count=m * n).reshape(m, n)


@pytest.mark.parametrize("shape", [(1, 1), (7, 3), (777, 1003), (5000, 2100)])
def test_binary_read_matches_reference_layout(lr, tmp_path, shape):
    rng = np.random.default_rng(sum(shape))
    a = rng.standard_normal(shape)
    a[0, -1] = np.nan
    path = tmp_path / "a.bin"
    write_ref(path, a)
    d = lr.read_matrix_binary_device(path)
    assert tuple(d.shape) == shape and d.stride(0) == 1
    got = d.cpu().numpy()
    assert np.array_equal(np.isnan(got), np.isnan(a)) and np.array_equal(np.nan_to_num(got), np.nan_to_num(a))


@pytest.mark.parametrize("shape", [(3, 5), (4100, 2050)])
def test_binary_write_round_trip(lr, tmp_path, shape):
    import torch
    rng = np.random.default_rng(shape[0])
    a = rng.standard_normal(shape)
    d = lr.empty_colmajor(*shape, "cuda")
    d.copy_(torch.from_numpy(a).cuda())
    path = tmp_path / "b.bin"
    lr.write_matrix_binary_device(path, d)
    assert os.path.getsize(path) == 16 + 8 * a.size
    assert np.array_equal(read_ref(path), a)
    assert np.array_equal(lr.read_matrix_binary_device(path).cpu().numpy(), a)


def test_binary_parse_errors(lr, tmp_path):
    with pytest.raises(lr.ParseError, match="cannot open file"):
        lr.read_matrix_binary_device(tmp_path / "missing.bin")
    bad = tmp_path / "hdr.bin"
    np.array([0, 4], dtype="<i8").tofile(bad)
    with pytest.raises(lr.ParseError, match="invalid binary matrix header"):
        lr.read_matrix_binary_device(bad)
    short = tmp_path / "short.bin"
    with open(short, "wb") as f:
        np.array([10, 10], dtype="<i8").tofile(f)
        np.zeros(99).tofile(f)
    with pytest.raises(lr.ParseError, match="truncated binary matrix payload"):
        lr.read_matrix_binary_device(short)
