"""Host-side mirror of the reference interface (no GPU needed)."""
import numpy as np
import pytest

from paper_1412_8447_b200 import lowrank as lr


def test_solve_strategy_factories():  # solve.hpp:16-32
    a = lr.SolveStrategy.automatic()
    assert (a.kind, a.threshold, a.escalate) == (lr.SolveKind.BackSubstitution, 1e-12, True)
    b = lr.SolveStrategy.back_substitution(1e-9)
    assert (b.kind, b.threshold, b.escalate) == (lr.SolveKind.BackSubstitution, 1e-9, False)
    p = lr.SolveStrategy.truncated_pinv()
    assert (p.kind, p.escalate) == (lr.SolveKind.TruncatedPinv, False)
    t = lr.SolveStrategy.tikhonov(0.3)
    assert (t.kind, t.ridge, t.escalate) == (lr.SolveKind.Tikhonov, 0.3, False)


def test_sketch_config_sample_count():  # sketch.hpp:29-32
    c = lr.SketchConfig()
    assert (c.oversample, c.power, c.seed) == (10, 0, 0)
    assert c.sample_count(500) == 510
    s = lr.SketchConfig(kind=lr.SketchKind.Srft)
    assert s.sample_count(7) == 14
    s.srft_samples = 9
    assert s.sample_count(7) == 9


def test_column_id_basis_has_identity_block():  # id.hpp:21-30, test_id.cpp:24-39
    piv = np.array([3, 0, 2, 1, 4])
    coeff = np.arange(6, dtype=float).reshape(2, 3)
    cid = lr.ColumnId(5, 2, piv, coeff)
    v = cid.basis()
    assert v.shape == (5, 2)
    assert np.array_equal(v[piv[:2]], np.eye(2))
    assert np.array_equal(v[piv[2:]], coeff.T)
    rid = lr.RowId(5, 2, piv, coeff)
    assert np.array_equal(rid.basis(), v)


@pytest.mark.gpu  # the reconstruction products run on the GPU (lr_gemm)
def test_reconstruct_two_sided():
    a = np.arange(12.0).reshape(4, 3)
    cid = lr.ColumnId(3, 3, np.array([0, 1, 2]), np.zeros((3, 0)))
    rid = lr.RowId(4, 3, np.array([0, 1, 2, 3]), np.zeros((3, 1)))
    t = lr.TwoSidedId(cid, rid, a[:3, :])
    assert np.allclose(lr.reconstruct(t)[:3], a[:3])
    assert np.allclose(lr.reconstruct(a, cid), a)


def test_ctypes_structs_match_header_layout():
    from paper_1412_8447_b200 import _lib
    import ctypes
    assert ctypes.sizeof(_lib.lr_solve_strategy) == 32
    assert ctypes.sizeof(_lib.lr_sketch_config) == 32
