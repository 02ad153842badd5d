"""The drop-in boundary: liblowrank_b200.so loads without a GPU, exports every
symbol declared in include/lowrank_b200.h, never links the oracle, and the
Python mirror binds each of them.  No compute calls here."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lowrank_b200.h")
LIB = os.path.join(ROOT, "paper_1412_8447_b200", "liblowrank_b200.so")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lr_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_reference_entry_points():
    syms = declared_symbols()
    for name in ["lr_gaussian_matrix", "lr_sketch_gaussian", "lr_cpqr_partial", "lr_cpqr_full",
                 "lr_stabilized_coeff_solve", "lr_svd", "lr_pinv", "lr_id_column", "lr_id_row", "lr_randomized_id",
                 "lr_tsid_from_column_id", "lr_cur_from_two_sided", "lr_randomized_cur", "lr_cur_id",
                 "lr_cur_error_fro"]:
        assert name in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.fail("liblowrank_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_1412_8447_b200 import _lib
    assert set(declared_symbols()) == set(_lib.SIGNATURES)
    _lib.load()


def test_product_library_does_not_link_the_oracle():
    out = subprocess.run(["nm", "-D", LIB], capture_output=True, text=True).stdout
    assert "lro_" not in out and "lref_" not in out
    deps = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "lowrank_oracle" not in deps and "lowrank_ref" not in deps


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_1412_8447_b200 import lowrank
    with pytest.raises(lowrank.LowrankCudaError):
        lowrank.Context(0)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)
