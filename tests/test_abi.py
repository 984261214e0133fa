"""The C-ABI library loads without a GPU and exports every entry point
declared in include/mpps_b200.h (no compute calls)."""
import ctypes
import os
import re

from paper_2312_17396_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mpps_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mpps_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_binding_surface():
    syms = declared_symbols()
    assert set(syms) == set(_lib.EXPORTED), syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.mpps_version() == 100


def test_struct_layout_matches_header():
    # void* + 2 long long + 5 int = 8 + 16 + 20 -> padded to 48 bytes
    assert ctypes.sizeof(_lib.CMat) == 48


def test_errors_without_gpu_are_loud():
    import torch
    if torch.cuda.is_available():
        return
    import pytest
    with pytest.raises(_lib.MppsCudaError):
        _lib.handle_for()
