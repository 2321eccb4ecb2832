"""CPU-side checks of the C ABI: the library builds, loads, and exports every
entry point include/rapdb_b200.h declares (no compute: there is no GPU here)."""

import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "rapdb_b200.h")
LIB = os.path.join(REPO, "paper_2605_29291_b200", "_rapdb_b200.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|long long)\s+(rapdb_\w+)\s*\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("rapdb_create", "rapdb_bind_dense", "rapdb_run", "rapdb_kkt", "rapdb_reinit",
                 "rapdb_smoothed_gap", "rapdb_probe_sweep"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("library not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    for name in declared():
        assert hasattr(lib, name), name


def test_binding_table_matches_header():
    from paper_2605_29291_b200 import _capi
    assert sorted(_capi.EXPORTS) == declared()


def test_missing_library_fails_loudly(tmp_path):
    from paper_2605_29291_b200 import _capi
    from paper_2605_29291_b200.errors import DeviceError
    saved = _capi._lib
    _capi._lib = None
    try:
        with pytest.raises(DeviceError):
            _capi.load(str(tmp_path / "nope.so"))
    finally:
        _capi._lib = saved


def test_no_cuda_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_29291_b200 import _capi
    from paper_2605_29291_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        _capi.Context(0)
