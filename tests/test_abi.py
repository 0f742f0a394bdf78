"""The C ABI library loads on a CPU-only host and exports every entry point
include/tsfrac_b200.h declares (no device calls)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2002_11978_b200 import _native

HEADER = Path(__file__).resolve().parent.parent / "include" / "tsfrac_b200.h"


def _declared():
    txt = HEADER.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tsf_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_python_export_list():
    assert _declared() == sorted(_native.EXPORTS)


def test_library_loads_and_exports_all_symbols():
    if not _native.LIB_PATH.exists():
        pytest.skip("libtsfrac_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in _declared():
        assert hasattr(lib, name), name
    lib.tsf_abi_version.restype = ctypes.c_int
    assert lib.tsf_abi_version() == 4


def test_invalid_arguments_fail_without_a_device():
    if not _native.LIB_PATH.exists():
        pytest.skip("library not built")
    lib = _native.load()
    assert lib.tsf_plan_create(None, 8, 32, None, None, 0) == -1
    assert b"NULL" in lib.tsf_last_error()
    h = ctypes.c_void_p()
    assert lib.tsf_plan_create(ctypes.byref(h), 8, 24, None, None, 0) == -1  # L not pow2
    assert lib.tsf_fft_debug(12, 0, 1, None, None, None) == -1
