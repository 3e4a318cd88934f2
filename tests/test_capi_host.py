"""Host-only checks of the C ABI library (no GPU needed): it loads, it exports
every entry point include/cpm.h declares, and argument errors are reported
through return codes + cpm_last_error without touching the device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "cpm.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(cpm_[a-z0-9_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2110_06322_b200._build import build

    build()
    from paper_2110_06322_b200 import load_library

    return load_library()


def test_every_declared_symbol_is_exported(lib):
    names = _header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/cpm.h but not exported"


def test_binding_covers_header(lib):
    from paper_2110_06322_b200.cpm import exported_symbols

    assert set(_header_functions()) <= set(exported_symbols())


def test_argument_errors_without_gpu(lib):
    from paper_2110_06322_b200 import cpm

    out = ctypes.c_void_p()
    s = cpm._Surface()
    s.kind = 1
    s.param[0] = 1.0
    assert lib.cpm_build_band(None, 0.1, 3, 2.0, None, ctypes.byref(out)) == -1
    assert b"null" in lib.cpm_last_error()
    assert lib.cpm_build_band(ctypes.byref(s), 0.1, 2, 2.0, None, ctypes.byref(out)) == -1
    assert b"p = 3" in lib.cpm_last_error()
    assert lib.cpm_build_band(ctypes.byref(s), -1.0, 3, 2.0, None, ctypes.byref(out)) == -1
    s.kind = 7
    assert lib.cpm_build_band(ctypes.byref(s), 0.1, 3, 2.0, None, ctypes.byref(out)) == -1
    assert lib.cpm_apply(None, 1.0, None, None, None) == -1
    assert lib.cpm_solve(None, 1.0, None, None, 1e-10, 30, 10, None, None, None) == -1
    assert lib.cpm_band_eval_order(None, None, None) == -1
    assert lib.cpm_band_item_rounds(None, None) == -1
    assert b"null" in lib.cpm_last_error()
    assert lib.cpm_profile_read(b"nope", None, None) == -1
    assert lib.cpm_profile_read(b"extend", None, None) == 0


def test_version(lib):
    assert b"sm_100a" in lib.cpm_version()
