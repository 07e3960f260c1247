"""The C-ABI library (no GPU needed): it loads, exports every entry point
include/qtm.h declares, and its host-side queries work without a device."""

import os
import re
import subprocess

import pytest

from paper_1810_03047_b200 import native

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "qtm.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(qtm_\w+)\s*\(", text,
                                 flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("qtm_problem_create", "qtm_run", "qtm_problem_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol():
    L = native.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (qtm_\w+)", out))
    assert set(declared_functions()) <= exported
    assert set(native.EXPORTS) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_queries_without_gpu():
    L = native.lib()
    assert L.qtm_abi_version() == native.ABI_VERSION
    v = native.variants()
    assert len(v) >= 10
    for threads, comps, rows in v:
        assert threads % 32 == 0 and comps >= 1 and (rows == 0 or 2 <= rows <= 13)
    assert L.qtm_device_count() >= 0


def test_create_rejects_bad_descriptor():
    import ctypes as C
    L = native.lib()
    h = C.c_void_p()
    desc = native.QtmProblemDesc()
    desc.abi_version = 999
    assert L.qtm_problem_create(C.byref(desc), C.byref(h)) == native.ERR_ARGS
    assert "ABI" in native.last_error()
    desc.abi_version = native.ABI_VERSION
    desc.dim = 2
    desc.method = 2  # neither ADAMS (0) nor BDF (1)
    assert L.qtm_problem_create(C.byref(desc), C.byref(h)) == native.ERR_ARGS
    assert "method" in native.last_error()
    desc.method = 1
    desc.max_order = 7  # BDF order <= 6 (ode.py:46)
    assert L.qtm_problem_create(C.byref(desc), C.byref(h)) == native.ERR_ARGS
    desc.max_order = 6
    desc.dim = 10000  # dense LU of I - h l0 G: dim <= 8192
    assert L.qtm_problem_create(C.byref(desc), C.byref(h)) == native.ERR_UNSUPPORTED


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(native, "_lib", None)
    monkeypatch.setattr(native, "LIB_PATH", str(tmp_path / "libqtm.so"))
    with pytest.raises(native.NativeLibraryError, match="no CPU fallback"):
        native.lib()
