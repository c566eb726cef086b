"""The C-ABI library loads (no GPU needed) and exports every symbol that
include/lmt_b200.h declares; the Python binding covers all of them."""

import ctypes
import os
import re

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "lmt_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lmt_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_1412_6986_b200 import _lib

    L = _lib.lib()
    names = header_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib.EXPORTS)


def test_version_and_validation_without_gpu():
    from paper_1412_6986_b200 import _lib

    assert b"sm_100a" in _lib.lib().lmt_version()
    rec = _lib.CInstance(64, 64, 32, 32, 0, 2, 2, 0, 1, 3, 2, 1, 1, 1, 1, 16, 16, 8, 8)
    buf = ctypes.create_string_buffer(512)
    n = _lib.lib().lmt_validate(ctypes.byref(rec), buf, 512)
    assert n == 1 and buf.value == b"grid size 256 < 512"


def test_execute_rejects_unaligned_in_without_gpu():
    """lmt_execute's argument contract (include/lmt_b200.h): the in pitch is a
    multiple of 4 floats and the base 16-byte aligned, checked before any
    device work."""
    from paper_1412_6986_b200 import _lib

    L = _lib.lib()
    rec = _lib.CInstance(1024, 1024, 1024, 1024, 5, 1, 1, 2, 1, 0, 0, 0, 0, 0, 0, 1024, 1024, 16, 16)
    fake = ctypes.c_void_p(1 << 20)
    for pitch, base in ((1042, 1 << 20), (1040, (1 << 20) + 4)):
        rc = L.lmt_execute(ctypes.byref(rec), None, 0, ctypes.c_void_p(base), 1026, 1026, pitch, fake, fake, None)
        assert rc == 4 and b"pitch" in L.lmt_last_error()


def test_struct_layouts_match_header():
    from paper_1412_6986_b200 import _lib

    assert ctypes.sizeof(_lib.CInstance) == 19 * 4
    assert ctypes.sizeof(_lib.CDevice) == 10 * 4
    assert ctypes.sizeof(_lib.CMeasurement) == 8 * 8 + 8 * 4
    assert ctypes.sizeof(_lib.CMeasureOpts) == 4 + 4 + 8 + 8 + 6 * 4 + 0  # + tune[6]


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    import pytest

    from paper_1412_6986_b200 import _lib
    from paper_1412_6986_b200.errors import LmtuneError

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(LmtuneError, match="no CPU fallback"):
        _lib.lib()
