"""CPU checks of the C ABI: the library builds, loads, exports every declared
symbol, and validates arguments before touching the device."""

import ctypes as C
import re
from pathlib import Path

import numpy as np

from paper_1611_09482_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "fastwavenet.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fw_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol(built_lib):
    lib = C.CDLL(str(built_lib))
    for name in declared():
        assert hasattr(lib, name), name


def test_version_and_validation_without_gpu(built_lib):
    lib = _lib.load(built_lib)
    assert lib.fw_version() == 100
    h = C.c_void_p()
    assert lib.fw_cell_create(None, 1, 0, 0, C.byref(h)) == _lib.FW_ERR_INVALID
    assert b"null descriptor" in lib.fw_last_error()
    dil = (C.c_int32 * 2)(1, 2)
    w = np.zeros(16, dtype=np.float32)
    p = w.ctypes.data
    desc = _lib.FwCellDesc(2, dil, 0, 4, 4, 4, 4, 0, p, p, p, p, p, p, p, p, p, p, p)
    assert lib.fw_cell_create(C.byref(desc), 1, 0, 0, C.byref(h)) == _lib.FW_ERR_INVALID
    assert b"channel" in lib.fw_last_error()
    pd = _lib.FwPlainDesc(1, 1, 1, 2, 1, 0, p, p)
    assert lib.fw_plain_create(C.byref(pd), 1, 0, C.byref(h)) == _lib.FW_ERR_INVALID
    assert b"filter_width" in lib.fw_last_error()
    assert lib.fw_destroy(None) == 0


def test_error_mapping():
    import pytest

    with pytest.raises(ValueError):
        _lib.check(_lib.FW_ERR_INVALID)
    with pytest.raises(_lib.QueueStateError):
        _lib.check(_lib.FW_ERR_STATE)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.FW_ERR_CUDA)
