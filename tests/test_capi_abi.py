"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a
GPU and exports every entry point include/sdg_gpu.h declares; the error
classes mirror the reference's (proj/src/errors.hpp:9-21)."""
import ctypes
import os
import re

import pytest

from paper_2008_04356_b200 import capi
from paper_2008_04356_b200 import types as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sdg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(capi.LIB_PATH):
        capi.build()
    lib = ctypes.CDLL(capi.LIB_PATH)
    names = declared("sdg_gpu.h")
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(capi.EXPORTED)


def test_binding_declares_every_symbol():
    lib = capi.lib()
    for n in capi.EXPORTED:
        assert getattr(lib, n).argtypes is not None or n in ("sdg_global_error",), n


def test_error_codes_map_to_reference_exceptions():
    for code, cls in [(T.ERR_CONFIG, T.ConfigError), (T.ERR_INVALID_STATE, T.InvalidStateError),
                      (T.ERR_PROTOCOL, T.ProtocolError)]:
        with pytest.raises(cls):
            T.raise_for(code, "x")
    T.raise_for(T.OK, "")


def test_struct_layout_matches_header():
    # sizes follow include/sdg_types.h field order (x86-64 ABI)
    assert ctypes.sizeof(T.BandSpec) == 24
    assert ctypes.sizeof(T.Gas) == 32
    assert ctypes.sizeof(T.MeshSpec) == 6 * 8 + 3 * 4 + 4 + 16 * 24 + 4 * 4 + 4 + 4 + 8
