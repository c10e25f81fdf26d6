"""CPU-side checks of the drop-in boundary: the C-ABI library loads without a
GPU and exports every entry point include/sdg_gpu.h declares; the error
classes mirror the reference's (proj/src/errors.hpp:9-21)."""
import ctypes
import os
import re

import numpy as np
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
    assert ctypes.sizeof(T.BandSpec) == 40
    assert ctypes.sizeof(T.Gas) == 32
    assert ctypes.sizeof(T.MeshSpec) == 6 * 8 + 3 * 4 + 4 + 16 * 40 + 4 * 4 + 4 + 4 + 8 + 4 + 4


def test_library_exports_nothing_but_the_c_abi():
    """-fvisibility=hidden: no symbol of namespace sdg leaks, so the library links
    next to the reference's own sdg_core (whose classes share that namespace).
    What remains besides the sdg_* entry points is libstdc++'s vague-linkage
    template instances (std::vector, ...)."""
    import subprocess
    if not os.path.exists(capi.LIB_PATH):
        capi.build()
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    names = [ln.split()[-1] for ln in out.splitlines() if ln.strip()]
    c_abi = sorted(n for n in names if n.startswith("sdg_"))
    assert c_abi == sorted(declared("sdg_gpu.h"))
    leaked = [n for n in names if not n.startswith("sdg_") and "3sdg" in n]
    assert not leaked, leaked[:10]
    others = [n for n in names if not n.startswith("sdg_") and not n.startswith(("_ZNSt", "_ZSt", "_ZTISt", "_ZTSSt",
                                                                               "_ZNKSt", "_ZTVSt", "_ZN9__gnu_cxx", "_ZZNSt"))]
    assert not others, others[:10]


def test_rk_coefficients_are_the_reference_scheme():
    """LowStorageRK (lsrk.cpp:7-29): Carpenter-Kennedy 5-stage 2N-storage RK4;
    c_s = sum of the b's the stage has seen through the a-recursion."""
    a, b, c = capi.rk_coefficients()
    assert a[0] == 0.0 and c[0] == 0.0
    assert abs(a[1] + 567301805773.0 / 1357537059087.0) < 1e-16
    assert abs(b[4] - 2277821191437.0 / 14882151754819.0) < 1e-16
    # consistency of the 2N scheme: c_{s+1} = c_s + b_s * (weight of reg in stage s)
    w = 1.0
    cs = [0.0]
    for s in range(4):
        cs.append(cs[-1] + b[s] * w)
        w = a[s + 1] * w + 1.0
    assert np.allclose(cs, c, atol=1e-15)
