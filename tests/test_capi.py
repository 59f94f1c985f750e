"""The C-ABI library loads without a GPU and exports exactly the entry points
include/netfuse_b200.h declares, with the ctypes signatures mirroring them."""

import ctypes
import re

from paper_2009_13062_b200 import _lib


def _declared():
    text = _lib.HEADER_PATH.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(nf_\w+)\s*\(([^;]*)\);", text, re.M)


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    decl = _declared()
    assert len(decl) >= 10
    for name, _ in decl:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes binding"


def test_ctypes_arity_matches_header():
    for name, params in _declared():
        params = params.strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        assert len(_lib.SIGNATURES[name]) == n, name


def test_status_strings_and_abi():
    lib = _lib.load()
    assert lib.nf_abi_version() == 2
    for code in range(4):
        assert isinstance(lib.nf_status_string(code), bytes)


def test_bad_arguments_fail_before_any_device_work():
    lib = _lib.load()
    # null pointers and non-positive sizes are rejected as shape errors
    assert lib.nf_grouped_linear(None, None, None, None, None, 1, 1, 1, 1, 0, 0, 0, 0,
                                 None) == _lib.NF_ERR_SHAPE
    assert lib.nf_attention(None, None, 1, 1, 1, 1, ctypes.c_float(1.0), 0, 0,
                            None) == _lib.NF_ERR_SHAPE
    assert lib.nf_pool2d(ctypes.c_void_p(16), ctypes.c_void_p(16), 1, 1, 4, 4, 7, 2, 2, 0, 0,
                         None) == _lib.NF_ERR_UNSUPPORTED
