"""The C-ABI library loads without a GPU and exports exactly what include/qmoe.h declares."""

import ctypes
import re

from conftest import ROOT

from paper_2503_09304_b200 import _lib


def declared_symbols():
    text = (ROOT / "include" / "qmoe.h").read_text()
    return set(re.findall(r"QMOE_API\s+[\w\s\*]+?\b(qmoe_\w+)\s*\(", text))


def test_header_and_binding_agree():
    decl = declared_symbols()
    assert len(decl) >= 13
    assert decl == set(_lib.SIGNATURES)


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.qmoe_version() == 1
    assert lib.qmoe_status_string(_lib.QMOE_ERR_PARTIAL) == b"partial token"


def test_host_side_validation_without_gpu():
    """Argument validation runs before any device work, so it is testable on CPU."""
    lib = _lib.load()
    st = lib.qmoe_router(None, None, 4, 16, 70, 2, _lib.QMOE_F32, 0, None, None, None, None)
    assert st == _lib.QMOE_ERR_INVALID
    assert b"E=70" in lib.qmoe_last_error()
    st = lib.qmoe_permute(None, None, 4, 2, 8, None, None, None, 0, None, None, 0, None)
    assert st == _lib.QMOE_ERR_INVALID
    ws = lib.qmoe_permute_workspace_bytes(100000, 2, 8)
    assert ws >= 49 * 8 * 4
    try:
        _lib.check(_lib.QMOE_ERR_PARTIAL, "x")
    except Exception as exc:  # noqa: BLE001
        from paper_2503_09304_b200.core import PartialTokenError

        assert isinstance(exc, PartialTokenError)
    else:
        raise AssertionError("check() did not raise")


def test_exported_symbols_have_default_visibility_only():
    """Internal kernels stay hidden; only qmoe_* is exported (nm -D equivalent via dlsym)."""
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    assert not hasattr(lib, "_ZN4qmoe9set_errorEPKcz")
