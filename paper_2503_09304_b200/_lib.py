"""ctypes binding of libqmoe.so (the C ABI in include/qmoe.h).

There is deliberately no fallback: if the shared library is missing or fails to load, every
kernel call raises.  Status codes map onto the reference's exception classes
(reference core.py:20-37) through ``check``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path
from typing import Optional

from .core import CacheCapacityError, PartialTokenError, StateCorruptionError

LIB_PATH = Path(__file__).resolve().parent / "libqmoe.so"

QMOE_OK = 0
QMOE_ERR_INVALID = 1
QMOE_ERR_STATE = 2
QMOE_ERR_PARTIAL = 3
QMOE_ERR_CAPACITY = 4
QMOE_ERR_CUDA = 5
QMOE_ERR_UNSUPPORTED = 6

QMOE_F64 = 0
QMOE_F32 = 1
QMOE_BF16 = 2

QMOE_ROUTE_TOPK_SOFTMAX = 0
QMOE_ROUTE_SOFTMAX_TOPK = 1

QMOE_EXPERT_TANH_AFFINE = 0
QMOE_EXPERT_SWIGLU = 1

QMOE_PATH_UNSUPPORTED = 0
QMOE_PATH_SWAP_AB = 1
QMOE_PATH_FUSED_1CTA = 2
QMOE_PATH_FUSED_PAIR = 3
QMOE_PATH_TWO_LAUNCH_1CTA = 4
QMOE_PATH_TWO_LAUNCH_PAIR = 5
QMOE_PATH_SWAP_PAIR = 6

_c_int = ctypes.c_int
_c_size = ctypes.c_size_t
_vp = ctypes.c_void_p

# name -> (restype, argtypes); must list every function include/qmoe.h declares.
SIGNATURES = {
    "qmoe_version": (_c_int, []),
    "qmoe_status_string": (ctypes.c_char_p, [_c_int]),
    "qmoe_last_error": (ctypes.c_char_p, []),
    "qmoe_router": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp]),
    "qmoe_router_shared": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp,
                                    _vp]),
    "qmoe_permute_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int]),
    "qmoe_permute": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _vp, _c_size, _vp, _vp, _c_size, _vp]),
    "qmoe_expert_ffn_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int, _c_int]),
    "qmoe_expert_ffn": (_c_int, [_c_int, _c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _c_int, _c_int,
                                 _c_int, _vp, _vp, _vp, _vp, _vp, _c_size, _vp]),
    "qmoe_expert_ffn_ex": (_c_int, [_c_int, _c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _c_int, _c_int,
                                    _c_int, _vp, _vp, _vp, _vp, _vp, _c_int, _vp, _c_size, _vp]),
    "qmoe_combine": (_c_int, [_c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp]),
    "qmoe_gather_rows": (_c_int, [_vp, _vp, _c_int, _c_size, _vp, _vp]),
    "qmoe_scatter_rows": (_c_int, [_vp, _vp, _c_int, _c_size, _vp, _vp]),
    "qmoe_cursor_advance": (_c_int, [_vp, _c_int, _vp, _vp]),
    "qmoe_resume_point": (_c_int, [_vp, _c_int, _vp, _vp, _c_int, _vp, _vp]),
    "qmoe_kv_append": (_c_int, [_vp, _vp, _vp, _c_int, _c_size, _vp]),
    "qmoe_kv_append_guarded": (_c_int, [_vp, _vp, _vp, _c_int, _c_size, _vp, _vp]),
    "qmoe_kv_gather": (_c_int, [_vp, _vp, _c_int, _c_size, _vp, _vp]),
    "qmoe_rmsnorm": (_c_int, [_vp, _vp, _vp, ctypes.c_float, _c_int, _c_int, _vp, _vp, _vp]),
    "qmoe_rope": (_c_int, [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _vp]),
    "qmoe_expert_ffn_path": (_c_int, [_c_int, _c_int, _c_int, _c_int]),
    "qmoe_paged_decode_attention_workspace_bytes": (_c_size, [_c_int, _c_int, _c_int]),
    "qmoe_paged_decode_attention": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int,
                                             _c_int, _c_int, ctypes.c_float, _vp, _vp, _c_size, _vp]),
    "qmoe_prefill_attention": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _vp, _c_int, _c_int, _c_int, _c_int, _c_int,
                                        ctypes.c_float, _vp, _c_int, _vp]),
    "qmoe_lm_head_argmax_workspace_bytes": (_c_size, []),
    "qmoe_lm_head_argmax": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _c_size, _vp]),
    "qmoe_expert_ffn_gather": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _c_int,
                                        _c_int, _vp, _vp, _vp, _vp, _vp, _c_size, _vp]),
    "qmoe_ipc_export": (_c_int, [_vp, _vp, ctypes.POINTER(_c_size)]),
    "qmoe_ipc_import": (_c_int, [_vp, _c_size, ctypes.POINTER(_vp)]),
    "qmoe_ep_dispatch": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_size, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "qmoe_ep_barrier": (_c_int, [_vp, _c_int, _c_int, _c_int, ctypes.c_longlong, _vp, _vp]),
    "qmoe_expert_ffn_peer": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _c_int, _vp, _vp, _vp,
                                      _c_size, _vp]),
    "qmoe_expert_ffn_peer_ex": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int,
                                         _c_int, _vp, _vp, _vp, _vp, _vp, _c_size, _vp]),
    "qmoe_ep_exchange_counts": (_c_int, [_vp, _c_int, _c_int, _c_int, _vp, _vp, _c_int, ctypes.c_longlong, _vp,
                                         _vp]),
    "qmoe_ep_dispatch_dev": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_size, _c_int, _c_int, _vp, _vp,
                                      _vp, _vp, _vp, _vp]),
    "qmoe_permute_ex": (_c_int, [_vp, _vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _c_size, _vp, _vp, _c_size,
                                 _vp]),
    "qmoe_expert_ffn_xs": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _vp,
                                    _vp, _vp, _vp, _vp, _c_int, _vp, _c_int, _c_int, _vp, _c_size, _vp]),
    "qmoe_kv_append_strided": (_c_int, [_vp, _vp, _vp, _c_int, _c_size, _c_size, _vp, _vp]),
    "qmoe_ep_share_rows": (_c_int, [_vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_size, _vp, _c_int, _c_int,
                                    _vp]),
    "qmoe_ep_collect_rows": (_c_int, [_vp, _vp, _vp, _vp, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _c_size,
                                      _vp]),
}

_lib: Optional[ctypes.CDLL] = None


class KernelLibraryMissing(RuntimeError):
    """libqmoe.so is not built or cannot be loaded; there is no CPU fallback."""


def load() -> ctypes.CDLL:
    """Load (once) and type the shared library; raises KernelLibraryMissing on failure."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("QMOE_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise KernelLibraryMissing(
            f"{path} not found: build it with `python -m paper_2503_09304_b200.build` (nvcc, sm_100a)"
        )
    try:
        lib = ctypes.CDLL(path)
    except OSError as exc:  # pragma: no cover - depends on the box
        raise KernelLibraryMissing(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    """Raise the exception class the reference uses for this failure kind."""
    if status == QMOE_OK:
        return
    lib = load()
    msg = lib.qmoe_last_error().decode(errors="replace")
    text = f"{what}: {lib.qmoe_status_string(status).decode()}: {msg}"
    if status == QMOE_ERR_INVALID:
        raise ValueError(text)
    if status == QMOE_ERR_STATE:
        raise StateCorruptionError(text)
    if status == QMOE_ERR_PARTIAL:
        raise PartialTokenError(text)
    if status == QMOE_ERR_CAPACITY:
        raise CacheCapacityError(text)
    raise RuntimeError(text)
