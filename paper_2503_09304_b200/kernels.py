"""Torch-facing wrappers over the libqmoe C ABI.

torch is plumbing here: it owns device memory and the current stream; every computation below
is one of the library's sm_100a kernels.  Each wrapper validates devices/dtypes/shapes, passes
raw pointers plus ``torch.cuda.current_stream()`` and maps status codes onto the reference's
exception classes.  Nothing here synchronises the host.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _lib
from ._lib import check

DTYPE_CODE = {torch.float64: _lib.QMOE_F64, torch.float32: _lib.QMOE_F32, torch.bfloat16: _lib.QMOE_BF16}

ROUTE_TOPK_SOFTMAX = _lib.QMOE_ROUTE_TOPK_SOFTMAX
ROUTE_SOFTMAX_TOPK = _lib.QMOE_ROUTE_SOFTMAX_TOPK
EXPERT_TANH_AFFINE = _lib.QMOE_EXPERT_TANH_AFFINE
EXPERT_SWIGLU = _lib.QMOE_EXPERT_SWIGLU

_workspaces: dict[tuple[int, int, str], torch.Tensor] = {}
_SHARED_DIRECT = __import__("os").environ.get("QMOE_SHARED_DIRECT", "1") != "0"


def _stream() -> int:
    # the raw cudaStream_t of the current device's current stream; torch.cuda.current_stream()
    # costs ~15 us of device-index resolution per call, which a serving layer pays ~20 times
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, name: str, dtype: Optional[torch.dtype] = None) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (libqmoe has no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")


def _code(t: torch.Tensor) -> int:
    try:
        return DTYPE_CODE[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}") from None


def acc_dtype(dtype: torch.dtype) -> torch.dtype:
    """Routing-weight dtype produced by the router for a given activation dtype."""
    return torch.float64 if dtype == torch.float64 else torch.float32


def workspace(nbytes: int, tag: str, device: torch.device) -> torch.Tensor:
    """Stream-ordered scratch, grown on demand and reused (one buffer per device/stream/tag).
    Zeroed when allocated: the expert-FFN workspace header must start zeroed (qmoe.h)."""
    key = (device.index or 0, _stream(), tag)
    buf = _workspaces.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
        _workspaces[key] = buf
    return buf


def router(x: torch.Tensor, w_router: torch.Tensor, k: int, mode: int = ROUTE_TOPK_SOFTMAX,
           want_logits: bool = False, n_shared: int = 0):
    """ids [T,k] int32 (ascending), weights [T,k] (f64 for f64 inputs else f32), optional logits.

    n_shared > 0 (qmoe_router_shared): w_router is [E + 1, d] with the shared expert's gate as the
    last row; ids / weights are [T, k + n_shared], the shared slots holding ids E.. with weight
    sigmoid(gate logit)."""
    _need(x, "x")
    _need(w_router, "w_router", x.dtype)
    T, d = x.shape
    rows = w_router.shape[0]
    E = rows - (1 if n_shared else 0)
    if w_router.shape[1] != d:
        raise ValueError("w_router must be [E, d]")
    ids = torch.empty((T, k + n_shared), dtype=torch.int32, device=x.device)
    w = torch.empty((T, k + n_shared), dtype=acc_dtype(x.dtype), device=x.device)
    logits = torch.empty((T, rows), dtype=w.dtype, device=x.device) if want_logits else None
    lib = _lib.load()
    if n_shared:
        check(lib.qmoe_router_shared(_ptr(x), _ptr(w_router), T, d, E, k, n_shared, _code(x), mode, _ptr(ids),
                                     _ptr(w), _ptr(logits), _stream()), "qmoe_router_shared")
    else:
        check(lib.qmoe_router(_ptr(x), _ptr(w_router), T, d, E, k, _code(x), mode, _ptr(ids), _ptr(w), _ptr(logits),
                              _stream()), "qmoe_router")
    return (ids, w, logits) if want_logits else (ids, w)


def permute(ids: torch.Tensor, num_experts: int, cursor: Optional[torch.Tensor] = None,
            x: Optional[torch.Tensor] = None, gather_e_end: Optional[int] = None):
    """Stable expert-major order of the pending slots.

    Returns (perm [T*k] int32 — only the first offsets[E] entries are meaningful,
    offsets [E+1] int32, xp [T*k, d] gathered rows or None).  gather_e_end: gather only the rows of
    experts below it (qmoe_permute_ex; the rest are read from x by expert_ffn(x_direct=...))."""
    _need(ids, "ids", torch.int32)
    T, k = ids.shape
    if cursor is not None:
        _need(cursor, "cursor", torch.int32)
        if cursor.shape != (T,):
            raise ValueError("cursor must be [T]")
    perm = torch.empty(T * k, dtype=torch.int32, device=ids.device)
    offsets = torch.empty(num_experts + 1, dtype=torch.int32, device=ids.device)
    xp = None
    row_bytes = 0
    if x is not None:
        _need(x, "x")
        if x.shape[0] != T:
            raise ValueError("x must have one row per token")
        xp = torch.empty((T * k, x.shape[1]), dtype=x.dtype, device=x.device)
        row_bytes = x.shape[1] * x.element_size()
    lib = _lib.load()
    nbytes = lib.qmoe_permute_workspace_bytes(T, k, num_experts)
    ws = workspace(nbytes, "permute", ids.device)
    if gather_e_end is None:
        check(lib.qmoe_permute(_ptr(ids), _ptr(cursor), T, k, num_experts, _ptr(perm), _ptr(offsets), _ptr(ws),
                               nbytes, _ptr(x), _ptr(xp), row_bytes, _stream()), "qmoe_permute")
    else:
        check(lib.qmoe_permute_ex(_ptr(ids), _ptr(cursor), T, k, num_experts, int(gather_e_end), _ptr(perm),
                                  _ptr(offsets), _ptr(ws), nbytes, _ptr(x), _ptr(xp), row_bytes, _stream()),
              "qmoe_permute_ex")
    return perm, offsets, xp


def expert_ffn(variant: int, xp: torch.Tensor, offsets: torch.Tensor, perm: torch.Tensor, w1: torch.Tensor,
               w2: torch.Tensor, y: torch.Tensor, e_begin: int = 0, e_end: Optional[int] = None,
               act_ws: Optional[torch.Tensor] = None, preempt_flag: Optional[torch.Tensor] = None,
               cursor_out: Optional[torch.Tensor] = None, progress: Optional[torch.Tensor] = None,
               progress_seq: int = 0, x_direct: Optional[torch.Tensor] = None, x_first: int = 0) -> None:
    """Run experts [e_begin, e_end) over their rows of xp; results land in y[perm[r]] (slot order).

    TANH_AFFINE: w1 = A [E, d, d], w2 = b [E, d].  SWIGLU: w1 = gate_up [E, 2F, d], w2 = down [E, d, F],
    act_ws = [rows, F] scratch.  preempt_flag: int32 device-visible flag polled at expert boundaries;
    cursor_out: int32 [1] device tensor receiving the first expert not completed.
    progress: pinned host int32 [E] (qmoe_expert_ffn_ex): progress[e] = progress_seq once expert e
    is drained on the device."""
    for name, t in (("xp", xp), ("w1", w1), ("w2", w2), ("y", y)):
        _need(t, name, xp.dtype)
    _need(offsets, "offsets", torch.int32)
    _need(perm, "perm", torch.int32)
    E = w1.shape[0]
    d = xp.shape[1]
    if variant == EXPERT_SWIGLU:
        F = w1.shape[1] // 2
        if w1.shape != (E, 2 * F, d) or w2.shape != (E, d, F):
            raise ValueError("SwiGLU weights must be gate_up [E, 2F, d] and down [E, d, F]")
        if act_ws is None:
            act_ws = torch.empty((xp.shape[0], F), dtype=xp.dtype, device=xp.device)
        _need(act_ws, "act_ws", xp.dtype)
        if act_ws.shape[0] < xp.shape[0] or act_ws.shape[1] != F:
            raise ValueError("act_ws must be [rows >= xp rows, F]")
    else:
        F = 0
        if w1.shape != (E, d, d) or w2.shape != (E, d):
            raise ValueError("tanh expert weights must be A [E, d, d] and b [E, d]")
    if offsets.shape != (E + 1,):
        raise ValueError("offsets must be [E+1]")
    if e_end is None:
        e_end = E
    if preempt_flag is not None and preempt_flag.dtype != torch.int32:
        raise ValueError("preempt_flag must be int32")
    lib = _lib.load()
    nbytes = lib.qmoe_expert_ffn_workspace_bytes(variant, _code(xp), d, xp.shape[0])
    ws = workspace(nbytes, "ffn", xp.device)
    if x_direct is not None:  # experts >= x_first read token rows straight from x (qmoe_expert_ffn_xs)
        _need(x_direct, "x_direct", xp.dtype)
        if progress is not None and (not progress.is_pinned() or progress.dtype != torch.int32):
            raise ValueError("progress must be a pinned host int32 tensor")
        check(lib.qmoe_expert_ffn_xs(_ptr(xp), _ptr(offsets), _ptr(perm), E, d, F, _ptr(w1), _ptr(w2), e_begin, e_end,
                                     xp.shape[0], _ptr(act_ws), _ptr(y), _ptr(preempt_flag), _ptr(cursor_out),
                                     _ptr(progress), int(progress_seq), _ptr(x_direct), x_direct.shape[0],
                                     int(x_first), _ptr(ws), nbytes, _stream()), "qmoe_expert_ffn_xs")
        return
    if progress is None:
        check(lib.qmoe_expert_ffn(variant, _code(xp), _ptr(xp), _ptr(offsets), _ptr(perm), E, d, F, _ptr(w1),
                                  _ptr(w2), e_begin, e_end, xp.shape[0], _ptr(act_ws), _ptr(y), _ptr(preempt_flag),
                                  _ptr(cursor_out), _ptr(ws), nbytes, _stream()), "qmoe_expert_ffn")
        return
    if not progress.is_pinned() or progress.dtype != torch.int32 or progress.numel() < E:
        raise ValueError("progress must be a pinned host int32 tensor with >= E entries")
    check(lib.qmoe_expert_ffn_ex(variant, _code(xp), _ptr(xp), _ptr(offsets), _ptr(perm), E, d, F, _ptr(w1), _ptr(w2),
                                 e_begin, e_end, xp.shape[0], _ptr(act_ws), _ptr(y), _ptr(preempt_flag),
                                 _ptr(cursor_out), _ptr(progress), int(progress_seq), _ptr(ws), nbytes, _stream()),
          "qmoe_expert_ffn_ex")


def combine(y: torch.Tensor, w: torch.Tensor, residual: Optional[torch.Tensor], out: Optional[torch.Tensor] = None):
    """out[t] = residual[t] + sum_j w[t,j] * y[t*k+j]  (j ascending expert id)."""
    T, k = w.shape
    d = y.shape[1]
    _need(y, "y")
    _need(w, "w", acc_dtype(y.dtype))
    if y.shape[0] != T * k:
        raise ValueError("y must hold T*k slot rows")
    if residual is not None:
        _need(residual, "residual", y.dtype)
    if out is None:
        out = torch.empty((T, d), dtype=y.dtype, device=y.device)
    lib = _lib.load()
    check(lib.qmoe_combine(_code(y), _ptr(y), _ptr(w), _ptr(residual), T, k, d, _ptr(out), _stream()),
          "qmoe_combine")
    return out


def gather_rows(src: torch.Tensor, idx: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """out[i] = src[idx[i]] (device row gather used to rebuild resumed batches)."""
    _need(src, "src")
    _need(idx, "idx", torch.int32)
    rows = idx.shape[0]
    if out is None:
        out = torch.empty((rows,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    row_bytes = src[0].numel() * src.element_size() if src.shape[0] else 1
    lib = _lib.load()
    check(lib.qmoe_gather_rows(_ptr(src), _ptr(idx), rows, row_bytes, _ptr(out), _stream()), "qmoe_gather_rows")
    return out


def scatter_rows(src: torch.Tensor, idx: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out[idx[i]] = src[i]."""
    _need(src, "src")
    _need(out, "out", src.dtype)
    _need(idx, "idx", torch.int32)
    rows = idx.shape[0]
    row_bytes = out[0].numel() * out.element_size() if out.shape[0] else 1
    lib = _lib.load()
    check(lib.qmoe_scatter_rows(_ptr(src), _ptr(idx), rows, row_bytes, _ptr(out), _stream()), "qmoe_scatter_rows")
    return out


def permute_launches(T: int, k: int, gather: bool = True) -> int:
    """Kernel launches qmoe_permute issues (mirrors csrc/permute.cu: chunk 2048 slots; a count
    pass only with >1 chunk; the wide gather only when more than 32 slots)."""
    S = T * k
    nblk = -(-S // 2048)
    return (1 if nblk > 1 else 0) + 1 + (1 if gather and S > 32 else 0)


def paged_decode_attention(q: torch.Tensor, pool: torch.Tensor, block_table: torch.Tensor, seq_lens: torch.Tensor,
                           max_len: int, scale: float, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """q [B, H, hd] bf16 (rows may be strided, e.g. a view into a packed qkv projection; the head
    and feature dimensions must be dense), pool [n_pages, page, 2, KV, hd] bf16, block_table
    [B, max_pages] int32, seq_lens [B] int32 -> out [B, H, hd] (one query per sequence)."""
    if not q.is_cuda or q.dtype != torch.bfloat16 or q.stride(2) != 1 or q.stride(1) != q.shape[2]:
        raise ValueError("q must be a CUDA bf16 [B, H, hd] tensor with dense heads")
    _need(pool, "pool", torch.bfloat16)
    _need(block_table, "block_table", torch.int32)
    _need(seq_lens, "seq_lens", torch.int32)
    B, H, hd = q.shape
    _, page, two, KV, hd2 = pool.shape
    if two != 2 or hd2 != hd:
        raise ValueError("pool must be [n_pages, page, 2, KV, head_dim]")
    max_pages = block_table.shape[1]
    if out is None:
        out = torch.empty((B, H, hd), dtype=q.dtype, device=q.device)
    lib = _lib.load()
    nbytes = lib.qmoe_paged_decode_attention_workspace_bytes(B, KV, max_pages)
    ws = workspace(nbytes, "attn", q.device)
    check(lib.qmoe_paged_decode_attention(_ptr(q), q.stride(0), _ptr(pool), _ptr(block_table), _ptr(seq_lens), B, H,
                                          KV, hd, page,
                                          max_pages, int(max_len), float(scale), _ptr(out), _ptr(ws), nbytes,
                                          _stream()), "qmoe_paged_decode_attention")
    return out


def prefill_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, cu_seqlens: torch.Tensor, max_len: int,
                      scale: float, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Causal varlen GQA attention of packed sequences: q [T, H, hd], k / v [T, KV, hd] bf16 (rows
    may be strided views into a packed qkv projection; heads and features dense), cu_seqlens
    [B + 1] int32 -> out [T, H, hd] bf16 (flash_attn_varlen_func(..., causal=True) semantics)."""
    for name, t in (("q", q), ("k", k), ("v", v)):
        if not t.is_cuda or t.dtype != torch.bfloat16 or t.dim() != 3 or t.stride(2) != 1 or t.stride(1) != t.shape[2]:
            raise ValueError(f"{name} must be a CUDA bf16 [T, heads, head_dim] tensor with dense heads")
    if k.stride(0) != v.stride(0) or k.shape != v.shape:
        raise ValueError("k and v must share shape and row stride")
    _need(cu_seqlens, "cu_seqlens", torch.int32)
    T, H, hd = q.shape
    KV = k.shape[1]
    B = cu_seqlens.shape[0] - 1
    if out is None:
        out = torch.empty((T, H, hd), dtype=q.dtype, device=q.device)
    lib = _lib.load()
    check(lib.qmoe_prefill_attention(_ptr(q), _ptr(k), _ptr(v), q.stride(0), k.stride(0), _ptr(cu_seqlens), B,
                                     int(max_len), H, KV, hd, float(scale), _ptr(out), out.stride(0), _stream()),
          "qmoe_prefill_attention")
    return out


def lm_head_argmax(h: torch.Tensor, w_out: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Greedy tokens [T] int32 on the device: argmax_v(w_out[v] . h[t]), lowest id on ties."""
    _need(h, "h", torch.bfloat16)
    _need(w_out, "w_out", torch.bfloat16)
    T, d = h.shape
    V = w_out.shape[0]
    if w_out.shape[1] != d:
        raise ValueError("w_out must be [V, d]")
    if out is None:
        out = torch.empty(T, dtype=torch.int32, device=h.device)
    _need(out, "out", torch.int32)
    lib = _lib.load()
    nbytes = lib.qmoe_lm_head_argmax_workspace_bytes()
    ws = workspace(nbytes, "lm_head", h.device)
    check(lib.qmoe_lm_head_argmax(_ptr(h), _ptr(w_out), T, d, V, _ptr(out), _ptr(ws), nbytes, _stream()),
          "qmoe_lm_head_argmax")
    return out


def resume_point(cursor: torch.Tensor, stop_dev: torch.Tensor, offsets: torch.Tensor) -> torch.Tensor:
    """Advance the cursors to the stop and return the resumed launch's offsets (experts below the
    stop emptied); the launch reuses the preempted launch's perm and Xp."""
    _need(cursor, "cursor", torch.int32)
    _need_stop(stop_dev)
    _need(offsets, "offsets", torch.int32)
    out = torch.empty_like(offsets)
    lib = _lib.load()
    check(lib.qmoe_resume_point(_ptr(cursor), cursor.shape[0], _ptr(stop_dev), _ptr(offsets), offsets.shape[0] - 1,
                                _ptr(out), _stream()), "qmoe_resume_point")
    return out


def _need_stop(t: torch.Tensor) -> None:
    """A launch's stop word: int32 in device memory or pinned host memory (device-accessible under
    UVA; the engine's stop ring lives there so the host reads it without a copy)."""
    if t.dtype != torch.int32 or not (t.is_cuda or t.is_pinned()):
        raise ValueError("stop must be an int32 CUDA or pinned host tensor")


def cursor_advance(cursor: torch.Tensor, stop_dev: torch.Tensor) -> None:
    _need(cursor, "cursor", torch.int32)
    _need_stop(stop_dev)
    lib = _lib.load()
    check(lib.qmoe_cursor_advance(_ptr(cursor), cursor.shape[0], _ptr(stop_dev), _stream()), "qmoe_cursor_advance")


def kv_append(pool: torch.Tensor, slot_mapping: torch.Tensor, rows: torch.Tensor,
              guard: Optional[torch.Tensor] = None) -> None:
    """pool[slot_mapping[i]] = rows[i]; with guard (the iteration's int32 device preempt flag) the
    append is skipped on the device when *guard < 0 (qmoe_kv_append_guarded).  rows [n, ...] may
    have a row stride (each row itself dense, e.g. a slice of packed qkv rows): no staging copy."""
    _need(pool, "pool")
    _need(slot_mapping, "slot_mapping", torch.int32)
    n = rows.shape[0]
    row_bytes = rows[0].numel() * rows.element_size() if n else 1
    lib = _lib.load()
    if not rows.is_contiguous():
        if not rows.is_cuda or rows.dtype != pool.dtype or not rows[0].is_contiguous():
            raise ValueError("rows must be CUDA rows of the pool dtype, each row dense")
        stride = rows.stride(0) * rows.element_size()
        if (stride | rows.data_ptr()) % 16:
            raise ValueError("strided rows must be 16-byte aligned")
        check(lib.qmoe_kv_append_strided(_ptr(pool), _ptr(slot_mapping), _ptr(rows), n, row_bytes, stride,
                                         _ptr(guard), _stream()), "qmoe_kv_append_strided")
        return
    _need(rows, "rows", pool.dtype)
    if guard is None:
        check(lib.qmoe_kv_append(_ptr(pool), _ptr(slot_mapping), _ptr(rows), n, row_bytes, _stream()),
              "qmoe_kv_append")
        return
    _need(guard, "guard", torch.int32)
    check(lib.qmoe_kv_append_guarded(_ptr(pool), _ptr(slot_mapping), _ptr(rows), n, row_bytes, _ptr(guard),
                                     _stream()), "qmoe_kv_append_guarded")


def kv_gather(pool: torch.Tensor, slot_mapping: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    _need(pool, "pool")
    _need(out, "out", pool.dtype)
    _need(slot_mapping, "slot_mapping", torch.int32)
    n = slot_mapping.shape[0]
    row_bytes = out[0].numel() * out.element_size() if n else 1
    lib = _lib.load()
    check(lib.qmoe_kv_gather(_ptr(pool), _ptr(slot_mapping), n, row_bytes, _ptr(out), _stream()), "qmoe_kv_gather")
    return out


def rmsnorm(x: torch.Tensor, weight: torch.Tensor, eps: float, add: Optional[torch.Tensor] = None):
    """rmsnorm(x [+ add]) * weight in one launch (bf16).  Returns out, or (out, x + add)."""
    _need(x, "x", torch.bfloat16)
    _need(weight, "weight", torch.bfloat16)
    T, d = x.shape
    out = torch.empty_like(x)
    summed = None
    if add is not None:
        _need(add, "add", torch.bfloat16)
        summed = torch.empty_like(x)
    lib = _lib.load()
    check(lib.qmoe_rmsnorm(_ptr(x), _ptr(add), _ptr(weight), float(eps), T, d, _ptr(out), _ptr(summed), _stream()),
          "qmoe_rmsnorm")
    return out if add is None else (out, summed)


def rope_(qkv: torch.Tensor, positions: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor, n_heads: int,
          n_kv_heads: int, head_dim: int) -> None:
    """In-place RoPE on the q and k parts of a packed [T, (H + 2*KV) * hd] qkv projection."""
    _need(qkv, "qkv", torch.bfloat16)
    _need(positions, "positions", torch.int64)
    _need(cos, "cos", torch.float32)
    _need(sin, "sin", torch.float32)
    T, width = qkv.shape
    k_ptr = qkv.data_ptr() + n_heads * head_dim * qkv.element_size()
    lib = _lib.load()
    check(lib.qmoe_rope(_ptr(qkv), k_ptr, _ptr(positions), _ptr(cos), _ptr(sin), T, n_heads, n_kv_heads, head_dim,
                        width, width, _stream()), "qmoe_rope")


# ------------------------------------------------------------------ expert parallel over peer memory

def ipc_export(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t in it)."""
    _need(t, "t")
    handle = ctypes.create_string_buffer(64)
    off = ctypes.c_size_t(0)
    lib = _lib.load()
    check(lib.qmoe_ipc_export(_ptr(t), handle, ctypes.byref(off)), "qmoe_ipc_export")
    return handle.raw, int(off.value)


def ipc_import(handle: bytes, offset: int) -> int:
    """Device address of a peer process's exported buffer (mapped once per allocation)."""
    out = ctypes.c_void_p(0)
    lib = _lib.load()
    check(lib.qmoe_ipc_import(ctypes.create_string_buffer(handle, 64), offset, ctypes.byref(out)), "qmoe_ipc_import")
    return int(out.value)


def ep_dispatch(x: torch.Tensor, perm: torch.Tensor, offsets: torch.Tensor, k: int, me: int, dest_rank: torch.Tensor,
                dest_base: torch.Tensor, x_peers: torch.Tensor, ret_peers: torch.Tensor) -> None:
    """Store every pending routed row of x into its owner's receive buffer (see qmoe.h)."""
    _need(x, "x")
    for name, t in (("perm", perm), ("offsets", offsets), ("dest_rank", dest_rank), ("dest_base", dest_base)):
        _need(t, name, torch.int32)
    _need(x_peers, "x_peers", torch.int64)
    _need(ret_peers, "ret_peers", torch.int64)
    T, d = x.shape
    lib = _lib.load()
    check(lib.qmoe_ep_dispatch(_ptr(x), _ptr(perm), _ptr(offsets), T, k, offsets.shape[0] - 1, d * x.element_size(),
                               me, _ptr(dest_rank), _ptr(dest_base), _ptr(x_peers), _ptr(ret_peers), _stream()),
          "qmoe_ep_dispatch")


def ep_barrier(flag_peers: torch.Tensor, me: int, world: int, epoch: int, error: Optional[torch.Tensor] = None,
               timeout_s: float = 10.0) -> None:
    """Stream-ordered device barrier over peer memory (flag_peers: int64 device [world])."""
    _need(flag_peers, "flag_peers", torch.int64)
    lib = _lib.load()
    check(lib.qmoe_ep_barrier(_ptr(flag_peers), me, world, epoch, int(timeout_s * 1e9), _ptr(error), _stream()),
          "qmoe_ep_barrier")


def expert_ffn_peer(xp: torch.Tensor, offsets: torch.Tensor, ret: torch.Tensor, gate_up: torch.Tensor,
                    down: torch.Tensor, y_peers: torch.Tensor, act_ws: Optional[torch.Tensor] = None) -> None:
    """Grouped SwiGLU experts over received rows; outputs go straight to their source ranks."""
    _need(xp, "xp", torch.bfloat16)
    _need(offsets, "offsets", torch.int32)
    _need(ret, "ret", torch.int32)
    _need(y_peers, "y_peers", torch.int64)
    E, twoF, d = gate_up.shape
    F = twoF // 2
    rows = xp.shape[0]
    if act_ws is None:
        act_ws = torch.empty((max(rows, 1), F), dtype=xp.dtype, device=xp.device)
    lib = _lib.load()
    nbytes = lib.qmoe_expert_ffn_workspace_bytes(EXPERT_SWIGLU, _lib.QMOE_BF16, d, rows)
    ws = workspace(nbytes, "ffn", xp.device)
    check(lib.qmoe_expert_ffn_peer(_ptr(xp), _ptr(offsets), _ptr(ret), E, d, F, _ptr(gate_up), _ptr(down), rows,
                                   _ptr(act_ws), _ptr(y_peers), _ptr(ws), nbytes, _stream()), "qmoe_expert_ffn_peer")


def ep_exchange_counts(offsets: torch.Tensor, me: int, world: int, counts_peers: torch.Tensor,
                       flag_peers: torch.Tensor, epoch: int, error: Optional[torch.Tensor] = None,
                       timeout_s: float = 10.0) -> None:
    """Publish this rank's queue lengths into every peer's counts[world][E] and barrier (see qmoe.h)."""
    _need(offsets, "offsets", torch.int32)
    _need(counts_peers, "counts_peers", torch.int64)
    _need(flag_peers, "flag_peers", torch.int64)
    lib = _lib.load()
    check(lib.qmoe_ep_exchange_counts(_ptr(offsets), offsets.shape[0] - 1, me, world, _ptr(counts_peers),
                                      _ptr(flag_peers), epoch, int(timeout_s * 1e9), _ptr(error), _stream()),
          "qmoe_ep_exchange_counts")


def ep_dispatch_dev(x: torch.Tensor, perm: torch.Tensor, offsets: torch.Tensor, k: int, me: int, world: int,
                    counts: torch.Tensor, bounds: torch.Tensor, x_peers: torch.Tensor, ret_peers: torch.Tensor,
                    loc_offsets: torch.Tensor) -> None:
    """Dispatch with device-built tables from the exchanged counts; writes loc_offsets."""
    _need(x, "x")
    for name, t in (("perm", perm), ("offsets", offsets), ("counts", counts), ("bounds", bounds),
                    ("loc_offsets", loc_offsets)):
        _need(t, name, torch.int32)
    _need(x_peers, "x_peers", torch.int64)
    _need(ret_peers, "ret_peers", torch.int64)
    T, d = x.shape
    lib = _lib.load()
    check(lib.qmoe_ep_dispatch_dev(_ptr(x), _ptr(perm), _ptr(offsets), T, k, offsets.shape[0] - 1, d * x.element_size(),
                                   me, world, _ptr(counts), _ptr(bounds), _ptr(x_peers), _ptr(ret_peers),
                                   _ptr(loc_offsets), _stream()), "qmoe_ep_dispatch_dev")


def ep_share_rows(y: torch.Tensor, perm: torch.Tensor, offsets: torch.Tensor, e_lo: int, e_hi: int,
                  recv_peers: torch.Tensor, me: int, world: int) -> None:
    """Push the output rows of experts [e_lo, e_hi) (queue positions of the launch) into the same
    slots of every peer's receive buffer (qmoe.h)."""
    _need(y, "y")
    _need(perm, "perm", torch.int32)
    _need(offsets, "offsets", torch.int32)
    _need(recv_peers, "recv_peers", torch.int64)
    lib = _lib.load()
    check(lib.qmoe_ep_share_rows(_ptr(y), _ptr(perm), _ptr(offsets), offsets.shape[0] - 1, e_lo, e_hi, y.shape[0],
                                 y.shape[1] * y.element_size(), _ptr(recv_peers), me, world, _stream()),
          "qmoe_ep_share_rows")


def ep_collect_rows(recv: torch.Tensor, y: torch.Tensor, perm: torch.Tensor, offsets: torch.Tensor, e_begin: int,
                    e_end: int, skip_lo: int, skip_hi: int) -> None:
    """y[perm[r]] = recv[perm[r]] for the launch's queue positions of the other ranks' experts."""
    _need(y, "y")
    _need(recv, "recv", y.dtype)
    _need(perm, "perm", torch.int32)
    _need(offsets, "offsets", torch.int32)
    if recv.shape[0] < y.shape[0] or recv.shape[1] != y.shape[1]:
        raise ValueError("recv must hold at least y's slots")
    lib = _lib.load()
    check(lib.qmoe_ep_collect_rows(_ptr(recv), _ptr(y), _ptr(perm), _ptr(offsets), offsets.shape[0] - 1, e_begin,
                                   e_end, skip_lo, skip_hi, y.shape[0], y.shape[1] * y.element_size(), _stream()),
          "qmoe_ep_collect_rows")


def expert_ffn_peer_ex(xp: torch.Tensor, offsets: torch.Tensor, ret: torch.Tensor, gate_up: torch.Tensor,
                       down: torch.Tensor, y_peers: torch.Tensor, rows_hint: int, act_ws: torch.Tensor,
                       e_begin: int = 0, e_end: Optional[int] = None, preempt_flag: Optional[torch.Tensor] = None,
                       cursor_out: Optional[torch.Tensor] = None) -> None:
    """Grouped SwiGLU experts over the received rows (count on the device, capacity = xp rows)."""
    _need(xp, "xp", torch.bfloat16)
    _need(offsets, "offsets", torch.int32)
    _need(ret, "ret", torch.int32)
    _need(y_peers, "y_peers", torch.int64)
    _need(act_ws, "act_ws", torch.bfloat16)
    E, twoF, d = gate_up.shape
    F = twoF // 2
    cap = xp.shape[0]
    if e_end is None:
        e_end = E
    lib = _lib.load()
    nbytes = lib.qmoe_expert_ffn_workspace_bytes(EXPERT_SWIGLU, _lib.QMOE_BF16, d, cap)
    ws = workspace(nbytes, "ffn", xp.device)
    check(lib.qmoe_expert_ffn_peer_ex(_ptr(xp), _ptr(offsets), _ptr(ret), E, d, F, _ptr(gate_up), _ptr(down), cap,
                                      int(rows_hint), e_begin, e_end, _ptr(act_ws), _ptr(y_peers), _ptr(preempt_flag),
                                      _ptr(cursor_out), _ptr(ws), nbytes, _stream()), "qmoe_expert_ffn_peer_ex")


# ------------------------------------------------------------------ fused row gather

PATH_SWAP_AB, PATH_FUSED_1CTA, PATH_FUSED_PAIR = _lib.QMOE_PATH_SWAP_AB, _lib.QMOE_PATH_FUSED_1CTA, _lib.QMOE_PATH_FUSED_PAIR
PATH_SWAP_PAIR = _lib.QMOE_PATH_SWAP_PAIR


def shared_direct_ok(d: int, F: int, E: int, rows: int) -> bool:
    """Whether the shared sub-experts may read their rows straight from X (qmoe_expert_ffn_xs): the
    single-launch 1-CTA path only; QMOE_SHARED_DIRECT=0 turns it off (A/B, tests)."""
    return _SHARED_DIRECT and expert_ffn_path(d, F, E, rows) == PATH_FUSED_1CTA


def expert_ffn_path(d: int, F: int, E: int, rows: int) -> int:
    """Which bf16 SwiGLU kernel qmoe_expert_ffn runs for `rows` routed rows over E experts."""
    return int(_lib.load().qmoe_expert_ffn_path(d, F, E, rows))


def gathers_rows(d: int, F: int, E: int, rows: int) -> bool:
    """True when expert_ffn_gather can run this shape (the kernel loads token rows from X itself
    with TMA tile::gather4, so the permute needs no Xp gather)."""
    return expert_ffn_path(d, F, E, rows) in (PATH_SWAP_AB, PATH_SWAP_PAIR, PATH_FUSED_1CTA, PATH_FUSED_PAIR)


def expert_ffn_gather(x: torch.Tensor, k: int, offsets: torch.Tensor, perm: torch.Tensor, gate_up: torch.Tensor,
                      down: torch.Tensor, y: torch.Tensor, e_begin: int = 0, e_end: Optional[int] = None,
                      act_ws: Optional[torch.Tensor] = None, preempt_flag: Optional[torch.Tensor] = None,
                      cursor_out: Optional[torch.Tensor] = None) -> None:
    """Grouped bf16 SwiGLU experts with the row gather fused into the GEMM (TMA tile::gather4):
    the i-th row of expert e is x[perm[offsets[e] + i] // k]; results land in y[perm[r]]."""
    _need(x, "x", torch.bfloat16)
    for name, t in (("gate_up", gate_up), ("down", down), ("y", y)):
        _need(t, name, torch.bfloat16)
    _need(offsets, "offsets", torch.int32)
    _need(perm, "perm", torch.int32)
    T, d = x.shape
    E, twoF, _ = gate_up.shape
    F = twoF // 2
    rows = T * k
    if act_ws is None:
        act_ws = torch.empty((max(rows, 1), F), dtype=x.dtype, device=x.device)
    if e_end is None:
        e_end = E
    lib = _lib.load()
    nbytes = lib.qmoe_expert_ffn_workspace_bytes(EXPERT_SWIGLU, _lib.QMOE_BF16, d, rows)
    ws = workspace(nbytes, "ffn", x.device)
    check(lib.qmoe_expert_ffn_gather(_ptr(x), T, k, _ptr(offsets), _ptr(perm), E, d, F, _ptr(gate_up), _ptr(down),
                                     e_begin, e_end, _ptr(act_ws), _ptr(y), _ptr(preempt_flag), _ptr(cursor_out),
                                     _ptr(ws), nbytes, _stream()), "qmoe_expert_ffn_gather")
