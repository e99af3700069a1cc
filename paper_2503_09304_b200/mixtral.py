"""Mixtral-8x7B- and Qwen1.5-MoE-A2.7B-shaped decoder plugins for the serving engine.

Random-init bf16 weights of the real architectures (no checkpoints exist offline): RMSNorm,
GQA attention with RoPE over the device paged KV cache, a sparse MoE block per layer, final
norm + LM head with greedy (lowest-id-on-tie) emission.  The MoE block is the hot path and runs
entirely on libqmoe (router, permute, tcgen05 grouped SwiGLU experts, combine with the residual
fused); attention runs on libqmoe too: the paged GQA decode kernel over
the engine-owned page pool and the causal varlen prefill kernel (flash-attn's kernels only for
A/B runs: QMOE_FA_DECODE=1 / QMOE_FA_PREFILL=1).

Layer semantics = HF MixtralDecoderLayer / Qwen2MoeDecoderLayer:
  h2 = h + o_proj(attn(rope(q), rope(k), v))          (ATTENTION stage: returns x=norm2(h2), res=h2)
  h' = h2 + sum_j w_j * expert_j(x)  [+ sigmoid(g.x) * shared(x) for Qwen]   (ROUTER + EXPERTS)
Qwen's shared expert runs inside the grouped expert launch as 4 F-wide sub-experts (moe_block.py).
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

import torch

from . import kernels as K
from .core import Phase, StateCorruptionError
from .moe_block import pack_shared, shared_sub_experts


@dataclass(frozen=True)
class DecoderConfig:
    name: str
    num_layers: int
    hidden_dim: int
    ffn_dim: int
    num_experts: int
    top_k: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    vocab_size: int
    rope_theta: float
    rms_eps: float
    route_mode: int = K.ROUTE_TOPK_SOFTMAX
    shared_ffn_dim: int = 0
    max_position: int = 4096


MIXTRAL_8X7B = DecoderConfig("mixtral-8x7b", 32, 4096, 14336, 8, 2, 32, 8, 128, 32000, 1e6, 1e-5)
QWEN15_MOE_A27B = DecoderConfig("qwen1.5-moe-a2.7b", 24, 2048, 1408, 60, 4, 16, 16, 128, 151936, 1e6, 1e-6,
                                route_mode=K.ROUTE_SOFTMAX_TOPK, shared_ffn_dim=5632)


def rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype) * w


class _Layer:
    pass


class _DirectRows:
    """Gathered routed rows plus the layer input x, whose rows the shared sub-experts read directly
    (kernels.expert_ffn(x_direct=...)); opaque to the engine, which only hands it back."""

    __slots__ = ("xp", "x")

    def __init__(self, xp, x):
        self.xp, self.x = xp, x


class DecoderMoEModel:
    """Device plugin (engine.py interface) for a Mixtral/Qwen-shaped decoder."""

    # flash-attn paged KV needs blocks of 256 tokens; 384 pages/layer hold 32 x 3072 tokens
    kv_page_kwargs = {"page_size": 256, "initial_pages": 384}

    def __init__(self, cfg: DecoderConfig, device: Optional[torch.device] = None, seed: int = 0,
                 dtype: torch.dtype = torch.bfloat16, expert_range: Optional[tuple[int, int]] = None):
        """expert_range: hold the weights of engine-view experts [lo, hi) only (expert parallelism,
        ep_serving.py); the random draws are those of the full model, so every rank's experts equal
        the single-GPU model's."""
        self.cfg = cfg
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.dtype = dtype
        # Qwen's shared expert runs as S extra experts of the routed width in the grouped launch
        # (moe_block.py): the engine sees E + S experts and k + S slots per token
        S = shared_sub_experts(cfg.shared_ffn_dim, cfg.ffn_dim) if cfg.shared_ffn_dim else 0
        self.n_shared = S
        self.config = replace(cfg, num_experts=cfg.num_experts + S, top_k=cfg.top_k + S)  # engine view
        lo, hi = expert_range if expert_range is not None else (0, cfg.num_experts + S)
        if not 0 <= lo < hi <= cfg.num_experts + S:
            raise ValueError(f"bad expert range [{lo}, {hi}) of {cfg.num_experts + S}")
        self.e_lo, self.e_hi = lo, hi
        g = torch.Generator(device=self.device).manual_seed(seed)
        d, F, E, hd = cfg.hidden_dim, cfg.ffn_dim, cfg.num_experts, cfg.head_dim
        H, KV = cfg.n_heads, cfg.n_kv_heads

        def rnd(shape, std):
            return (torch.randn(shape, generator=g, device=self.device, dtype=torch.float32) * std).to(dtype)

        self.embedding = rnd((cfg.vocab_size, d), 1.0)
        self.layers = []
        for _ in range(cfg.num_layers):
            L = _Layer()
            L.ln1 = torch.ones(d, dtype=dtype, device=self.device)
            L.ln2 = torch.ones(d, dtype=dtype, device=self.device)
            L.w_qkv = rnd(((H + 2 * KV) * hd, d), d ** -0.5)
            L.w_o = rnd((d, H * hd), (H * hd) ** -0.5)
            L.w_router = torch.empty((E + (1 if S else 0), d), dtype=dtype, device=self.device)
            L.w_router[:E] = rnd((E, d), d ** -0.5)
            L.gate_up = torch.empty((hi - lo, 2 * F, d), dtype=dtype, device=self.device)
            L.down = torch.empty((hi - lo, d, F), dtype=dtype, device=self.device)
            for e in range(E):  # per expert to bound the fp32 temporary
                gu, dn = rnd((2 * F, d), d ** -0.5), rnd((d, F), F ** -0.5)
                if lo <= e < hi:
                    L.gate_up[e - lo], L.down[e - lo] = gu, dn
            if S:
                Fs = cfg.shared_ffn_dim
                sh_gate_up = rnd((2 * Fs, d), d ** -0.5)
                if hi - lo == E + S:
                    pack_shared(L.gate_up, L.down, E, sh_gate_up[:Fs], sh_gate_up[Fs:], rnd((d, Fs), Fs ** -0.5))
                else:
                    sgu = torch.empty((S, 2 * F, d), dtype=dtype, device=self.device)
                    sdn = torch.empty((S, d, F), dtype=dtype, device=self.device)
                    pack_shared(sgu, sdn, 0, sh_gate_up[:Fs], sh_gate_up[Fs:], rnd((d, Fs), Fs ** -0.5))
                    for e in range(max(lo, E), hi):
                        L.gate_up[e - lo], L.down[e - lo] = sgu[e - E], sdn[e - E]
                L.w_router[E:] = rnd((1, d), d ** -0.5)  # the shared expert's sigmoid gate
            self.layers.append(L)
        self.final_norm = torch.ones(d, dtype=dtype, device=self.device)
        self.lm_head = rnd((cfg.vocab_size, d), d ** -0.5)
        inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, device=self.device, dtype=torch.float32) / hd))
        ang = torch.arange(cfg.max_position, device=self.device, dtype=torch.float32)[:, None] * inv[None, :]
        emb = torch.cat([ang, ang], -1)
        self._cos, self._sin = emb.cos(), emb.sin()
        self._stop = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._pass = None  # (members, handles, ns, decode, expected cached entries, metadata) of the pass
        self.pass_serial = 0  # bumped by the engine at every execute (new_expert_state buffers)
        self._direct_shared = True  # shared sub-experts read x directly where the path allows it
        self._pass_bufs = None
        self.preempt_guard = None  # set by the engine per iteration (device-preempt mode)
        self._pinned_tok = None
        # decode attention: libqmoe's paged kernel (default) or flash-attn's (QMOE_FA_DECODE=1, A/B)
        import os

        self._fa_decode = os.environ.get("QMOE_FA_DECODE", "0") == "1"
        self._fa_prefill = os.environ.get("QMOE_FA_PREFILL", "0") == "1"  # flash-attn varlen prefill (A/B)
        if self._fa_decode or self._fa_prefill:  # library kernels only for A/B runs
            from flash_attn import flash_attn_varlen_func, flash_attn_with_kvcache

            self._fa_varlen, self._fa_kvcache = flash_attn_varlen_func, flash_attn_with_kvcache

    # ------------------------------------------------------------------ cache geometry
    def kv_row_shape(self):
        return (2, self.cfg.n_kv_heads, self.cfg.head_dim)

    def kv_entry_bytes(self) -> int:
        return 2 * self.cfg.n_kv_heads * self.cfg.head_dim * 2  # real bf16 K+V bytes per token per layer

    @property
    def kv_dtype(self):
        return self.dtype

    # ------------------------------------------------------------------ engine interface
    def embed_batch(self, tokens: list[int]) -> torch.Tensor:
        return self.embedding.index_select(0, torch.tensor(tokens, dtype=torch.long, device=self.device))

    def _rope(self, t: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
        cos, sin = self._cos[pos][:, None, :], self._sin[pos][:, None, :]
        tf = t.float()
        half = tf.shape[-1] // 2
        rot = torch.cat([-tf[..., half:], tf[..., :half]], -1)
        return (tf * cos + rot * sin).to(t.dtype)

    def attention_batch(self, layer: int, h: torch.Tensor, members, cache):
        cfg, L = self.cfg, self.layers[layer]
        H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
        T = h.shape[0]
        x = K.rmsnorm(h, L.ln1, cfg.rms_eps)
        qkv = x @ L.w_qkv.T
        # Per-pass state (handles, expected cached counts) and metadata (positions, slot mapping,
        # block table, lengths) are identical in every layer of a decode/prefill pass: built at the
        # pass's first layer (keyed by the engine's member list, one object per pass) and reused.
        pas = self._pass
        if pas is None or pas[0] is not members:
            decode = members[0].seq.phase is Phase.DECODE
            for m in members:
                if (m.seq.phase is Phase.DECODE) != decode:
                    raise StateCorruptionError(f"sequence {m.seq.id}: mixed phases in one batch")
            handles = [m.seq.cache_handle for m in members]
            expect = [m.seq.tokens_fed() for m in members] if decode else [0] * len(members)
            pas = self._pass = (members, handles, [m.n for m in members], decode, expect, {})
        _, handles, ns, decode, expect, meta = pas
        # every member must hold exactly its fed tokens at this layer (one list comparison)
        haves = cache.counts_at(handles, layer)
        if haves != expect:
            bad = next(i for i, (a, b) in enumerate(zip(haves, expect)) if a != b)
            raise StateCorruptionError(f"sequence {members[bad].seq.id} layer {layer}: {haves[bad]} cached entries")
        slots = cache.reserve_batch(handles, layer, ns, want_slots=not meta)
        if not meta:
            pos = [p for have, n in zip(expect, ns) for p in range(have, have + n)]
            meta["pos"] = torch.tensor(pos, dtype=torch.long, device=self.device)
            meta["slots"] = torch.tensor(slots, dtype=torch.int32, device=self.device)
            if decode:
                tables = [cache.page_table(h_) for h_ in handles]
                width = max(len(t) for t in tables)
                meta["bt"] = torch.tensor([t + [0] * (width - len(t)) for t in tables], dtype=torch.int32,
                                          device=self.device)
                lens = [have + n for have, n in zip(expect, ns)]
                meta["lens"] = torch.tensor(lens, dtype=torch.int32, device=self.device)
                meta["max_len"] = max(lens)
            else:
                cu = [0]
                for n in ns:
                    cu.append(cu[-1] + n)
                meta["cu"] = torch.tensor(cu, dtype=torch.int32, device=self.device)
                meta["max"] = max(ns)
        K.rope_(qkv, meta["pos"], self._cos, self._sin, H, KV, hd)
        q = qkv[:, : H * hd].view(T, H, hd)
        k = qkv[:, H * hd:(H + KV) * hd].view(T, KV, hd)
        v = qkv[:, (H + KV) * hd:].view(T, KV, hd)
        # guard: the engine's per-iteration preempt flag in device-preempt mode (no append once an
        # expert launch of this iteration stopped early, see engine._experts_device_preempt)
        # the K|V half of each packed qkv row is the pool's [2, KV, hd] entry layout: appended in place
        cache.scatter(layer, meta["slots"], qkv[:, H * hd:].view(T, 2, KV, hd), guard=self.preempt_guard)
        if decode and not self._fa_decode:
            # hand-written paged GQA decode attention on the page pool (csrc/attention.cu)
            attn = K.paged_decode_attention(q, cache.pool(layer), meta["bt"], meta["lens"], meta["max_len"],
                                            hd ** -0.5).view(T, H * hd)
        elif decode:
            pool = cache.pool(layer)
            attn = self._fa_kvcache(q.view(T, 1, H, hd), pool[:, :, 0], pool[:, :, 1], cache_seqlens=meta["lens"],
                                    block_table=meta["bt"], causal=True).view(T, H * hd)
        elif not self._fa_prefill:
            # hand-written causal varlen GQA prefill attention (csrc/attention_prefill.cu)
            attn = K.prefill_attention(q, k, v, meta["cu"], meta["max"], hd ** -0.5).view(T, H * hd)
        else:
            attn = self._fa_varlen(q, k, v, meta["cu"], meta["cu"], meta["max"], meta["max"],
                                   causal=True).reshape(T, H * hd)
        x_in, h2 = K.rmsnorm(attn @ L.w_o.T, L.ln2, cfg.rms_eps, add=h)  # h2 = h + o, x_in = norm2(h2)
        return x_in, h2

    def route_batch(self, layer: int, x: torch.Tensor):
        return K.router(x, self.layers[layer].w_router, self.cfg.top_k, self.cfg.route_mode, n_shared=self.n_shared)

    def new_expert_state(self, T: int):
        """Expert outputs y (fresh per layer) and per-token cursors.  One cursor vector serves every
        layer of an engine pass (pass_serial, set by the engine per execute): within a pass the
        cursors stay zero (only a preemption advances them, and it ends the pass), and a checkpoint
        keeps views of its own pass's vector only -- one fill kernel per pass instead of per layer.
        (y is not shared: a launch behind an early stop, run ahead by the host, may still write its
        split-K reduction rows.)"""
        y = torch.empty((T * self.config.top_k, self.cfg.hidden_dim), dtype=self.dtype, device=self.device)
        b = self._pass_bufs
        if b is None or b[0] != self.pass_serial or b[1] != T:
            b = self._pass_bufs = (self.pass_serial, T, torch.zeros(T, dtype=torch.int32, device=self.device))
        return y, b[2]

    def permute(self, ids, cursor, x):
        """Queues (+ gathered rows).  Qwen on the 1-CTA path: the shared sub-experts' rows are not
        gathered; the returned rows object then carries x as well (_DirectRows), which the engine
        passes back to run_experts unchanged (also across a queue-reusing resume)."""
        E = self.config.num_experts
        # only with this pass's fresh (all-zero) cursor: every token is then pending for every shared
        # sub-expert (a merged resume group may mix cursors, and its queues are subsets of x's rows)
        fresh = self._pass_bufs is not None and cursor is self._pass_bufs[2]
        if self.n_shared and fresh and self._direct_shared and K.shared_direct_ok(self.cfg.hidden_dim,
                                                                                  self.cfg.ffn_dim, E, ids.numel()):
            perm, offsets, xp = K.permute(ids, E, cursor=cursor, x=x, gather_e_end=self.cfg.num_experts)
            return perm, offsets, _DirectRows(xp, x)
        return K.permute(ids, E, cursor=cursor, x=x)

    def run_experts(self, layer: int, xp, offsets, perm, y, e_begin: int, e_end: int, preempt_flag=None,
                    progress=None, progress_seq: int = 0, cursor_out=None):
        L = self.layers[layer]
        x_direct = None
        if isinstance(xp, _DirectRows):
            xp, x_direct = xp.xp, xp.x
        rows = xp.shape[0]
        F = self.cfg.ffn_dim
        act = K.workspace(rows * F * 2, "act", self.device).view(self.dtype)[: rows * F].view(rows, F)
        stop = self._stop if cursor_out is None else cursor_out
        K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, L.gate_up, L.down, y, e_begin=e_begin, e_end=e_end,
                     act_ws=act, preempt_flag=preempt_flag, cursor_out=stop, progress=progress,
                     progress_seq=progress_seq, x_direct=x_direct, x_first=self.cfg.num_experts)
        return stop

    def advance_cursor(self, cursor, stop_dev):
        K.cursor_advance(cursor, stop_dev)

    def resume_point(self, cursor, stop_dev, offsets):
        return K.resume_point(cursor, stop_dev, offsets)

    def combine_batch(self, layer: int, y, w, res, x):
        # routed and (Qwen) shared-expert slots in one weighted sum, residual fused
        return K.combine(y, w, res)

    def emit_batch(self, h: torch.Tensor, rows: list[int]) -> list[int]:
        """Final norm + LM head + greedy argmax (lowest id on ties, reference model.py:166-169) in
        two launches (qmoe_rmsnorm, qmoe_lm_head_argmax: no [T, V] logits); the token ids reach
        the host through one pinned copy -- the scheduler routes them (EOS, lengths) on the host."""
        if self._pinned_tok is None or self._pinned_tok.numel() < len(rows):
            self._pinned_tok = torch.empty(max(64, len(rows)), dtype=torch.int32, pin_memory=True)
            self._tok_ready = torch.cuda.Event()
        if len(rows) == h.shape[0] and rows[-1] == len(rows) - 1:  # decode: every row is a last token
            hl = h
        else:
            hl = h.index_select(0, torch.tensor(rows, dtype=torch.long, device=self.device))
        tok = K.lm_head_argmax(K.rmsnorm(hl.contiguous(), self.final_norm, self.cfg.rms_eps), self.lm_head)
        out = self._pinned_tok[: len(rows)]
        out.copy_(tok, non_blocking=True)
        self._tok_ready.record()
        self._tok_ready.synchronize()
        return out.tolist()

    @staticmethod
    def cat_rows(parts):
        return parts[0] if len(parts) == 1 else torch.cat(parts, 0)
