"""Device model plugins for the preemptive MoE engine.

``ModelConfig`` / ``MoEModel`` reproduce the reference's toy model (reference model.py:33-169):
identical seeded parameters (same numpy draw order, model.py:86-102), toy single-head attention,
affine-tanh experts, greedy LM head with the EOS logit penalty.  Parameters live on the device
in the chosen precision (f64 = the reference's arithmetic, f32, or bf16 on tensor cores).

Every MoE-path computation is a libqmoe kernel: router (qmoe_router), queue build + gather
(qmoe_permute), experts (qmoe_expert_ffn, tcgen05 for bf16), combine (qmoe_combine).  The
attention stage, embedding and LM head are outside the hot path and use plain torch.

Two interfaces:
  * the engine's batched device interface (``*_batch`` / ``permute`` / ``run_experts`` ...),
    documented in engine.py;
  * the reference's plugin API with host numpy in/out (``route``, ``route_many``,
    ``expert_forward``, ``expert_forward_many``, ``combine``, ``emit_token``, ``embed``,
    ``kv_project``, ``router_scores``) — same names, argument meaning and errors as
    reference model.py:104-169, computed by the same kernels.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import kernels as K
from .core import PartialTokenError, StateCorruptionError

NORM_EPS = 1e-9
EOS_LOGIT_PENALTY = 0.5


@dataclass(frozen=True)
class ModelConfig:
    """Shape and seed of the reference toy model (reference model.py:33-50)."""

    num_layers: int = 8
    hidden_dim: int = 16
    num_experts: int = 8
    top_k: int = 2
    vocab_size: int = 256
    seed: int = 0

    def validate(self) -> None:
        if not 1 <= self.num_layers <= 32:
            raise ValueError("num_layers must be in [1, 32]")
        if min(self.hidden_dim, self.num_experts, self.vocab_size) < 1:
            raise ValueError("all dimensions must be >= 1")
        if not 1 <= self.top_k <= self.num_experts:
            raise ValueError("top_k must satisfy 1 <= k <= num_experts")


@dataclass
class MemberRows:
    """One batch member's token rows inside the batch tensors."""

    seq: object
    row0: int
    n: int


def draw_toy_parameters(cfg: ModelConfig) -> dict[str, object]:
    """numpy arrays in the reference's draw order: embedding; w_key[l]; w_value[l]; w_router[l];
    expert_weight[l]; expert_bias[l]; w_out; b_out (all but the embedding scaled by 1/sqrt(d));
    then b_out[0] -= EOS_LOGIT_PENALTY."""
    d, e, v, L = cfg.hidden_dim, cfg.num_experts, cfg.vocab_size, cfg.num_layers
    rng = np.random.default_rng(cfg.seed)
    s = 1.0 / math.sqrt(d)
    p: dict[str, object] = {"embedding": rng.standard_normal((v, d))}
    for name, shape in (("w_key", (d, d)), ("w_value", (d, d)), ("w_router", (e, d)),
                        ("expert_weight", (e, d, d)), ("expert_bias", (e, d))):
        p[name] = [rng.standard_normal(shape) * s for _ in range(L)]
    p["w_out"] = rng.standard_normal((v, d)) * s
    b_out = rng.standard_normal(v) * s
    b_out[0] -= EOS_LOGIT_PENALTY
    p["b_out"] = b_out
    return p


class MoEModel:
    """The reference toy model, device-resident."""

    route_mode = K.ROUTE_TOPK_SOFTMAX
    expert_variant = K.EXPERT_TANH_AFFINE

    def __init__(self, config: ModelConfig, dtype: torch.dtype = torch.float64,
                 device: Optional[torch.device] = None):
        config.validate()
        self.config = config
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        p = draw_toy_parameters(config)
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(dtype).to(self.device)  # noqa: E731
        # Attention / LM head stay in at least f32 (outside the MoE hot path).
        side = torch.float64 if dtype == torch.float64 else torch.float32
        ts = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(side).to(self.device)  # noqa: E731
        self.embedding = ts(p["embedding"])
        self.w_key = [ts(a) for a in p["w_key"]]
        self.w_value = [ts(a) for a in p["w_value"]]
        self.w_router = [t(a) for a in p["w_router"]]
        self.expert_weight = [t(a) for a in p["expert_weight"]]
        self.expert_bias = [t(a) for a in p["expert_bias"]]
        self.w_out = ts(p["w_out"])
        self.b_out = ts(p["b_out"])
        self.side_dtype = side
        self._stop = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.preempt_guard = None  # set by the engine per iteration (device-preempt mode)

    # ------------------------------------------------------------------ cache geometry
    def kv_row_shape(self) -> tuple[int, ...]:
        return (2, self.config.hidden_dim)

    def kv_entry_bytes(self) -> int:
        return 2 * self.config.hidden_dim * 8  # reference units (model.py:277)

    @property
    def kv_dtype(self) -> torch.dtype:
        return self.side_dtype

    # ------------------------------------------------------------------ engine interface
    def embed_batch(self, tokens: list[int]) -> torch.Tensor:
        idx = torch.tensor(tokens, dtype=torch.long, device=self.device)
        return self.embedding.index_select(0, idx)

    @staticmethod
    def _normalize(v: torch.Tensor) -> torch.Tensor:
        return v / (torch.sqrt((v * v).sum(-1, keepdim=True)) + NORM_EPS)

    def attention_batch(self, layer: int, h: torch.Tensor, members: list[MemberRows], cache):
        """Toy attention stage (reference engine.py:252-301): append K/V of every new token to the
        member's cache pages, then attention over the member's entries; decode members are batched
        through one padded gather.  Returns (expert input, residual) — the same tensor here."""
        from .core import Phase

        hs = h.to(self.side_dtype)
        kv = torch.stack([hs @ self.w_key[layer].T, hs @ self.w_value[layer].T], 1).contiguous()  # [T, 2, d]
        slots: list[int] = []
        decode: list[MemberRows] = []
        for m in members:
            seq = m.seq
            have = cache.count(seq.cache_handle, layer)
            if seq.phase is Phase.DECODE:
                if have != seq.tokens_fed():
                    raise StateCorruptionError(
                        f"sequence {seq.id} layer {layer}: {have} cached entries, expected {seq.tokens_fed()}")
                decode.append(m)
            elif have != 0:
                raise StateCorruptionError(
                    f"sequence {seq.id} layer {layer}: prefill expects an empty layer, found {have} entries")
            slots += cache.reserve(seq.cache_handle, layer, m.n)
        cache.scatter(layer, slots, kv, guard=self.preempt_guard)  # guard: engine's device-preempt flag
        out = torch.empty_like(hs)
        decode_ids = {id(m) for m in decode}
        for m in members:
            if id(m) in decode_ids:
                continue
            r = slice(m.row0, m.row0 + m.n)
            q, keys, vals = hs[r], kv[r, 0], kv[r, 1]
            scores = q @ keys.T
            mask = torch.ones((m.n, m.n), dtype=torch.bool, device=self.device).tril_()
            scores = scores.masked_fill(~mask, float("-inf"))
            z = torch.exp(scores - scores.max(1, keepdim=True).values)
            wts = z / z.sum(1, keepdim=True)
            out[r] = self._normalize(q + wts @ vals)
        if decode:
            lens = [cache.count(m.seq.cache_handle, layer) for m in decode]
            Lmax = max(lens)
            idx = []
            for m, n in zip(decode, lens):
                s = cache.slots(m.seq.cache_handle, 0, n)
                idx += s + [s[0]] * (Lmax - n)
            gathered = torch.empty((len(idx), 2, self.config.hidden_dim), dtype=self.side_dtype, device=self.device)
            K.kv_gather(cache.pool(layer), torch.tensor(idx, dtype=torch.int32, device=self.device), gathered)
            g = gathered.view(len(decode), Lmax, 2, -1)
            rows = torch.tensor([m.row0 for m in decode], dtype=torch.long, device=self.device)
            q = hs.index_select(0, rows)
            scores = torch.einsum("bld,bd->bl", g[:, :, 0], q)
            valid = torch.arange(Lmax, device=self.device)[None, :] < torch.tensor(lens, device=self.device)[:, None]
            scores = scores.masked_fill(~valid, float("-inf"))
            z = torch.exp(scores - scores.max(1, keepdim=True).values)
            wts = z / z.sum(1, keepdim=True)
            out.index_copy_(0, rows, self._normalize(q + torch.einsum("bl,bld->bd", wts, g[:, :, 1])))
        x = out.to(self.dtype).contiguous()
        return x, x

    def route_batch(self, layer: int, x: torch.Tensor):
        return K.router(x, self.w_router[layer], self.config.top_k, self.route_mode)

    def new_expert_state(self, T: int):
        y = torch.empty((T * self.config.top_k, self.config.hidden_dim), dtype=self.dtype, device=self.device)
        cursor = torch.zeros(T, dtype=torch.int32, device=self.device)
        return y, cursor

    def permute(self, ids: torch.Tensor, cursor: torch.Tensor, x: torch.Tensor):
        return K.permute(ids, self.config.num_experts, cursor=cursor, x=x)

    def run_experts(self, layer: int, xp, offsets, perm, y, e_begin: int, e_end: int,
                    preempt_flag: Optional[torch.Tensor] = None, progress: Optional[torch.Tensor] = None,
                    progress_seq: int = 0, cursor_out: Optional[torch.Tensor] = None) -> torch.Tensor:
        stop = self._stop if cursor_out is None else cursor_out  # device or pinned host int32 [1]
        K.expert_ffn(self.expert_variant, xp, offsets, perm, self.expert_weight[layer], self.expert_bias[layer], y,
                     e_begin=e_begin, e_end=e_end, preempt_flag=preempt_flag, cursor_out=stop,
                     progress=progress, progress_seq=progress_seq)
        return stop

    def advance_cursor(self, cursor: torch.Tensor, stop_dev: torch.Tensor) -> None:
        K.cursor_advance(cursor, stop_dev)

    def resume_point(self, cursor: torch.Tensor, stop_dev: torch.Tensor, offsets: torch.Tensor) -> torch.Tensor:
        return K.resume_point(cursor, stop_dev, offsets)

    def combine_batch(self, layer: int, y, w, res, x) -> torch.Tensor:
        return K.combine(y, w, res)

    def emit_batch(self, h: torch.Tensor, rows: list[int]) -> list[int]:
        hl = h.index_select(0, torch.tensor(rows, dtype=torch.long, device=self.device)).to(self.side_dtype)
        logits = hl @ self.w_out.T + self.b_out
        return torch.argmax(logits, dim=1).tolist()  # first maximal index: ties to the lowest id

    @staticmethod
    def cat_rows(parts: list[torch.Tensor]) -> torch.Tensor:
        return parts[0] if len(parts) == 1 else torch.cat(parts, 0)

    # ------------------------------------------------------------------ reference plugin API (numpy in/out)
    def _dev(self, a) -> torch.Tensor:
        return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(self.dtype).to(self.device)

    def embed(self, token: int) -> np.ndarray:
        return self.embedding[token].double().cpu().numpy()

    def kv_project(self, h, layer: int):
        hs = self._dev(h).to(self.side_dtype)
        return (self.w_key[layer] @ hs).double().cpu().numpy(), (self.w_value[layer] @ hs).double().cpu().numpy()

    def router_scores(self, h, layer: int) -> np.ndarray:
        _, _, logits = K.router(self._dev(h)[None], self.w_router[layer], self.config.top_k, self.route_mode,
                                want_logits=True)
        return logits[0].double().cpu().numpy()

    def route_many(self, hiddens, layer: int) -> list[dict[int, float]]:
        ids, w = self.route_batch(layer, self._dev(hiddens).reshape(-1, self.config.hidden_dim))
        return [{int(e): float(x) for e, x in zip(ri, rw)} for ri, rw in zip(ids.tolist(), w.double().tolist())]

    def route(self, h, layer: int) -> dict[int, float]:
        return self.route_many(np.asarray(h)[None], layer)[0]

    def expert_forward_many(self, expert_id: int, layer: int, hiddens) -> np.ndarray:
        X = self._dev(hiddens).reshape(-1, self.config.hidden_dim)
        n = X.shape[0]
        E = self.config.num_experts
        offsets = torch.tensor([0] * (expert_id + 1) + [n] * (E - expert_id), dtype=torch.int32, device=self.device)
        perm = torch.arange(n, dtype=torch.int32, device=self.device)
        y = torch.empty_like(X)
        K.expert_ffn(self.expert_variant, X, offsets, perm, self.expert_weight[layer], self.expert_bias[layer], y,
                     e_begin=expert_id, e_end=expert_id + 1)
        return y.double().cpu().numpy()

    def expert_forward(self, expert_id: int, layer: int, h) -> np.ndarray:
        return self.expert_forward_many(expert_id, layer, np.asarray(h)[None])[0]

    def combine(self, residual, routing: dict[int, float], outputs: dict[int, object], pending: set[int]):
        """residual + sum of weighted expert outputs in ascending expert id (reference model.py:147-164)."""
        if pending:
            raise PartialTokenError(f"cannot combine token with pending experts {sorted(pending)}")
        if set(outputs) != set(routing):
            raise StateCorruptionError("expert outputs do not match the routed set")
        order = sorted(outputs)
        Y = self._dev(np.stack([np.asarray(outputs[e]) for e in order]))
        w = torch.tensor([[routing[e] for e in order]], dtype=K.acc_dtype(self.dtype), device=self.device)
        return K.combine(Y, w, self._dev(residual)[None])[0].double().cpu().numpy()

    def emit_token(self, h) -> int:
        return self.emit_batch(self._dev(h)[None], [0])[0]
