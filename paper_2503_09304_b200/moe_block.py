"""HF-style MoE block replacement (north-star "HF-style MoE block replacement").

``SparseMoeBlock`` is a drop-in for transformers' ``MixtralSparseMoeBlock`` (forward(hidden_states
[B, S, d]) -> [B, S, d]; parameters ``gate.weight [E, d]``, ``experts.gate_up_proj [E, 2F, d]``,
``experts.down_proj [E, d, F]`` — the installed transformers 5.5.0 layout) and, with
``shared_expert_intermediate_size``, for ``Qwen2MoeSparseMoeBlock`` (softmax-then-top-k routing
without renormalisation, plus a sigmoid-gated shared SwiGLU expert).

The forward is four libqmoe launch groups: router, permute (+row gather), grouped SwiGLU experts
on tcgen05 (gate_up with fused SiLU*up, then down scattered to slot order), combine.  Routing
follows the reference rule (softmax over the k picked logits, lower id wins ties, reference
model.py:122-134), which equals HF Mixtral's softmax -> top-k -> renormalise up to rounding and
tie order.  ``forward(x, residual=r)`` fuses the residual add into the combine.

Qwen's shared expert is not a second launch.  A SwiGLU of width Fs = S*F is the sum of S SwiGLUs
over its F-wide column blocks (down(silu(g) * u) = sum_s down[:, s] (silu(g_s) * u_s)), so it
runs as S extra experts of the routed width E..E+S-1 in the SAME grouped launch, every token
routed to all S of them with weight sigmoid(shared_expert_gate . h).  The router emits those
slots itself (qmoe_router_shared: the gate is one more logit row), and the combine sums routed
and shared slots in one pass.  Weights live in one [E+S, 2F, d] / [E+S, d, F] buffer pair; the
HF-named parameters are views of its first E experts.
"""

from __future__ import annotations

from typing import Optional

import torch
from torch import nn

from . import kernels as K


class _Gate(nn.Module):
    def __init__(self, weight: torch.Tensor):
        super().__init__()
        self.weight = nn.Parameter(weight, requires_grad=False)


class _Experts(nn.Module):
    def __init__(self, gate_up: torch.Tensor, down: torch.Tensor):
        super().__init__()
        self.gate_up_proj = nn.Parameter(gate_up, requires_grad=False)
        self.down_proj = nn.Parameter(down, requires_grad=False)


def shared_sub_experts(Fs: int, F: int) -> int:
    """Number of F-wide sub-experts a shared expert of width Fs runs as."""
    if Fs % F:
        raise ValueError(f"shared expert width {Fs} is not a multiple of the routed expert width {F}")
    return Fs // F


@torch.no_grad()
def pack_shared(gate_up_all: torch.Tensor, down_all: torch.Tensor, E: int, gate_proj: torch.Tensor,
                up_proj: torch.Tensor, down_proj: torch.Tensor) -> None:
    """Write an HF shared expert (gate_proj / up_proj [Fs, d], down_proj [d, Fs]) into sub-experts
    E.. of the grouped weight buffers (gate_up [E+S, 2F, d], down [E+S, d, F])."""
    F = down_all.shape[2]
    for s in range(gate_up_all.shape[0] - E):
        cols = slice(s * F, (s + 1) * F)
        gate_up_all[E + s, :F].copy_(gate_proj[cols])
        gate_up_all[E + s, F:].copy_(up_proj[cols])
        down_all[E + s].copy_(down_proj[:, cols])


class SparseMoeBlock(nn.Module):
    def __init__(self, hidden_size: int, intermediate_size: int, num_experts: int, top_k: int,
                 dtype: torch.dtype = torch.bfloat16, device: Optional[torch.device] = None,
                 route_mode: int = K.ROUTE_TOPK_SOFTMAX, shared_expert_intermediate_size: int = 0):
        super().__init__()
        device = device or torch.device("cuda")
        d, F, E = hidden_size, intermediate_size, num_experts
        self.hidden_dim, self.ffn_dim, self.num_experts, self.top_k = d, F, E, top_k
        self.route_mode = route_mode
        self.shared_ffn_dim = shared_expert_intermediate_size
        S = shared_sub_experts(shared_expert_intermediate_size, F) if shared_expert_intermediate_size else 0
        self.n_shared = S
        self._w_router = torch.empty((E + (1 if S else 0), d), dtype=dtype, device=device)
        self._gate_up = torch.empty((E + S, 2 * F, d), dtype=dtype, device=device)
        self._down = torch.empty((E + S, d, F), dtype=dtype, device=device)
        self.gate = _Gate(self._w_router[:E])
        self.experts = _Experts(self._gate_up[:E], self._down[:E])
        if S:
            self.shared_expert_gate = _Gate(self._w_router[E:])
        self.last_routing = None

    @classmethod
    def from_config(cls, config, **kw) -> "SparseMoeBlock":
        """Build from a transformers MixtralConfig / Qwen2MoeConfig."""
        if hasattr(config, "num_local_experts"):
            return cls(config.hidden_size, config.intermediate_size, config.num_local_experts,
                       config.num_experts_per_tok, **kw)
        return cls(config.hidden_size, config.moe_intermediate_size, config.num_experts, config.num_experts_per_tok,
                   route_mode=K.ROUTE_TOPK_SOFTMAX if config.norm_topk_prob else K.ROUTE_SOFTMAX_TOPK,
                   shared_expert_intermediate_size=config.shared_expert_intermediate_size, **kw)

    @torch.no_grad()
    def load_hf(self, block) -> "SparseMoeBlock":
        """Copy weights from a transformers Mixtral/Qwen2-MoE sparse block."""
        self.gate.weight.copy_(block.gate.weight)
        self.experts.gate_up_proj.copy_(block.experts.gate_up_proj)
        self.experts.down_proj.copy_(block.experts.down_proj)
        if self.n_shared:
            se = block.shared_expert
            pack_shared(self._gate_up, self._down, self.num_experts, se.gate_proj.weight, se.up_proj.weight,
                        se.down_proj.weight)
            self.shared_expert_gate.weight.copy_(block.shared_expert_gate.weight)
        return self

    @torch.no_grad()
    def init_random(self, seed: int = 0) -> "SparseMoeBlock":
        """W_r, W1, W3 ~ N(0, 1/d); W2 ~ N(0, 1/F) (SURVEY.md §8d paper workload); the shared expert
        likewise (down ~ N(0, 1/Fs)) and its gate ~ N(0, 1/d)."""
        g = torch.Generator(device=self._gate_up.device).manual_seed(seed)
        d, F, E = self.hidden_dim, self.ffn_dim, self.num_experts

        def rnd(shape, std):
            return torch.randn(shape, generator=g, device=self._gate_up.device, dtype=torch.float32).mul_(std)

        self.gate.weight.copy_(rnd((E, d), d ** -0.5))
        self.experts.gate_up_proj.copy_(rnd((E, 2 * F, d), d ** -0.5))
        self.experts.down_proj.copy_(rnd((E, d, F), F ** -0.5))
        if self.n_shared:
            Fs = self.shared_ffn_dim
            gu, dn = rnd((2 * Fs, d), d ** -0.5), rnd((d, Fs), Fs ** -0.5)
            pack_shared(self._gate_up, self._down, E, gu[:Fs], gu[Fs:], dn)
            self.shared_expert_gate.weight.copy_(rnd((1, d), d ** -0.5))
        return self

    def shared_expert_weights(self):
        """The shared expert in HF form: (gate_proj [Fs, d], up_proj [Fs, d], down_proj [d, Fs])."""
        E, F = self.num_experts, self.ffn_dim
        sub = self._gate_up[E:]
        return (sub[:, :F].reshape(-1, self.hidden_dim), sub[:, F:].reshape(-1, self.hidden_dim),
                torch.cat(list(self._down[E:]), 1))

    @torch.no_grad()
    def forward(self, hidden_states: torch.Tensor, residual: Optional[torch.Tensor] = None) -> torch.Tensor:
        shape = hidden_states.shape
        x = hidden_states.reshape(-1, self.hidden_dim).contiguous()
        T, k, S, d, F = x.shape[0], self.top_k, self.n_shared, self.hidden_dim, self.ffn_dim
        ids, w = K.router(x, self._w_router, k, self.route_mode, n_shared=S)
        slots, EE = k + S, self.num_experts + S
        # the shared sub-experts' queues are x's rows in token order: on the 1-CTA path their A
        # rows come straight from x and the permute gathers only the routed rows
        direct = S > 0 and K.shared_direct_ok(d, F, EE, T * slots)
        perm, offsets, xp = K.permute(ids, EE, x=x, gather_e_end=self.num_experts if direct else None)
        y = torch.empty((T * slots, d), dtype=x.dtype, device=x.device)
        act = K.workspace(T * slots * F * x.element_size(), "act", x.device).view(x.dtype)[: T * slots * F]
        K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, self._gate_up, self._down, y,
                     act_ws=act.view(T * slots, F), x_direct=x if direct else None, x_first=self.num_experts)
        res = None if residual is None else residual.reshape(-1, d).contiguous()
        self.last_routing = (ids[:, :k], w[:, :k])
        return K.combine(y, w, res).reshape(shape)
