"""HF-style MoE block replacement (north-star "HF-style MoE block replacement").

``SparseMoeBlock`` is a drop-in for transformers' ``MixtralSparseMoeBlock`` (forward(hidden_states
[B, S, d]) -> [B, S, d]; parameters ``gate.weight [E, d]``, ``experts.gate_up_proj [E, 2F, d]``,
``experts.down_proj [E, d, F]`` — the installed transformers 5.5.0 layout) and, with
``shared_expert_intermediate_size``, for ``Qwen2MoeSparseMoeBlock`` (softmax-then-top-k routing
without renormalisation, plus a sigmoid-gated shared SwiGLU expert).

The forward is four libqmoe launches groups: router, permute (+row gather), grouped SwiGLU
experts on tcgen05 (gate_up with fused SiLU*up, then down scattered to slot order), combine.
Routing follows the reference rule (softmax over the k picked logits, lower id wins ties,
reference model.py:122-134), which equals HF Mixtral's softmax -> top-k -> renormalise up to
rounding and tie order.  ``forward(x, residual=r)`` fuses the residual add into the combine.
"""

from __future__ import annotations

from typing import Optional

import torch
from torch import nn

from . import kernels as K


class _Gate(nn.Module):
    def __init__(self, E: int, d: int, dtype, device):
        super().__init__()
        self.weight = nn.Parameter(torch.empty((E, d), dtype=dtype, device=device), requires_grad=False)


class _Experts(nn.Module):
    def __init__(self, E: int, d: int, F: int, dtype, device):
        super().__init__()
        self.gate_up_proj = nn.Parameter(torch.empty((E, 2 * F, d), dtype=dtype, device=device), requires_grad=False)
        self.down_proj = nn.Parameter(torch.empty((E, d, F), dtype=dtype, device=device), requires_grad=False)


class SparseMoeBlock(nn.Module):
    def __init__(self, hidden_size: int, intermediate_size: int, num_experts: int, top_k: int,
                 dtype: torch.dtype = torch.bfloat16, device: Optional[torch.device] = None,
                 route_mode: int = K.ROUTE_TOPK_SOFTMAX, shared_expert_intermediate_size: int = 0):
        super().__init__()
        device = device or torch.device("cuda")
        self.hidden_dim, self.ffn_dim, self.num_experts, self.top_k = hidden_size, intermediate_size, num_experts, top_k
        self.route_mode = route_mode
        self.gate = _Gate(num_experts, hidden_size, dtype, device)
        self.experts = _Experts(num_experts, hidden_size, intermediate_size, dtype, device)
        self.shared_ffn_dim = shared_expert_intermediate_size
        if shared_expert_intermediate_size:
            # Qwen2-MoE shared expert, stored as a 1-expert grouped problem for the same kernel
            self.shared_expert = _Experts(1, hidden_size, shared_expert_intermediate_size, dtype, device)
            self.shared_expert_gate = _Gate(1, hidden_size, dtype, device)
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
        if self.shared_ffn_dim:
            se = block.shared_expert
            self.shared_expert.gate_up_proj[0].copy_(torch.cat([se.gate_proj.weight, se.up_proj.weight], 0))
            self.shared_expert.down_proj[0].copy_(se.down_proj.weight)
            self.shared_expert_gate.weight.copy_(block.shared_expert_gate.weight)
        return self

    @torch.no_grad()
    def init_random(self, seed: int = 0) -> "SparseMoeBlock":
        """W_r, W1, W3 ~ N(0, 1/d); W2 ~ N(0, 1/F) (SURVEY.md §8d paper workload)."""
        g = torch.Generator(device=self.gate.weight.device).manual_seed(seed)
        d, F = self.hidden_dim, self.ffn_dim
        for t, std in ((self.gate.weight, d ** -0.5), (self.experts.gate_up_proj, d ** -0.5),
                       (self.experts.down_proj, F ** -0.5)):
            t.copy_(torch.randn(t.shape, generator=g, device=t.device, dtype=torch.float32).mul_(std))
        if self.shared_ffn_dim:
            Fs = self.shared_ffn_dim
            for t, std in ((self.shared_expert.gate_up_proj, d ** -0.5), (self.shared_expert.down_proj, Fs ** -0.5),
                           (self.shared_expert_gate.weight, d ** -0.5)):
                t.copy_(torch.randn(t.shape, generator=g, device=t.device, dtype=torch.float32).mul_(std))
        return self

    def _shared(self, x: torch.Tensor) -> torch.Tensor:
        T = x.shape[0]
        dev = x.device
        offsets = (torch.arange(0, 2 * T, T, dtype=torch.int32, device=dev) if T  # [0, T] without an H2D sync
                   else torch.zeros(2, dtype=torch.int32, device=dev))
        perm = torch.arange(T, dtype=torch.int32, device=dev)
        ys = torch.empty_like(x)
        K.expert_ffn(K.EXPERT_SWIGLU, x, offsets, perm, self.shared_expert.gate_up_proj, self.shared_expert.down_proj,
                     ys, act_ws=K.workspace(T * self.shared_ffn_dim * x.element_size(), "act_shared", dev)
                     .view(x.dtype)[: T * self.shared_ffn_dim].view(T, self.shared_ffn_dim))
        return ys

    @torch.no_grad()
    def forward(self, hidden_states: torch.Tensor, residual: Optional[torch.Tensor] = None) -> torch.Tensor:
        shape = hidden_states.shape
        x = hidden_states.reshape(-1, self.hidden_dim).contiguous()
        T, k, E, d, F = x.shape[0], self.top_k, self.num_experts, self.hidden_dim, self.ffn_dim
        ids, w = K.router(x, self.gate.weight, k, self.route_mode)
        perm, offsets, xp = K.permute(ids, E, x=x)
        y = torch.empty((T * k, d), dtype=x.dtype, device=x.device)
        act = K.workspace(T * k * F * x.element_size(), "act", x.device).view(x.dtype)[: T * k * F].view(T * k, F)
        K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, self.experts.gate_up_proj, self.experts.down_proj, y,
                     act_ws=act)
        res = None if residual is None else residual.reshape(-1, d).contiguous()
        if self.shared_ffn_dim:
            # res + sigmoid(g . x) * shared(x): a one-slot combine on the shared expert's output
            gate = torch.sigmoid(K.router(x, self.shared_expert_gate.weight, 1, want_logits=True)[2])
            res = K.combine(self._shared(x), gate, res)
        self.last_routing = (ids, w)
        return K.combine(y, w, res).reshape(shape)
