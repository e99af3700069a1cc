"""Pin the oracle's SwiGLU / Qwen functions to the third-party source they restate.

The reference (moesim) has a tanh toy expert only; north_star's SwiGLU expert, the Qwen
``norm_topk_prob=False`` routing rule and the sigmoid-gated shared expert follow HF
transformers 5.5.0 (installed here, not in /root/reference):
  * modeling_mixtral.py  MixtralTopKRouter / MixtralExperts / MixtralSparseMoeBlock
  * modeling_qwen2_moe.py Qwen2MoeTopKRouter / Qwen2MoeMLP / Qwen2MoeSparseMoeBlock
These tests run those modules in fp64 on CPU on sliced shapes and require the oracle to agree
(ids bit-exact wherever the top-k margin exceeds HF's fp32 softmax rounding; outputs to 1e-6,
the fp32 routing-weight precision HF uses even for fp64 models).  Together with
tests/test_oracle.py (toy path pinned to the reference) this pins every oracle function the GPU
parity tests use.
"""

import numpy as np
import pytest
import torch

from oracle import moe_oracle as om

transformers = pytest.importorskip("transformers")
from transformers import MixtralConfig, Qwen2MoeConfig  # noqa: E402
from transformers.models.mixtral.modeling_mixtral import MixtralSparseMoeBlock  # noqa: E402
from transformers.models.qwen2_moe.modeling_qwen2_moe import Qwen2MoeSparseMoeBlock  # noqa: E402


def _init(block, seed):
    g = torch.Generator().manual_seed(seed)
    with torch.no_grad():
        for p in block.parameters():
            p.copy_(torch.randn(p.shape, generator=g, dtype=torch.float64) * p.shape[-1] ** -0.5)
    return block


def _margin_ok(scores: np.ndarray, k: int, tol: float) -> np.ndarray:
    """Rows whose k-th and (k+1)-th largest scores differ by more than tol."""
    s = -np.sort(-scores, axis=1)
    return (s[:, k - 1] - s[:, k]) > tol if s.shape[1] > k else np.ones(len(s), bool)


def _hf_ids(block, x):
    _, _, idx = block.gate(x)
    return np.sort(idx.numpy(), axis=1)


@pytest.mark.parametrize("T,d,F,E,k", [(64, 64, 96, 8, 2), (37, 128, 80, 8, 2), (16, 32, 48, 4, 4)])
def test_mixtral_block_matches_oracle(T, d, F, E, k):
    cfg = MixtralConfig(hidden_size=d, intermediate_size=F, num_local_experts=E, num_experts_per_tok=k)
    blk = _init(MixtralSparseMoeBlock(cfg).double().eval(), seed=T)
    x = torch.randn((1, T, d), generator=torch.Generator().manual_seed(1), dtype=torch.float64)
    with torch.no_grad():
        ref = blk(x).reshape(T, d).numpy()
        hf_ids = _hf_ids(blk, x.reshape(T, d))
    W = blk.gate.weight.detach().numpy()
    ids, w, out = om.sparse_moe_block(W, blk.experts.gate_up_proj.detach().numpy(),
                                      blk.experts.down_proj.detach().numpy(), x.reshape(T, d).numpy(), k)
    ok = _margin_ok(x.reshape(T, d).numpy() @ W.T, k, 1e-5)
    assert ok.mean() > 0.9
    assert np.array_equal(ids[ok], hf_ids[ok])
    assert np.abs(out - ref).max() / np.abs(ref).max() < 1e-6


@pytest.mark.parametrize("T,d,F,Fs,E,k", [(48, 64, 48, 96, 12, 4), (20, 32, 24, 64, 60, 4)])
def test_qwen2moe_block_matches_oracle(T, d, F, Fs, E, k):
    cfg = Qwen2MoeConfig(hidden_size=d, moe_intermediate_size=F, shared_expert_intermediate_size=Fs, num_experts=E,
                         num_experts_per_tok=k, norm_topk_prob=False)
    blk = _init(Qwen2MoeSparseMoeBlock(cfg).double().eval(), seed=T + 1)
    x = torch.randn((2, T // 2, d), generator=torch.Generator().manual_seed(2), dtype=torch.float64)
    H = x.reshape(T, d).numpy()
    with torch.no_grad():
        ref = blk(x).reshape(T, d).numpy()
        hf_ids = _hf_ids(blk, x.reshape(T, d))
    se = blk.shared_expert
    sgu = np.concatenate([se.gate_proj.weight.detach().numpy(), se.up_proj.weight.detach().numpy()], 0)
    ids, w, out = om.sparse_moe_block(blk.gate.weight.detach().numpy(), blk.experts.gate_up_proj.detach().numpy(),
                                      blk.experts.down_proj.detach().numpy(), H, k, qwen=True, shared_gate_up=sgu,
                                      shared_down=se.down_proj.weight.detach().numpy(),
                                      shared_gate=blk.shared_expert_gate.weight.detach().numpy())
    ok = _margin_ok(H @ blk.gate.weight.detach().numpy().T, k, 1e-5)
    assert ok.mean() > 0.9
    assert np.array_equal(ids[ok], hf_ids[ok])
    # norm_topk_prob=False: the weights are the full softmax at the picked ids (no renormalisation)
    with torch.no_grad():
        probs, hf_w, hf_idx = blk.gate(x.reshape(T, d))
    hf_w = np.take_along_axis(hf_w.numpy(), np.argsort(hf_idx.numpy(), axis=1), axis=1)
    assert np.abs(w[ok] - hf_w[ok]).max() < 1e-6
    assert np.all(w.sum(1) < 1.0)
    assert np.abs(out - ref).max() / np.abs(ref).max() < 1e-6


def test_reference_routing_rule_equals_hf_mixtral_renormalised_topk():
    """The reference's softmax over the k picked logits (model.py:122-134) equals HF Mixtral's
    softmax over all experts -> top-k -> renormalise (algebraically; here to fp32 rounding)."""
    rng = np.random.default_rng(5)
    W, H = rng.standard_normal((8, 16)), rng.standard_normal((200, 16))
    ids, w = om.route_many(W, H, 2)
    s = H @ W.T
    p = np.exp(s - s.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    top = np.take_along_axis(p, ids, 1)
    assert np.abs(w - top / top.sum(1, keepdims=True)).max() < 1e-12
