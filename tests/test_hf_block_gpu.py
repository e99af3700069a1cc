"""The HF drop-in is real: transformers 5.5.0 MixtralSparseMoeBlock / Qwen2MoeSparseMoeBlock,
loaded into SparseMoeBlock through from_config + load_hf, give the same layer output.

Shapes are the real Mixtral-8x7B and Qwen1.5-MoE-A2.7B MoE layers (BASELINE configs 2 and 4),
at decode (32), mid (1024) and the bench's prefill size (8192 tokens), so every kernel path the
bench runs (swap-AB, swap-AB CTA pair, the Qwen 1-CTA token tiles) is checked against HF itself.
The HF block runs in fp32 on the same bf16-rounded weights and inputs (so the comparison measures
the kernels' bf16 act/output rounding, not weight quantisation).  Bar: north_star's 1e-2 relative
(Frobenius over the layer output), and routing ids equal to HF's wherever HF's own top-k margin
exceeds the fp32-vs-bf16-accumulation band.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

transformers = pytest.importorskip("transformers")
from transformers import MixtralConfig, Qwen2MoeConfig  # noqa: E402
from transformers.models.mixtral.modeling_mixtral import MixtralSparseMoeBlock  # noqa: E402
from transformers.models.qwen2_moe.modeling_qwen2_moe import Qwen2MoeSparseMoeBlock  # noqa: E402

from paper_2503_09304_b200.moe_block import SparseMoeBlock  # noqa: E402


def _bf16_params(block, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    with torch.no_grad():
        for name, p in block.named_parameters():
            fan_in = p.shape[-1]
            p.copy_((torch.randn(p.shape, generator=g, device="cuda") * fan_in ** -0.5).bfloat16().float())
    return block


def _check(hf, ours, T, d, k, seed):
    x = torch.randn((1, T, d), generator=torch.Generator(device="cuda").manual_seed(seed), device="cuda").bfloat16()
    with torch.no_grad():
        ref = hf(x.float()).reshape(T, d)
        logits = x.reshape(T, d).float() @ hf.gate.weight.T
        _, _, hf_idx = hf.gate(x.reshape(T, d).float())
    got = ours(x).float().reshape(T, d)
    rel = ((got - ref).norm() / ref.norm()).item()
    ids, _ = ours.last_routing
    srt = logits.sort(1, descending=True).values
    safe = (srt[:, k - 1] - srt[:, k]) > 1e-3
    same = (ids.long() == hf_idx.sort(1).values).all(1)
    print(f"T={T}: rel {rel:.3e}, ids equal on {int(same[safe].sum())}/{int(safe.sum())} safe rows, "
          f"{int((~safe).sum())} near-tie rows")
    assert bool(same[safe].all())
    assert rel < 1e-2, rel
    return rel


@pytest.mark.parametrize("T", [32, 1024, 8192])
def test_mixtral_8x7b_block_matches_transformers(cuda, T):
    cfg = MixtralConfig(hidden_size=4096, intermediate_size=14336, num_local_experts=8, num_experts_per_tok=2)
    hf = _bf16_params(MixtralSparseMoeBlock(cfg).cuda().eval(), seed=11)
    ours = SparseMoeBlock.from_config(cfg, device=cuda).load_hf(hf)
    assert ours.gate.weight.dtype == torch.bfloat16
    _check(hf, ours, T, 4096, 2, seed=T)
    del hf, ours
    torch.cuda.empty_cache()


@pytest.mark.parametrize("T", [32, 1024, 8192])
def test_qwen15_moe_block_matches_transformers(cuda, T):
    cfg = Qwen2MoeConfig(hidden_size=2048, moe_intermediate_size=1408, shared_expert_intermediate_size=5632,
                         num_experts=60, num_experts_per_tok=4, norm_topk_prob=False)
    hf = _bf16_params(Qwen2MoeSparseMoeBlock(cfg).cuda().eval(), seed=12)
    ours = SparseMoeBlock.from_config(cfg, device=cuda).load_hf(hf)
    assert ours.shared_ffn_dim == 5632
    _check(hf, ours, T, 2048, 4, seed=T + 1)
    del hf, ours
    torch.cuda.empty_cache()
