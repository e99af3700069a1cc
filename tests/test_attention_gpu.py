"""Paged GQA decode attention (qmoe_paged_decode_attention) against a torch
fp32 restatement over the same page pool, for Mixtral's (32 query / 8 KV heads) and Qwen's
(16 / 16) head layouts, ragged lengths crossing page boundaries, and a non-contiguous block table.
Also against flash-attn's paged kernel (the library path it replaces)."""

import pytest
import torch

from paper_2503_09304_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _case(H, KV, lens, page=256, hd=128, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    B = len(lens)
    max_pages = max((n + page - 1) // page for n in lens)
    n_pages = B * max_pages + 3
    pool = torch.randn((n_pages, page, 2, KV, hd), device="cuda", generator=g).bfloat16()
    perm = torch.randperm(n_pages, device="cuda", generator=g)[: B * max_pages].int()  # scattered pages
    bt = perm.view(B, max_pages).contiguous()
    q = torch.randn((B, H, hd), device="cuda", generator=g).bfloat16()
    return q, pool, bt, torch.tensor(lens, dtype=torch.int32, device="cuda")


def _torch_ref(q, pool, bt, lens, scale):
    B, H, hd = q.shape
    page, KV = pool.shape[1], pool.shape[3]
    out = torch.empty((B, H, hd), dtype=torch.float32, device="cuda")
    for b in range(B):
        n = int(lens[b])
        rows = pool[bt[b].long()].reshape(-1, 2, KV, hd)[:n].float()  # [n, 2, KV, hd]
        k, v = rows[:, 0], rows[:, 1]
        for h in range(H):
            gq = h // (H // KV)
            p = torch.softmax((k[:, gq] @ q[b, h].float()) * scale, 0)
            out[b, h] = p @ v[:, gq]
    return out


@pytest.mark.parametrize("H,KV", [(32, 8), (16, 16), (16, 8)])
@pytest.mark.parametrize("lens", [[1], [255, 256, 257], [700, 3, 129, 512, 1], [180] * 32])
def test_paged_decode_matches_torch(cuda, H, KV, lens):
    q, pool, bt, ln = _case(H, KV, lens)
    scale = 128 ** -0.5
    got = K.paged_decode_attention(q, pool, bt, ln, max(lens), scale)
    ref = _torch_ref(q, pool, bt, ln, scale)
    err = (got.float() - ref).abs().max().item()
    assert err < 2e-2, err
    # repeated launches: the arrival counters are left zeroed
    assert torch.equal(K.paged_decode_attention(q, pool, bt, ln, max(lens), scale), got)


@pytest.mark.parametrize("H,KV", [(8, 2), (4, 4)])
def test_paged_decode_head_dim_64(cuda, H, KV):
    lens = [1, 64, 300, 513]
    q, pool, bt, ln = _case(H, KV, lens, hd=64, seed=9)
    got = K.paged_decode_attention(q, pool, bt, ln, max(lens), 64 ** -0.5)
    ref = _torch_ref(q, pool, bt, ln, 64 ** -0.5)
    assert (got.float() - ref).abs().max().item() < 2e-2


def test_workspace_reused_across_shapes(cuda):
    """Decode batches change shape every iteration and share one workspace: a small call after a
    large one must not find stale page partials where its arrival counters are (a bug this caught:
    counters placed after the shape-dependent partials)."""
    scale = 128 ** -0.5
    for H, KV, lens in [(32, 8, [700, 3, 129, 512, 1]), (16, 16, [300] * 8), (16, 8, [1]), (32, 8, [5, 260]),
                        (16, 16, [1, 2]), (32, 8, [900])]:
        q, pool, bt, ln = _case(H, KV, lens, seed=len(lens))
        got = K.paged_decode_attention(q, pool, bt, ln, max(lens), scale)
        ref = _torch_ref(q, pool, bt, ln, scale)
        assert (got.float() - ref).abs().max().item() < 2e-2, (H, KV, lens)


def test_paged_decode_matches_flash_attn(cuda):
    fa = pytest.importorskip("flash_attn")
    lens = [180 + 37 * i for i in range(32)]
    q, pool, bt, ln = _case(32, 8, lens, seed=3)
    got = K.paged_decode_attention(q, pool, bt, ln, max(lens), 128 ** -0.5)
    ref = fa.flash_attn_with_kvcache(q.view(32, 1, 32, 128), pool[:, :, 0], pool[:, :, 1], cache_seqlens=ln,
                                     block_table=bt, causal=True).view(32, 32, 128)
    assert (got.float() - ref.float()).abs().max().item() < 2e-2
