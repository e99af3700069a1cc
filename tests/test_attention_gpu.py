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


# ------------------------------------------------------------------------- prefill (varlen, causal)

def _prefill_case(H, KV, lens, hd=128, seed=0):
    """q / k / v as strided views into one packed [T, (H + 2 KV) hd] projection, as the decoders
    hold them."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    T = sum(lens)
    qkv = torch.randn((T, (H + 2 * KV) * hd), device="cuda", generator=g).bfloat16()
    q = qkv[:, : H * hd].view(T, H, hd)
    k = qkv[:, H * hd:(H + KV) * hd].view(T, KV, hd)
    v = qkv[:, (H + KV) * hd:].view(T, KV, hd)
    cu = [0]
    for n in lens:
        cu.append(cu[-1] + n)
    return q, k, v, torch.tensor(cu, dtype=torch.int32, device="cuda")


def _prefill_ref(q, k, v, cu, scale):
    T, H, hd = q.shape
    KV = k.shape[1]
    out = torch.empty((T, H, hd), dtype=torch.float32, device="cuda")
    c = cu.tolist()
    for b in range(len(c) - 1):
        s, e = c[b], c[b + 1]
        n = e - s
        mask = torch.ones((n, n), dtype=torch.bool, device="cuda").tril()
        for h in range(H):
            gq = h // (H // KV)
            sc = (q[s:e, h].float() @ k[s:e, gq].float().T) * scale
            p = torch.softmax(sc.masked_fill(~mask, float("-inf")), -1)
            out[s:e, h] = p @ v[s:e, gq].float()
    return out


@pytest.mark.parametrize("H,KV", [(32, 8), (16, 16), (8, 2)])
@pytest.mark.parametrize("lens", [[1], [64], [65, 3, 200], [513, 17, 64, 1000, 2], [1100, 5, 130]])
def test_prefill_attention_matches_torch(cuda, H, KV, lens):
    q, k, v, cu = _prefill_case(H, KV, lens)
    scale = 128 ** -0.5
    got = K.prefill_attention(q, k, v, cu, max(lens), scale)
    ref = _prefill_ref(q, k, v, cu, scale)
    err = (got.float() - ref).abs().max().item()
    assert err < 2e-2, err
    assert torch.equal(K.prefill_attention(q, k, v, cu, max(lens), scale), got)  # deterministic


@pytest.mark.parametrize("H,KV", [(8, 2), (4, 4)])
def test_prefill_attention_head_dim_64(cuda, H, KV):
    lens = [1, 64, 300, 129]
    q, k, v, cu = _prefill_case(H, KV, lens, hd=64, seed=5)
    got = K.prefill_attention(q, k, v, cu, max(lens), 64 ** -0.5)
    ref = _prefill_ref(q, k, v, cu, 64 ** -0.5)
    assert (got.float() - ref).abs().max().item() < 2e-2


def test_prefill_attention_matches_flash_attn(cuda):
    """Against the library kernel it replaces (flash_attn_varlen_func, causal), Mixtral heads."""
    flash_attn = pytest.importorskip("flash_attn")
    lens = [700, 1, 256, 31, 2048]
    q, k, v, cu = _prefill_case(32, 8, lens, seed=3)
    got = K.prefill_attention(q, k, v, cu, max(lens), 128 ** -0.5)
    fa = flash_attn.flash_attn_varlen_func(q, k, v, cu, cu, max(lens), max(lens), causal=True)
    err = (got.float() - fa.float()).abs().max().item()
    assert err < 1e-2, err


@pytest.mark.parametrize("H,KV,hd", [(32, 8, 128), (16, 16, 128), (8, 2, 64)])
def test_prefill_attention_kernels_agree_bit_for_bit(cuda, H, KV, hd):
    """max_len is only a host-side bound (it sizes the grid): a bound >= 1024 selects the
    128-query kernel with 32 rows per warp, a tight bound of short prompts the 64-query kernel.
    Per query row both run the same arithmetic, so the outputs are identical."""
    lens = [700, 1, 64, 129, 333]
    q, k, v, cu = _prefill_case(H, KV, lens, hd=hd, seed=11)
    narrow = K.prefill_attention(q, k, v, cu, max(lens), hd ** -0.5)
    wide = K.prefill_attention(q, k, v, cu, 2048, hd ** -0.5)
    assert torch.equal(narrow, wide)
