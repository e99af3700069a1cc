"""Mixtral/Qwen-shaped decoder plugin on the B200: fused RMSNorm / RoPE kernels against torch,
and a small 2-layer decoder driven through the engine (paged KV, flash-attn, libqmoe MoE block)
against an independent pure-torch implementation (full causal attention, dense per-token MoE)."""

from dataclasses import replace

import pytest
import torch

from paper_2503_09304_b200 import kernels as K
from paper_2503_09304_b200.core import Phase, Priority, SchedulerDirective, batch_form, sequence_new
from paper_2503_09304_b200.engine import InferenceEngine, VirtualClock
from paper_2503_09304_b200.kvcache import UnifiedDynamicCache
from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, QWEN15_MOE_A27B, DecoderMoEModel, rms_norm

pytestmark = pytest.mark.gpu


def test_fused_rmsnorm_matches_torch(cuda):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn((37, 4096), device="cuda", generator=g).bfloat16()
    a = torch.randn((37, 4096), device="cuda", generator=g).bfloat16()
    w = (1 + 0.1 * torch.randn(4096, device="cuda", generator=g)).bfloat16()
    out = K.rmsnorm(x, w, 1e-5)
    ref = rms_norm(x, w, 1e-5)
    assert ((out.float() - ref.float()).abs() <= ref.float().abs() * 2 ** -7 + 1e-6).all()
    out2, s = K.rmsnorm(x, w, 1e-5, add=a)
    assert torch.equal(s, x + a)
    ref2 = rms_norm(x + a, w, 1e-5)
    assert ((out2.float() - ref2.float()).abs() <= ref2.float().abs() * 2 ** -7 + 1e-6).all()


def test_fused_rope_matches_torch(cuda):
    m = DecoderMoEModel.__new__(DecoderMoEModel)  # only the RoPE tables / reference helper
    cfg = MIXTRAL_8X7B
    m.cfg = cfg
    hd = cfg.head_dim
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, device="cuda", dtype=torch.float32) / hd))
    ang = torch.arange(512, device="cuda", dtype=torch.float32)[:, None] * inv[None, :]
    emb = torch.cat([ang, ang], -1)
    m._cos, m._sin = emb.cos().contiguous(), emb.sin().contiguous()
    T, H, KV = 19, cfg.n_heads, cfg.n_kv_heads
    qkv = torch.randn((T, (H + 2 * KV) * hd), device="cuda").bfloat16()
    pos = torch.randint(0, 500, (T,), device="cuda")
    q_ref = m._rope(qkv[:, : H * hd].reshape(T, H, hd), pos)
    k_ref = m._rope(qkv[:, H * hd:(H + KV) * hd].reshape(T, KV, hd), pos)
    v_before = qkv[:, (H + KV) * hd:].clone()
    K.rope_(qkv, pos, m._cos, m._sin, H, KV, hd)
    for got, ref in ((qkv[:, : H * hd].reshape(T, H, hd), q_ref), (qkv[:, H * hd:(H + KV) * hd].reshape(T, KV, hd), k_ref)):
        assert ((got.float() - ref.float()).abs() <= ref.float().abs() * 2 ** -7 + 1e-3).all()
    assert torch.equal(qkv[:, (H + KV) * hd:], v_before)


SMALL = replace(MIXTRAL_8X7B, name="mixtral-small", num_layers=2, hidden_dim=512, ffn_dim=1024, n_heads=8,
                n_kv_heads=2, head_dim=64, vocab_size=1000, max_position=1024)


def torch_reference_hidden(m: DecoderMoEModel, tokens: list[int]) -> torch.Tensor:
    """Final-layer hidden state of the last token, recomputing everything without a cache."""
    cfg = m.cfg
    H, KV, hd = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim
    h = m.embedding[torch.tensor(tokens, device="cuda")]
    T = h.shape[0]
    pos = torch.arange(T, device="cuda")
    for L in m.layers:
        x = rms_norm(h, L.ln1, cfg.rms_eps)
        qkv = x @ L.w_qkv.T
        q = m._rope(qkv[:, : H * hd].reshape(T, H, hd), pos)
        k = m._rope(qkv[:, H * hd:(H + KV) * hd].reshape(T, KV, hd), pos)
        v = qkv[:, (H + KV) * hd:].reshape(T, KV, hd)
        rep = H // KV
        att = torch.nn.functional.scaled_dot_product_attention(
            q.transpose(0, 1).float(), k.repeat_interleave(rep, 1).transpose(0, 1).float(),
            v.repeat_interleave(rep, 1).transpose(0, 1).float(), is_causal=True).transpose(0, 1)
        h2 = h + (att.reshape(T, H * hd).to(h.dtype) @ L.w_o.T)
        xm = rms_norm(h2, L.ln2, cfg.rms_eps)
        logits = xm.float() @ L.w_router.float().T
        out = h2.float().clone()
        for t in range(T):
            sel = sorted(torch.topk(logits[t], cfg.top_k).indices.tolist())
            wts = torch.softmax(logits[t, sel], 0)
            for j, e in enumerate(sel):
                gu = L.gate_up[e].float() @ xm[t].float()
                a = (torch.nn.functional.silu(gu[: cfg.ffn_dim]) * gu[cfg.ffn_dim:]).bfloat16().float()
                out[t] += wts[j] * (L.down[e].float() @ a)
        h = out.to(h.dtype)
    return h[-1].float()


def test_small_mixtral_decoder_prefill_and_decode_match_torch(cuda):
    m = DecoderMoEModel(SMALL, seed=3)
    cache = UnifiedDynamicCache(SMALL.num_layers, m.kv_row_shape(), m.kv_dtype, m.device, m.kv_entry_bytes(),
                                **m.kv_page_kwargs)
    eng = InferenceEngine(m, cache, VirtualClock(), max_batch_size=8)
    prompts = [[5, 17, 99, 3], [250, 7, 7, 8, 9, 10, 11], [42]]
    seqs = []
    for i, p in enumerate(prompts):
        s = sequence_new(p, Priority.BEST_EFFORT, 8, 0.0, seq_id=i)
        s.cache_handle = i
        cache.register(i)
        seqs.append(s)
    captured = {}
    orig = m.emit_batch

    def capture(h, rows):
        captured["h"] = h.index_select(0, torch.tensor(rows, device="cuda")).float()
        return orig(h, rows)

    m.emit_batch = capture
    cont = lambda r: SchedulerDirective.CONTINUE  # noqa: E731
    out = eng.execute(batch_form(seqs, Phase.PREFILL, 8, eng.next_batch_id()), seqs, cont)
    for step in range(3):
        for i, s in enumerate(seqs):
            ref = torch_reference_hidden(m, s.prompt + s.generated)
            rel = ((captured["h"][i] - ref).norm() / ref.norm()).item()
            print(f"decoder step {step} seq {i}: rel {rel:.3e}")
            assert rel < 1e-2, (step, i, rel)
        for s in seqs:
            s.generated.append(out.tokens[s.id])
            if s.phase is Phase.PREFILL:
                s.advance_phase(Phase.DECODE)
        out = eng.execute(batch_form(seqs, Phase.DECODE, 8, eng.next_batch_id()), seqs, cont)


def test_qwen_shape_block_runs_with_shared_expert(cuda):
    cfg = replace(QWEN15_MOE_A27B, num_layers=1, vocab_size=1000)
    m = DecoderMoEModel(cfg, seed=1)
    """The shared expert runs inside the grouped launch as 4 sub-experts (ids 60..63, weight
    sigmoid(gate . x)); routing is checked against the oracle (HF norm_topk_prob=False rule, pinned
    in test_hf_parity.py) and the layer against the oracle's SparseMoeBlock restatement."""
    import numpy as np

    from oracle import moe_oracle as om

    T, E, F, Fs = 40, cfg.num_experts, cfg.ffn_dim, cfg.shared_ffn_dim
    x = torch.randn((T, cfg.hidden_dim), device="cuda").bfloat16()
    ids, w = m.route_batch(0, x)
    assert ids.shape == (T, 8)
    assert (ids[:, 4:] == torch.arange(E, E + 4, device="cuda")).all()
    L = m.layers[0]
    xd = x.double().cpu().numpy()
    wr = L.w_router.double().cpu().numpy()
    oi, ow = om.route_many_qwen(wr[:E], xd, 4)
    srt = -np.sort(-(xd @ wr[:E].T), axis=1)
    safe = (srt[:, 3] - srt[:, 4]) > 1e-3
    assert np.array_equal(ids[:, :4].cpu().numpy()[safe], oi[safe])
    np.testing.assert_allclose(w[:, :4].cpu().numpy()[safe], ow[safe], rtol=0, atol=1e-5)
    gate = 1 / (1 + np.exp(-(xd @ wr[E])))
    np.testing.assert_allclose(w[:, 4:].cpu().numpy(), np.repeat(gate[:, None], 4, 1), rtol=1e-5, atol=1e-6)
    y, cursor = m.new_expert_state(T)
    perm, offsets, xp = m.permute(ids, cursor, x)
    m.run_experts(0, xp, offsets, perm, y, 0, m.config.num_experts)
    out = m.combine_batch(0, y, w, x, x)
    # oracle layer on the bf16 weights (shared expert in HF form: gate/up [Fs, d], down [d, Fs])
    gu = L.gate_up.double().cpu().numpy()
    dn = L.down.double().cpu().numpy()
    sgu = np.concatenate([gu[E:, :F].reshape(Fs, -1), gu[E:, F:].reshape(Fs, -1)], 0)
    sdn = np.concatenate(list(dn[E:]), 1)
    _, _, ref = om.sparse_moe_block(wr[:E], gu[:E], dn[:E], xd, 4, qwen=True, shared_gate_up=sgu, shared_down=sdn,
                                    shared_gate=wr[E])
    ref = ref + xd
    got = out.double().cpu().numpy()
    rel = np.linalg.norm(got[safe] - ref[safe]) / np.linalg.norm(ref[safe])
    print(f"qwen block rel {rel:.3e} ({int(safe.sum())}/{T} rows outside the top-k tie band)")
    assert rel < 1e-2, rel
