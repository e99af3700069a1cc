"""Kernel parity on the B200: every libqmoe kernel against the oracle / golden fixtures.

Bars (written in each test): expert ids, queue order (perm/offsets) and combine in f64 are
bit-exact; f64 weights/outputs within 1e-12; f32 within 1e-5; bf16 within 1e-2 relative of a
torch fp32 reference applied to the same bf16-rounded inputs.
"""

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import moe_oracle as om
from paper_2503_09304_b200 import kernels as K

pytestmark = pytest.mark.gpu

TINY = om.ToyConfig(num_layers=2, hidden_dim=256, num_experts=8, top_k=2, vocab_size=256, seed=0)


@pytest.fixture(scope="module")
def tiny():
    return np.load(GOLDEN / "tiny_layer.npz")


@pytest.fixture(scope="module")
def params():
    return om.ToyParams(TINY)


def dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(dtype).cuda()


# --------------------------------------------------------------------------------- router

@pytest.mark.parametrize("layer", [0, 1])
def test_router_f64_bit_exact_ids(cuda, tiny, params, layer):
    ids, w = K.router(dev(tiny[f"H{layer}"]), dev(params.w_router[layer]), 2)
    assert np.array_equal(ids.cpu().numpy(), tiny[f"ids{layer}"])
    np.testing.assert_allclose(w.cpu().numpy(), tiny[f"w{layer}"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("layer", [0, 1])
def test_router_f32_ids_and_weights(cuda, tiny, params, layer):
    ids, w = K.router(dev(tiny[f"H{layer}"], torch.float32), dev(params.w_router[layer], torch.float32), 2)
    assert np.array_equal(ids.cpu().numpy(), tiny[f"ids{layer}"])
    np.testing.assert_allclose(w.cpu().numpy(), tiny[f"w{layer}"], rtol=0, atol=1e-5)


def test_router_tie_break_prefers_lower_id(cuda):
    # logits [0.1, 0.9, 0.5, 0.5] and [9, 0, 3.5, .1, .2, 3.5] (reference tests/test_model.py:67-73)
    for scores, want in (([0.1, 0.9, 0.5, 0.5], [1, 2]), ([9.0, 0.0, 3.5, 0.1, 0.2, 3.5], [0, 2])):
        E = len(scores)
        wr = torch.tensor(scores, dtype=torch.float64).reshape(E, 1).cuda()
        x = torch.ones((3, 1), dtype=torch.float64).cuda()
        ids, _ = K.router(x, wr, 2)
        assert ids.cpu().tolist() == [want] * 3


def test_router_k_equals_e(cuda):
    rng = np.random.default_rng(1)
    x, wr = rng.standard_normal((5, 4)), rng.standard_normal((4, 4))
    ids, w = K.router(dev(x), dev(wr), 4)
    assert ids.cpu().tolist() == [[0, 1, 2, 3]] * 5
    np.testing.assert_allclose(w.sum(1).cpu().numpy(), 1.0, atol=1e-12)


@pytest.mark.parametrize("T,d,E,k,qwen", [(1, 4096, 8, 2, 0), (32, 4096, 8, 2, 0), (3000, 4096, 8, 2, 0),
                                          (700, 2048, 60, 4, 0), (4100, 2048, 60, 4, 1), (2000, 1024, 16, 2, 0),
                                          (33, 2048, 60, 4, 1), (300, 512, 5, 2, 0),
                                          (512, 1024, 24, 3, 0), (8192, 4096, 8, 2, 0), (8192, 2048, 60, 4, 1),
                                          (2500, 1024, 16, 2, 0), (2049, 2048, 24, 3, 0), (6150, 4096, 7, 2, 0),
                                          (64, 2048, 60, 4, 1), (17, 4096, 8, 2, 0), (48, 1024, 16, 2, 0),
                                          (5, 512, 24, 3, 0), (4500, 1024, 24, 3, 0), (4097, 3072, 40, 4, 1),
                                          (16384, 4096, 8, 2, 0)])
def test_router_bf16_against_oracle_on_same_inputs(cuda, T, d, E, k, qwen):
    """T <= 64 bf16 runs the decode cluster kernel (router_decode_kernel), T >= 4096 the tcgen05
    kernel (router_tc_kernel, d split over a cluster), 256 <= T < 4096 the mma.sync kernels
    (register-streamed or cp.async-staged), the rest the SIMT one."""
    g = torch.Generator().manual_seed(T)
    x = torch.randn((T, d), generator=g).bfloat16()
    wr = (torch.randn((E, d), generator=g) / d ** 0.5).bfloat16()
    mode = K.ROUTE_SOFTMAX_TOPK if qwen else K.ROUTE_TOPK_SOFTMAX
    ids, w, logits = K.router(x.cuda(), wr.cuda(), k, mode, want_logits=True)
    ref_logits = x.double() @ wr.double().T
    np.testing.assert_allclose(logits.cpu().double().numpy(), ref_logits.numpy(), rtol=0, atol=2e-4)
    # ids bit-exact wherever the k-th/(k+1)-th logit margin exceeds the fp32 accumulation error
    route = om.route_many_qwen if qwen else om.route_many
    oi, ow = route(wr.double().numpy(), x.double().numpy(), k)
    srt = np.sort(ref_logits.numpy(), axis=1)[:, ::-1]
    band = 1e-3  # > 5x the fp32 logit error bound asserted above
    safe = (srt[:, k - 1] - srt[:, k]) > band
    got = ids.cpu().numpy()
    near = int((~safe).sum())
    print(f"router T={T} E={E} k={k}: {near} near-tie rows of {T} (k-th/(k+1)-th margin <= {band}), "
          f"{int((got[~safe] != oi[~safe]).any(1).sum())} of them pick another set")
    assert safe.mean() > 0.95
    assert np.array_equal(got[safe], oi[safe])
    np.testing.assert_allclose(w.cpu().numpy()[safe], ow[safe], rtol=0, atol=1e-4)
    # every near-tie row: the picked set is a valid top-k within the tie band (each chosen logit is
    # within band of the exact k-th largest), ascending, no duplicates
    kth = srt[:, k - 1]
    chosen = np.take_along_axis(ref_logits.numpy(), got.astype(np.int64), 1)
    assert np.all(chosen[~safe] >= kth[~safe, None] - band)
    assert np.all(np.diff(got, axis=1) > 0)


@pytest.mark.parametrize("T,d,E,k,qwen,ns", [(8192, 4096, 8, 2, 0, 0), (8192, 2048, 60, 4, 1, 4), (4500, 1024, 24, 3, 0, 0),
                                             (5000, 2048, 60, 4, 1, 0), (4097, 4096, 7, 2, 0, 0),
                                             (6000, 2048, 16, 2, 1, 2), (300, 4096, 8, 2, 0, 0),
                                             (2000, 2048, 60, 4, 1, 4), (2500, 1024, 16, 2, 0, 0),
                                             (2049, 2048, 24, 3, 1, 0), (1000, 4096, 8, 2, 0, 0)])
def test_router_group_selection_is_select_token_bit_for_bit(cuda, T, d, E, k, qwen, ns):
    """The bf16 prefill routers' selection (select_group: G lanes per token, in the tcgen05 kernel
    from 3-4k tokens and the register-streamed mma.sync kernels below) against the per-warp
    select_token of the f32 SIMT router run on the very same logits (x = the bf16 kernel's fp32
    logits, W_router = identity, so every f32 logit is exact): ids and weights bit-identical, the
    shared gate slots included."""
    g = torch.Generator().manual_seed(T + E)
    rows = E + (1 if ns else 0)
    x = torch.randn((T, d), generator=g).bfloat16().cuda()
    wr = (torch.randn((rows, d), generator=g) / d ** 0.5).bfloat16().cuda()
    mode = K.ROUTE_SOFTMAX_TOPK if qwen else K.ROUTE_TOPK_SOFTMAX
    ids, w, logits = K.router(x, wr, k, mode, want_logits=True, n_shared=ns)
    eye = torch.eye(rows, dtype=torch.float32, device="cuda")
    ids2, w2, logits2 = K.router(logits.contiguous(), eye, k, mode, want_logits=True, n_shared=ns)
    assert torch.equal(logits2, logits)
    assert torch.equal(ids, ids2)
    assert torch.equal(w, w2)


def test_router_qwen_softmax_topk_mode(cuda):
    rng = np.random.default_rng(3)
    x, wr = rng.standard_normal((257, 64)), rng.standard_normal((60, 64)) / 8
    ids, w = K.router(dev(x), dev(wr), 4, mode=K.ROUTE_SOFTMAX_TOPK)
    oi, ow = om.route_many_qwen(wr, x, 4)
    assert np.array_equal(ids.cpu().numpy(), oi)
    np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=0, atol=1e-12)


# --------------------------------------------------------------------------------- permute

@pytest.mark.parametrize("layer", [0, 1])
def test_permute_matches_reference_queue_order(cuda, tiny, layer):
    ids = dev(tiny[f"ids{layer}"], torch.int32)
    H = dev(tiny[f"H{layer}"])
    perm, offsets, xp = K.permute(ids, 8, x=H)
    R = int(offsets[-1])
    assert np.array_equal(offsets.cpu().numpy(), tiny[f"offsets{layer}"])
    assert np.array_equal(perm[:R].cpu().numpy(), tiny[f"perm{layer}"])
    assert torch.equal(xp[:R], H[perm[:R].long() // 2])


@pytest.mark.parametrize("layer", [0, 1])
def test_permute_resume_cursor_matches_reference(cuda, tiny, layer):
    ids = dev(tiny[f"ids{layer}"], torch.int32)
    cur = dev(tiny[f"cursor{layer}"], torch.int32)
    perm, offsets, _ = K.permute(ids, 8, cursor=cur)
    R = int(offsets[-1])
    assert np.array_equal(perm[:R].cpu().numpy(), tiny[f"perm_resume{layer}"])
    assert int(offsets[4]) == 0


@pytest.mark.parametrize("T,k,E", [(1, 2, 8), (37, 2, 8), (5000, 2, 8), (20000, 4, 60), (65536, 2, 8)])
def test_permute_random_against_oracle(cuda, T, k, E):
    rng = np.random.default_rng(T)
    ids = np.sort(np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]), axis=1)
    cursor = rng.integers(0, E + 1, size=T)
    for cur in (None, cursor):
        perm, offsets, _ = K.permute(dev(ids, torch.int32), E, cursor=None if cur is None else dev(cur, torch.int32))
        op, oo = om.permute(ids, cur, E)
        assert np.array_equal(offsets.cpu().numpy(), oo)
        assert np.array_equal(perm[: oo[-1]].cpu().numpy(), op)


def test_permute_empty_batch(cuda):
    perm, offsets, _ = K.permute(torch.empty((0, 2), dtype=torch.int32, device="cuda"), 8)
    assert offsets.cpu().tolist() == [0] * 9


# --------------------------------------------------------------------------------- experts

def _tiny_expert_inputs(tiny, params, layer, dtype):
    ids = dev(tiny[f"ids{layer}"], torch.int32)
    H = dev(tiny[f"H{layer}"], dtype)
    perm, offsets, xp = K.permute(ids, 8, x=H)
    A = dev(params.expert_weight[layer], dtype)
    b = dev(params.expert_bias[layer], dtype)
    return perm, offsets, xp, A, b, H.shape[0]


@pytest.mark.parametrize("layer", [0, 1])
def test_expert_tanh_f64_matches_reference(cuda, tiny, params, layer):
    perm, offsets, xp, A, b, T = _tiny_expert_inputs(tiny, params, layer, torch.float64)
    y = torch.zeros((T * 2, 256), dtype=torch.float64, device="cuda")
    K.expert_ffn(K.EXPERT_TANH_AFFINE, xp, offsets, perm, A, b, y)
    np.testing.assert_allclose(y.cpu().numpy(), tiny[f"Y{layer}"], rtol=0, atol=1e-12)


def test_expert_tanh_f32(cuda, tiny, params):
    perm, offsets, xp, A, b, T = _tiny_expert_inputs(tiny, params, 0, torch.float32)
    y = torch.zeros((T * 2, 256), dtype=torch.float32, device="cuda")
    K.expert_ffn(K.EXPERT_TANH_AFFINE, xp, offsets, perm, A, b, y)
    np.testing.assert_allclose(y.cpu().numpy(), tiny["Y0"], rtol=0, atol=1e-5)


def test_expert_tanh_bf16_tcgen05(cuda, tiny, params):
    perm, offsets, xp, A, b, T = _tiny_expert_inputs(tiny, params, 1, torch.bfloat16)
    y = torch.zeros((T * 2, 256), dtype=torch.bfloat16, device="cuda")
    K.expert_ffn(K.EXPERT_TANH_AFFINE, xp, offsets, perm, A, b, y)
    # torch fp32 reference on the same bf16-rounded operands
    ids = tiny["ids1"]
    ref = torch.zeros((T * 2, 256), dtype=torch.float32)
    Hb, Ab, bb = xp.float().cpu(), A.float().cpu(), b.float().cpu()
    pc, oc = perm.cpu().long(), offsets.cpu().long()
    for e in range(8):
        rows = pc[oc[e]:oc[e + 1]]
        ref[rows] = torch.tanh(Hb[oc[e]:oc[e + 1]] @ Ab[e].T + bb[e])
    err = (y.float().cpu() - ref).abs().max().item()
    assert err < 1e-2, err
    assert ids.shape[0] == T


def _swiglu_problem(T, d, F, E, k, seed, dtype=torch.bfloat16):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn((T, d), generator=g)
    wr = torch.randn((E, d), generator=g) / d ** 0.5
    gate_up = torch.randn((E, 2 * F, d), generator=g) / d ** 0.5
    down = torch.randn((E, d, F), generator=g) / F ** 0.5
    return [t.to(dtype).cuda() for t in (x, wr, gate_up, down)]


def _swiglu_ref(xp, offsets, perm, gate_up, down, T, k, e_hi=None):
    xp32, gu, dn = xp.float(), gate_up.float(), down.float()
    F = gu.shape[1] // 2
    ref = torch.zeros((T * k, xp.shape[1]), dtype=torch.float32, device=xp.device)
    oc = offsets.cpu().long().tolist()
    E = gu.shape[0] if e_hi is None else e_hi
    for e in range(E):
        a, b_ = oc[e], oc[e + 1]
        if a == b_:
            continue
        h = xp32[a:b_] @ gu[e].T
        act = (torch.nn.functional.silu(h[:, :F]) * h[:, F:]).bfloat16().float()
        ref[perm[a:b_].long()] = act @ dn[e].T
    return ref


@pytest.mark.parametrize("T,d,F,E,k", [(64, 1024, 2048, 8, 2), (1000, 512, 1408, 60, 4), (8, 4096, 14336, 8, 2),
                                       (2048, 4096, 14336, 8, 2), (1, 4096, 14336, 8, 2), (64, 2048, 1408, 60, 4),
                                       (256, 1024, 1024, 2, 1), (3, 512, 1024, 16, 2), (128, 2048, 1408, 60, 4),
                                       (32, 4096, 14336, 8, 2), (200, 768, 640, 5, 2), (40, 512, 576, 4, 2),
                                       (300, 384, 192, 3, 1)])
def test_expert_swiglu_bf16_tcgen05_against_torch_fp32(cuda, T, d, F, E, k):
    """T*k <= 512 routed rows take the swap-AB single-launch kernel (expert_swap.cu, incl. multi
    token tiles per expert, empty experts, K-split down), larger batches the 128/256-row tiles."""
    x, wr, gate_up, down = _swiglu_problem(T, d, F, E, k, seed=T + d)
    ids, w = K.router(x, wr, k)
    perm, offsets, xp = K.permute(ids, E, x=x)
    y = torch.zeros((T * k, d), dtype=torch.bfloat16, device="cuda")
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gate_up, down, y)
    ref = _swiglu_ref(xp, offsets, perm, gate_up, down, T, k)
    rel = (y.float() - ref).norm() / ref.norm()
    assert rel.item() < 1e-2, rel.item()
    err = (y.float() - ref).abs().max().item()
    assert err < 0.05 * ref.abs().max().item()


def test_expert_swiglu_f32_simt_against_oracle(cuda):
    x, wr, gate_up, down = _swiglu_problem(100, 64, 128, 8, 2, seed=5, dtype=torch.float32)
    ids, w = K.router(x, wr, 2)
    perm, offsets, xp = K.permute(ids, 8, x=x)
    y = torch.zeros((200, 64), dtype=torch.float32, device="cuda")
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gate_up, down, y)
    ref = np.zeros((200, 64))
    pc, oc = perm.cpu().numpy(), offsets.cpu().numpy()
    for e in range(8):
        ref[pc[oc[e]:oc[e + 1]]] = om.expert_swiglu(gate_up[e].double().cpu().numpy(), down[e].double().cpu().numpy(),
                                                    xp[oc[e]:oc[e + 1]].double().cpu().numpy())
    np.testing.assert_allclose(y.cpu().numpy(), ref, rtol=0, atol=1e-5)


@pytest.mark.parametrize("dtype,T,d,F", [(torch.float64, 300, 128, 256), (torch.bfloat16, 300, 128, 256),
                                         (torch.bfloat16, 100, 1024, 4096)])
def test_expert_range_and_cursor_out(cuda, dtype, T, d, F):
    """Launch experts [0, 3) then [3, 8): union equals one full launch; cursor_out == e_end.
    (T=100 bf16 exercises the split-K down projection with its deterministic reduce.)"""
    x, wr, gate_up, down = _swiglu_problem(T, d, F, 8, 2, seed=11, dtype=dtype)
    ids, w = K.router(x, wr, 2)
    perm, offsets, xp = K.permute(ids, 8, x=x)
    full = torch.zeros((2 * T, d), dtype=dtype, device="cuda")
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gate_up, down, full)
    part = torch.zeros_like(full)
    cur = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gate_up, down, part, e_begin=0, e_end=3, cursor_out=cur)
    assert int(cur) == 3
    oc = offsets.cpu().tolist()
    done = perm[: oc[3]].long()
    assert torch.equal(part[done], full[done])
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gate_up, down, part, e_begin=3, e_end=8, cursor_out=cur)
    assert int(cur) == 8
    assert torch.equal(part, full)


@pytest.mark.parametrize("dtype,T,d,F", [(torch.float32, 4096, 256, 512), (torch.bfloat16, 4096, 256, 512),
                                         (torch.bfloat16, 200, 256, 512), (torch.bfloat16, 16, 1024, 4096)])
def test_preempt_flag_stops_at_expert_boundary(cuda, dtype, T, d, F):
    """A raised device flag (s = 3) stops the launch at the first expert boundary >= 3:
    cursor_out = 3, experts 0..2 are complete and correct, later experts are left for the
    resume launch, which completes the layer bit-identically.  (T <= 256: the swap-AB kernel,
    whose down units must run for exactly the experts below the stop.)"""
    x, wr, gate_up, down = _swiglu_problem(T, d, F, 8, 2, seed=3, dtype=dtype)
    ids, w = K.router(x, wr, 2)
    perm, offsets, xp = K.permute(ids, 8, x=x)
    full = torch.zeros((2 * T, d), dtype=dtype, device="cuda")
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gate_up, down, full)
    # raised before launch with s = 3: experts 0..2 must complete, nothing later starts
    flag = torch.full((1,), 3, dtype=torch.int32, device="cuda")
    cur = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    y = torch.zeros_like(full)
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gate_up, down, y, preempt_flag=flag, cursor_out=cur)
    c = int(cur)
    oc = offsets.cpu().tolist()
    # the first expert boundary >= 3 that exists (an expert without rows has no boundary)
    assert c == next((e for e in range(3, 8) if oc[e + 1] > oc[e]), 8)
    assert torch.equal(y[perm[: oc[c]].long()], full[perm[: oc[c]].long()])
    # resume from the cursor with the flag lowered completes the layer bit-identically
    flag.zero_()
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gate_up, down, y, e_begin=c, cursor_out=cur)
    assert int(cur) == 8
    assert torch.equal(y, full)


# --------------------------------------------------------------------------------- combine & state

@pytest.mark.parametrize("layer", [0, 1])
def test_combine_f64_bit_exact(cuda, tiny, layer):
    out = K.combine(dev(tiny[f"Y{layer}"]), dev(tiny[f"w{layer}"]), dev(tiny[f"H{layer}"]))
    assert np.array_equal(out.cpu().numpy(), tiny[f"out{layer}"])


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_combine_bf16(cuda, k):
    g = torch.Generator().manual_seed(k)
    T, d = 333, 2048
    y = torch.randn((T * k, d), generator=g).bfloat16()
    w = torch.rand((T, k), generator=g)
    res = torch.randn((T, d), generator=g).bfloat16()
    out = K.combine(y.cuda(), w.cuda(), res.cuda())
    ref = res.float() + (w[:, :, None] * y.float().reshape(T, k, d)).sum(1)
    # bf16 output: one rounding of the fp32 sum, |err| <= 2^-8 |ref| (+ tiny slack)
    assert ((out.float().cpu() - ref).abs() <= ref.abs() * 2 ** -8 + 1e-3).all()
    out2 = K.combine(y.cuda(), w.cuda(), None)
    ref2 = (w[:, :, None] * y.float().reshape(T, k, d)).sum(1)
    assert ((out2.float().cpu() - ref2).abs() <= ref2.abs() * 2 ** -8 + 1e-3).all()


def test_gather_rows_and_kv_round_trip(cuda):
    src = torch.randn((100, 48), dtype=torch.float64, device="cuda")
    idx = torch.tensor([5, 0, 99, 5, 17], dtype=torch.int32, device="cuda")
    assert torch.equal(K.gather_rows(src, idx), src[idx.long()])
    pool = torch.zeros((64, 2, 48), dtype=torch.float64, device="cuda")
    slots = torch.tensor([7, 3, 40], dtype=torch.int32, device="cuda")
    rows = torch.randn((3, 2, 48), dtype=torch.float64, device="cuda")
    K.kv_append(pool, slots, rows)
    out = torch.empty_like(rows)
    K.kv_gather(pool, slots, out)
    assert torch.equal(out, rows)


def test_cursor_advance(cuda):
    cur = torch.tensor([0, 3, 6, 8], dtype=torch.int32, device="cuda")
    stop = torch.tensor([5], dtype=torch.int32, device="cuda")
    K.cursor_advance(cur, stop)
    assert cur.cpu().tolist() == [5, 5, 6, 8]


_SPLIT_PROBE = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2503_09304_b200 import kernels as K
from oracle import moe_oracle as om
bad = 0
for T, d, E, k, qwen in ((700, 1024, 8, 2, 0), (1000, 2048, 61, 4, 1), (513, 4096, 24, 3, 0)):
    g = torch.Generator().manual_seed(T)
    x = torch.randn((T, d), generator=g).bfloat16()
    wr = (torch.randn((E, d), generator=g) / d ** 0.5).bfloat16()
    mode = K.ROUTE_SOFTMAX_TOPK if qwen else K.ROUTE_TOPK_SOFTMAX
    ids, w, lg = K.router(x.cuda(), wr.cuda(), k, mode, want_logits=True)
    ref = x.double() @ wr.double().T
    err = float((lg.cpu().double() - ref).abs().max())
    oi, ow = (om.route_many_qwen if qwen else om.route_many)(wr.double().numpy(), x.double().numpy(), k)
    srt = np.sort(ref.numpy(), axis=1)[:, ::-1]
    safe = (srt[:, k - 1] - srt[:, k]) > 1e-3
    bad += int(err > 2e-4) + int(not np.array_equal(ids.cpu().numpy()[safe], oi[safe]))
print("BAD", bad)
"""


@pytest.mark.parametrize("split", [1, 2, 4])
def test_router_tcgen05_every_d_split(cuda, split):
    """Every d split of the tcgen05 router (QMOE_ROUTER_TC_S, read once per process, so each runs in
    a fresh interpreter) at every logit-row padding (16 / 32 / 64): fp32 logits within 2e-4 of fp64
    and ids equal to the oracle's outside the tie band."""
    import os
    import pathlib
    import subprocess
    import sys

    root = str(pathlib.Path(__file__).resolve().parents[1])
    env = dict(os.environ, QMOE_ROUTER_TC_MIN="256", QMOE_ROUTER_TC_S=str(split))
    out = subprocess.run([sys.executable, "-c", _SPLIT_PROBE.format(root=root)], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "BAD 0" in out.stdout, out.stdout + out.stderr[-2000:]
