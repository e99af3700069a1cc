"""Every bf16 expert-FFN code path, forced through the QMOE_SWAP_AB / QMOE_SWAP_PAIR / QMOE_CTA_PAIR switches (read
once per process, so each configuration runs in its own interpreter), against the torch fp32
restatement of HF MixtralExperts on the same bf16 inputs: swap-AB with 32/64/128-row token tiles,
the swap-AB CTA pair (256 weight rows x token tiles of <= 256 rows), the 1-CTA 128-row tcgen05
kernel and the CTA-pair 256-row kernel, plus a preempted launch and its resume on each path
(bit-identical to the uninterrupted launch)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys
import torch
sys.path.insert(0, sys.argv[1])
from paper_2503_09304_b200 import kernels as K
res = []
for (T, d, F, E, k) in json.loads(sys.argv[2]):
    g = torch.Generator().manual_seed(T * 7 + E)
    x = torch.randn((T, d), generator=g).bfloat16().cuda()
    wr = (torch.randn((E, d), generator=g) / d ** 0.5).bfloat16().cuda()
    gu = (torch.randn((E, 2 * F, d), generator=g) / d ** 0.5).bfloat16().cuda()
    dn = (torch.randn((E, d, F), generator=g) / F ** 0.5).bfloat16().cuda()
    ids, w = K.router(x, wr, k)
    perm, offsets, xp = K.permute(ids, E, x=x)
    y = torch.zeros((T * k, d), dtype=torch.bfloat16, device="cuda")
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y)
    oc = offsets.cpu().tolist()
    ref = torch.zeros((T * k, d), device="cuda")
    for e in range(E):
        a, b = oc[e], oc[e + 1]
        if a < b:
            h = xp[a:b].float() @ gu[e].float().T
            act = (torch.nn.functional.silu(h[:, :F]) * h[:, F:]).bfloat16().float()
            ref[perm[a:b].long()] = act @ dn[e].float().T
    rel = ((y.float() - ref).norm() / ref.norm()).item()
    # preempt at the first boundary >= 3, resume from the cursor: must equal the full launch
    flag = torch.full((1,), 3, dtype=torch.int32, device="cuda")
    cur = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    y2 = torch.zeros_like(y)
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y2, preempt_flag=flag, cursor_out=cur)
    c = int(cur)
    first = next((e for e in range(3, E) if oc[e + 1] > oc[e]), E)
    done = perm[: oc[c]].long()
    part_ok = c == first and torch.equal(y2[done], y[done])
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y2, e_begin=c)
    # the fused row gather (TMA tile::gather4 from X): identical to the Xp path, also when preempted
    gather = K.gathers_rows(d, F, E, T * k)
    gather_ok = True
    if gather:
        y3 = torch.zeros_like(y)
        K.expert_ffn_gather(x, k, offsets, perm, gu, dn, y3)
        y4 = torch.zeros_like(y)
        flag.fill_(3)
        K.expert_ffn_gather(x, k, offsets, perm, gu, dn, y4, preempt_flag=flag, cursor_out=cur)
        c4 = int(cur)
        K.expert_ffn_gather(x, k, offsets, perm, gu, dn, y4, e_begin=c4)
        gather_ok = torch.equal(y3, y) and torch.equal(y4, y) and c4 == first
    import hashlib
    res.append({"shape": [T, d, F, E, k], "rel": rel, "stop": c, "want_stop": first, "partial_ok": part_ok,
                "resume_identical": torch.equal(y2, y), "gather": gather, "gather_ok": gather_ok,
                "sha": hashlib.sha1(y.view(torch.int16).cpu().numpy().tobytes()).hexdigest()})
print(json.dumps(res))
"""

SHAPES = [(16, 1024, 2048, 8, 2), (160, 1024, 2048, 8, 2), (700, 1024, 2048, 8, 2), (1200, 512, 1408, 8, 2),
          (2500, 512, 1024, 8, 2)]


def _run(env, shapes):
    out = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), json.dumps(shapes)], capture_output=True, text=True,
                         env={**os.environ, **env}, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    for r in res:
        assert r["rel"] < 1e-2, r
        assert r["stop"] == r["want_stop"] and r["partial_ok"], r
        assert r["resume_identical"], r
        assert r["gather_ok"], r
    return res


@pytest.mark.parametrize("env", [{"QMOE_SWAP_AB": "1"}, {"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "1"},
                                 {"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "0", "QMOE_CTA_PAIR": "0"},
                                 {"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "0", "QMOE_CTA_PAIR": "1"}],
                         ids=["swap-ab", "swap-pair", "tc-1cta-single-launch", "tc-pair"])
def test_forced_expert_path(cuda, env):
    _run(env, SHAPES if env.get("QMOE_SWAP_AB") == "1" or env.get("QMOE_SWAP_PAIR") == "1"
         else [s for s in SHAPES if s[0] * s[4] > 512])


@pytest.mark.parametrize("pair", ["0", "1"], ids=["1cta", "cta-pair"])
def test_fused_row_gather_is_used(cuda, pair):
    res = _run({"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "0", "QMOE_CTA_PAIR": pair}, [s for s in SHAPES if s[0] * s[4] > 512])
    assert all(r["gather"] for r in res)


@pytest.mark.parametrize("env", [{"QMOE_SWAP_AB": "1"}, {"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "1"}],
                         ids=["swap-ab", "swap-pair"])
def test_fused_row_gather_swap_ab(cuda, env):
    """The swap-AB kernels' token tiles gathered from X (tile::gather4)."""
    res = _run(env, SHAPES)
    assert all(r["gather"] for r in res)


@pytest.mark.parametrize("pair", ["0", "1"], ids=["1cta", "cta-pair"])
def test_single_launch_equals_two_launches(cuda, pair):
    """The single-launch kernels (expert_fused.cu, 1-CTA and CTA pair) compute every tile exactly
    like the two-launch paths (same tiles, same MMA order, same epilogue): bit-identical outputs."""
    shapes = [s for s in SHAPES if s[0] * s[4] > 512]
    one = _run({"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "0", "QMOE_CTA_PAIR": pair}, shapes)
    two = _run({"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "0", "QMOE_CTA_PAIR": pair, "QMOE_FUSED": "0"}, shapes)
    assert [r["sha"] for r in one] == [r["sha"] for r in two]


RACE = r"""
import json, sys
import torch
sys.path.insert(0, sys.argv[1])
from paper_2503_09304_b200 import kernels as K
out = []
for (T, d, F, E, k, delay) in json.loads(sys.argv[2]):
    g = torch.Generator().manual_seed(T + delay)
    x = torch.randn((T, d), generator=g).bfloat16().cuda()
    wr = (torch.randn((E, d), generator=g) / d ** 0.5).bfloat16().cuda()
    gu = (torch.randn((E, 2 * F, d), generator=g) / d ** 0.5).bfloat16().cuda()
    dn = (torch.randn((E, d, F), generator=g) / F ** 0.5).bfloat16().cuda()
    ids, w = K.router(x, wr, k)
    perm, offsets, xp = K.permute(ids, E, x=x)
    full = torch.zeros((T * k, d), dtype=torch.bfloat16, device="cuda")
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, full)
    oc = offsets.cpu().tolist()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    cur = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    y = torch.zeros_like(full)
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(side):  # raise "stop at the first boundary >= 2" while the GEMM runs
        torch.cuda._sleep(delay)
        flag.fill_(2)
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, preempt_flag=flag, cursor_out=cur)
    torch.cuda.synchronize()
    c = int(cur)
    done = perm[: oc[c]].long()
    ok_prefix = torch.equal(y[done], full[done])
    flag.zero_()
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, e_begin=c, cursor_out=cur)
    out.append({"shape": [T, d, F, E, k], "delay": delay, "stop": c, "path": K.expert_ffn_path(d, F, E, T * k),
                "prefix_ok": ok_prefix, "resume_ok": torch.equal(y, full) and int(cur) == E})
print(json.dumps(out))
"""


ENVS = {"default-paths": ({}, {1, 6}), "token-row-tiles": ({"QMOE_SWAP_PAIR": "0"}, {1, 2}),
        "pair-tiles": ({"QMOE_SWAP_PAIR": "0", "QMOE_CTA_PAIR": "1"}, {1, 3})}


@pytest.mark.parametrize("env", list(ENVS))
def test_preempt_flag_raised_mid_launch(cuda, env):
    """The device flag raised by another stream WHILE the grouped GEMM runs (the serving engine's
    wall-clock path) on every bf16 kernel path: the launch stops at an expert boundary >= 2 (or runs
    to the end if the flag came too late), every expert below the stop is complete and equal to an
    uninterrupted launch, and resuming from the cursor completes the layer bit-identically."""
    cases = [(32, 2048, 4096, 8, 2, d) for d in (0, 20000, 200000)]           # swap-AB
    cases += [(1200, 2048, 4096, 8, 2, d) for d in (0, 20000, 60000)]        # swap-AB pair / fused 128-row tiles
    cases += [(3000, 1024, 1408, 60, 4, d) for d in (0, 10000, 30000)]       # swap-AB pair / fused 256-row pair
    env, paths = ENVS[env]
    out = subprocess.run([sys.executable, "-c", RACE, str(ROOT), json.dumps(cases)], capture_output=True, text=True,
                         env={**os.environ, **env}, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert {r["path"] for r in res} >= paths, res
    assert any(r["stop"] < 8 for r in res), res  # at least some launches really stopped mid-way
    for r in res:
        assert r["stop"] >= 2, r
        assert r["prefix_ok"] and r["resume_ok"], r


def test_all_single_launch_kernels_agree_bit_for_bit(cuda):
    """The tcgen05 kernels differ in tile orientation (weights or tokens on the MMA's M side), CTA
    pairing and tile shape, but accumulate every output over K in the same 64-wide blocks and round
    act and Y identically, so the swap-AB, swap-AB CTA-pair, 1-CTA and CTA-pair kernels return the
    same bits; the kernel-path heuristics therefore never change numerics (only the K-split decode
    and two-launch split-K paths, with their fp32 partials, round differently)."""
    shapes = [s for s in SHAPES if s[0] * s[4] > 512] + [(3000, 1024, 1408, 8, 2)]
    runs = [_run(env, shapes) for env in ({"QMOE_SWAP_AB": "1"}, {"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "1"},
                                          {"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "0", "QMOE_CTA_PAIR": "0"},
                                          {"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "0", "QMOE_CTA_PAIR": "1"})]
    for k in range(len(shapes)):
        assert len({r[k]["sha"] for r in runs}) == 1, [r[k] for r in runs]


def test_swap_pair_wide_last_tile_is_bit_identical(cuda):
    """With QMOE_SP_MERGE=128 the swap-AB pair folds an expert's remainder rows (<= 128 after its
    full 256-row tiles) into its last token tile (one weight pass, two TMEM accumulators, two ring stages per K block):
    outputs, preemption stops and resumes are bit-identical to running the remainder as its own
    tile (QMOE_SP_MERGE=0)."""
    shapes = [(1100, 1024, 2048, 8, 2), (1200, 512, 1408, 8, 2), (2500, 512, 1024, 8, 2), (300, 512, 1024, 2, 2)]
    env = {"QMOE_SWAP_AB": "0", "QMOE_SWAP_PAIR": "1"}
    wide = _run({**env, "QMOE_SP_MERGE": "128"}, shapes)
    narrow = _run({**env, "QMOE_SP_MERGE": "0"}, shapes)
    assert [r["sha"] for r in wide] == [r["sha"] for r in narrow]


def test_shared_sub_experts_read_x_directly_bit_identical(cuda):
    """Qwen-shaped block on the 1-CTA path: the shared sub-experts read their token rows straight
    from x (qmoe_permute_ex gathers only the routed rows, qmoe_expert_ffn_xs) -- the layer output
    is bit-identical to the fully gathered path, with and without a preemption stop and resume."""
    import torch

    from paper_2503_09304_b200 import kernels as K
    from paper_2503_09304_b200.moe_block import SparseMoeBlock

    d, F, E, k, Fs = 1024, 512, 30, 4, 2048
    blk = SparseMoeBlock(d, F, E, k, route_mode=K.ROUTE_SOFTMAX_TOPK, shared_expert_intermediate_size=Fs,
                         device=torch.device("cuda")).init_random(4)
    S = Fs // F
    for T in (2000, 4100):
        x = torch.randn((T, d), device="cuda").bfloat16()
        assert K.expert_ffn_path(d, F, E + S, T * (k + S)) == K.PATH_FUSED_1CTA
        K._SHARED_DIRECT = True
        direct = blk(x)
        K._SHARED_DIRECT = False
        try:
            gathered = blk(x)
        finally:
            K._SHARED_DIRECT = True
        assert torch.equal(direct, gathered), T
        # preempt inside the shared sub-experts, resume from the cursor: same bits
        ids, w = K.router(x, blk._w_router, k, K.ROUTE_SOFTMAX_TOPK, n_shared=S)
        perm, offsets, xp = K.permute(ids, E + S, x=x, gather_e_end=E)
        y_full = torch.zeros((T * (k + S), d), dtype=torch.bfloat16, device="cuda")
        K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, blk._gate_up, blk._down, y_full, x_direct=x, x_first=E)
        y = torch.zeros_like(y_full)
        flag = torch.full((1,), E + 2, dtype=torch.int32, device="cuda")
        cur = torch.zeros(1, dtype=torch.int32, device="cuda")
        K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, blk._gate_up, blk._down, y, preempt_flag=flag, cursor_out=cur,
                     x_direct=x, x_first=E)
        stop = int(cur)
        assert E + 2 <= stop <= E + S
        flag.zero_()
        K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, blk._gate_up, blk._down, y, e_begin=stop, x_direct=x,
                     x_first=E)
        torch.cuda.synchronize()
        assert torch.equal(y, y_full)
