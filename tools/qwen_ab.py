"""Whole Qwen1.5-MoE layer (60 routed experts top-4 + shared expert as 4 sub-experts, one grouped
launch) timed with CUDA events (L2 flushed) at several token counts; run once per QMOE_* setting
for same-box A/B of kernel paths (e.g. QMOE_CTA_PAIR=0/1)."""
import json, os, statistics, sys
sys.path.insert(0, ".")
import torch
from paper_2503_09304_b200 import kernels as K

d, F, E, k, S = 2048, 1408, 60, 4, 4
g = torch.Generator(device="cuda").manual_seed(7)
wr = (torch.randn((E + 1, d), device="cuda", generator=g) * d ** -0.5).bfloat16()
gu = (torch.randn((E + S, 2 * F, d), device="cuda", generator=g) * d ** -0.5).bfloat16()
dn = (torch.randn((E + S, d, F), device="cuda", generator=g) * F ** -0.5).bfloat16()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
env = {k_: v for k_, v in os.environ.items() if k_.startswith("QMOE_")}
for T in [int(t) for t in (sys.argv[1] if len(sys.argv) > 1 else "1024,2048,4096,8192,16384").split(",")]:
    x = torch.randn((T, d), device="cuda", generator=g).bfloat16()
    y = torch.empty((T * (k + S), d), dtype=torch.bfloat16, device="cuda")
    act = torch.empty((T * (k + S), F), dtype=torch.bfloat16, device="cuda")
    # the product's choice (moe_block.SparseMoeBlock): shared sub-experts read x directly on the
    # 1-CTA path unless QMOE_SHARED_DIRECT=0
    direct = K.shared_direct_ok(d, F, E + S, T * (k + S))
    ge, xd = (E, x) if direct else (None, None)
    ids, w = K.router(x, wr, k, K.ROUTE_SOFTMAX_TOPK, n_shared=S)
    perm, offsets, xp = K.permute(ids, E + S, x=x, gather_e_end=ge)

    def ffn():
        K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, act_ws=act, x_direct=xd, x_first=E)

    def layer():
        i, w_ = K.router(x, wr, k, K.ROUTE_SOFTMAX_TOPK, n_shared=S)
        p, o, xp_ = K.permute(i, E + S, x=x, gather_e_end=ge)
        K.expert_ffn(K.EXPERT_SWIGLU, xp_, o, p, gu, dn, y, act_ws=act, x_direct=xd, x_first=E)
        K.combine(y, w_, x)

    res = {}
    for name, fn in (("ffn", ffn), ("layer", layer)):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[name] = statistics.median(ts)
    fl = 6.0 * T * (k + S) * d * F
    print(json.dumps({"env": env, "T": T, "path": K.expert_ffn_path(d, F, E + S, T * (k + S)), "ffn_ms": res["ffn"],
                      "layer_ms": res["layer"], "ffn_tflops": fl / res["ffn"] / 1e9,
                      "layer_tflops": fl / res["layer"] / 1e9}), flush=True)
