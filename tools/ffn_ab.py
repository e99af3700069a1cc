"""Eager A/B timing of the grouped expert FFN alone (median of 10 launches, L2 flushed before each)
for one layer shape over a list of token counts; run once per QMOE_* setting and compare.
    SHAPE=qwen python tools/ffn_ab.py 2048 8192"""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_09304_b200 import kernels as K  # noqa: E402

SHAPES = {"mixtral": (4096, 14336, 8, 2), "qwen": (2048, 1408, 60, 4), "qwen_shared": (2048, 5632, 1, 1)}
d, F, E, k = SHAPES[os.environ.get("SHAPE", "mixtral")]
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(7)
wr = (torch.randn((E, d), device=dev, generator=g) * d ** -0.5).bfloat16()
gu = (torch.randn((E, 2 * F, d), device=dev, generator=g) * d ** -0.5).bfloat16()
dn = (torch.randn((E, d, F), device=dev, generator=g) * F ** -0.5).bfloat16()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
for T in [int(t) for t in sys.argv[1:]]:
    x = torch.randn((T, d), device=dev, generator=g).bfloat16()
    y = torch.empty((T * k, d), dtype=torch.bfloat16, device=dev)
    act = torch.empty((T * k, F), dtype=torch.bfloat16, device=dev)
    ids, w = K.router(x, wr, k, K.ROUTE_SOFTMAX_TOPK)
    perm, offsets, xp = K.permute(ids, E, x=x)
    for _ in range(3):
        K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, act_ws=act)
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, act_ws=act)
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in ts)
    print(f"{os.environ.get('SHAPE', 'mixtral')} T={T} path {K.expert_ffn_path(d, F, E, T * k)} ffn {ms:.3f} ms "
          f"{6.0 * T * k * d * F / ms / 1e9:.0f} TFLOP/s", flush=True)
