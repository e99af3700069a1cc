"""Minimal driver for `ncu --set full` on the router / permute / combine kernels of one MoE layer
(Mixtral shape by default, SHAPE=qwen for Qwen), T tokens: warm-up, then one layer pass."""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2503_09304_b200 import kernels as K

SHAPES = {"mixtral": (4096, 14336, 8, 2, K.ROUTE_TOPK_SOFTMAX), "qwen": (2048, 1408, 60, 4, K.ROUTE_SOFTMAX_TOPK)}
d, F, E, k, mode = SHAPES[os.environ.get("SHAPE", "mixtral")]
T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = torch.Generator(device="cuda").manual_seed(0)
wr = (torch.randn((E, d), device="cuda", generator=g) * d ** -0.5).bfloat16()
x = torch.randn((T, d), device="cuda", generator=g).bfloat16()
y = torch.randn((T * k, d), device="cuda", generator=g).bfloat16()
for _ in range(3):
    ids, w = K.router(x, wr, k, mode)
    perm, offsets, xp = K.permute(ids, E, x=x)
    out = K.combine(y, w, x)
torch.cuda.synchronize()
