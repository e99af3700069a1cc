"""Minimal driver for an ncu capture of the router at 8192 tokens, Mixtral then Qwen (+shared gate)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2503_09304_b200 import kernels as K

for d, E, k, S, mode in ((4096, 8, 2, 0, K.ROUTE_TOPK_SOFTMAX), (2048, 60, 4, 4, K.ROUTE_SOFTMAX_TOPK)):
    wr = (torch.randn((E + (1 if S else 0), d), device="cuda") / d ** 0.5).bfloat16()
    x = torch.randn((8192, d), device="cuda").bfloat16()
    for _ in range(2):
        K.router(x, wr, k, mode, n_shared=S)
torch.cuda.synchronize()
