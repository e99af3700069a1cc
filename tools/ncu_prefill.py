"""Minimal driver for an ncu capture of qmoe_prefill_attention: Mixtral heads (32 q / 8 kv, hd 128),
one 4096-token prompt and 8 x 256-token prompts."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2503_09304_b200 import kernels as K

H, KV, hd = 32, 8, 128
for B, n in ((1, 4096), (8, 256)):
    T = B * n
    qkv = torch.randn((T, (H + 2 * KV) * hd), device="cuda").bfloat16()
    q = qkv[:, : H * hd].view(T, H, hd)
    k = qkv[:, H * hd:(H + KV) * hd].view(T, KV, hd)
    v = qkv[:, (H + KV) * hd:].view(T, KV, hd)
    cu = torch.arange(0, T + 1, n, dtype=torch.int32, device="cuda")
    for _ in range(2):
        K.prefill_attention(q, k, v, cu, n, hd ** -0.5)
torch.cuda.synchronize()
