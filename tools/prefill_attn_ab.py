"""Prefill attention alone (CUDA events, median of 20): qmoe_prefill_attention vs flash-attn's
varlen kernel on the same packed qkv views, Mixtral (32 q / 8 kv heads) and Qwen (16 / 16) heads,
hd 128, batches of equal-length prompts.  Prints one JSON line per case."""
import json, statistics, sys
sys.path.insert(0, ".")
import torch
from flash_attn import flash_attn_varlen_func
from paper_2503_09304_b200 import kernels as K

def timeit(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)

for name, H, KV in (("mixtral", 32, 8), ("qwen", 16, 16)):
    for B, n in ((1, 512), (8, 256), (4, 1024), (2, 2048), (1, 4096), (16, 64)):
        hd = 128
        T = B * n
        qkv = torch.randn((T, (H + 2 * KV) * hd), device="cuda").bfloat16()
        q = qkv[:, : H * hd].view(T, H, hd)
        k = qkv[:, H * hd:(H + KV) * hd].view(T, KV, hd)
        v = qkv[:, (H + KV) * hd:].view(T, KV, hd)
        cu = torch.arange(0, T + 1, n, dtype=torch.int32, device="cuda")
        ours = timeit(lambda: K.prefill_attention(q, k, v, cu, n, hd ** -0.5))
        fa = timeit(lambda: flash_attn_varlen_func(q, k, v, cu, cu, n, n, causal=True))
        flops = 4 * B * H * hd * n * (n + 1) / 2  # causal QK^T + PV
        print(json.dumps({"shape": name, "B": B, "len": n, "ours_ms": round(ours, 4), "flash_attn_ms": round(fa, 4),
                          "ours_tflops": round(flops / ours / 1e9, 1), "fa_tflops": round(flops / fa / 1e9, 1)}),
              flush=True)
