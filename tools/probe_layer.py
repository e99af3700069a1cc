"""Quick per-kernel timing of one Mixtral-shaped MoE layer (dev probe, not the bench)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2503_09304_b200 import kernels as K

import os
SHAPES = {"mixtral": (4096, 14336, 8, 2, K.ROUTE_TOPK_SOFTMAX), "qwen": (2048, 1408, 60, 4, K.ROUTE_SOFTMAX_TOPK),
          "qwen_shared": (2048, 5632, 1, 1, K.ROUTE_SOFTMAX_TOPK)}
d, F, E, k, mode = SHAPES[os.environ.get("SHAPE", "mixtral")]
g = torch.Generator(device="cuda").manual_seed(0)
wr = (torch.randn((E, d), device="cuda", generator=g) / 64).bfloat16()
gu = (torch.randn((E, 2 * F, d), device="cuda", generator=g) / 64).bfloat16()
dn = (torch.randn((E, d, F), device="cuda", generator=g) / 120).bfloat16()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

def timeit(fn, iters=10):
    """Device time of fn: captured in a CUDA graph so host launch overhead is excluded."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3): fn()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        fn()
    ts = []
    for _ in range(iters):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); graph.replay(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[len(ts) // 2]

for T in [int(t) for t in sys.argv[1:]] or [32, 256, 1024, 4096, 8192, 16384]:
    x = torch.randn((T, d), device="cuda", generator=g).bfloat16()
    ids, w = K.router(x, wr, k, mode)
    perm, offsets, xp = K.permute(ids, E, x=x)
    y = torch.empty((T * k, d), dtype=torch.bfloat16, device="cuda")
    act = torch.empty((T * k, F), dtype=torch.bfloat16, device="cuda")
    t_r = timeit(lambda: K.router(x, wr, k, mode))
    gather = K.gathers_rows(d, F, E, T * k) and os.environ.get("PROBE_GATHER") is not None
    if gather:  # the kernel gathers X rows itself (TMA tile::gather4), the permute skips Xp
        t_p = timeit(lambda: K.permute(ids, E))
        t_f = timeit(lambda: K.expert_ffn_gather(x, k, offsets, perm, gu, dn, y, act_ws=act))
    else:
        t_p = timeit(lambda: K.permute(ids, E, x=x))
        t_f = timeit(lambda: K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, act_ws=act))
    t_c = timeit(lambda: K.combine(y, w, x))
    flops = 6.0 * T * k * d * F
    hit = int((offsets[1:] > offsets[:-1]).sum())
    wbytes = hit * 3 * d * F * 2
    print(f"T={T:6d} router {t_r*1e3:8.1f}us permute {t_p*1e3:8.1f}us ffn {t_f*1e3:9.1f}us "
          f"({flops/t_f/1e9:7.1f} TFLOP/s, weights {wbytes/t_f/1e6:7.1f} GB/s) combine {t_c*1e3:7.1f}us "
          f"path {K.expert_ffn_path(d, F, E, T * k)}{' gather' if gather else ''} "
          f"total {(t_r + t_p + t_f + t_c) * 1e3:8.1f}us", flush=True)
