"""Kernel timeline of the bench's Qwen layer step (8192 tokens, L2 flushed before each step, eager
launches exactly as bench.py's qwen leg) under torch.profiler (CUPTI): per step the device time of
each kernel and the idle gaps between them, to split the layer-minus-FFN time into kernel time and
launch / host gaps.  python tools/qwen_layer_timeline.py [T]"""
import json, sys
sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2503_09304_b200 import kernels as K

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
d, F, E, k, S = 2048, 1408, 60, 4, 4
g = torch.Generator(device="cuda").manual_seed(7)
wr = (torch.randn((E + 1, d), device="cuda", generator=g) * d ** -0.5).bfloat16()
gu = (torch.randn((E + S, 2 * F, d), device="cuda", generator=g) * d ** -0.5).bfloat16()
dn = (torch.randn((E + S, d, F), device="cuda", generator=g) * F ** -0.5).bfloat16()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
x = torch.randn((T, d), device="cuda", generator=g).bfloat16()
y = torch.empty((T * (k + S), d), dtype=torch.bfloat16, device="cuda")
act = torch.empty((T * (k + S), F), dtype=torch.bfloat16, device="cuda")
direct = K.shared_direct_ok(d, F, E + S, T * (k + S))


def layer():
    ids, w = K.router(x, wr, k, K.ROUTE_SOFTMAX_TOPK, n_shared=S)
    perm, offsets, xp = K.permute(ids, E + S, x=x, gather_e_end=E if direct else None)
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, act_ws=act, x_direct=x if direct else None, x_first=E)
    return K.combine(y, w, x)


for _ in range(3):
    layer()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        flush.zero_()
        layer()
    torch.cuda.synchronize()
ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
            if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0)
steps, cur = [], None
for s, e, n in ev:
    if "qmoe" not in n and cur is not None and cur:
        steps.append(cur)
        cur = []
    elif "qmoe" in n:
        cur = (cur or []) + [(s, e, n)]
    else:
        cur = []
if cur:
    steps.append(cur)
for st in steps:
    span = st[-1][1] - st[0][0]
    busy = sum(e - s for s, e, _ in st)
    parts = [{"kernel": n.split("(")[0].replace("void ", "")[:48], "us": round(e - s, 1),
              "gap_before_us": round(s - (st[i - 1][1] if i else s), 1)} for i, (s, e, n) in enumerate(st)]
    print(json.dumps({"T": T, "span_us": round(span, 1), "kernel_us": round(busy, 1), "gaps_us": round(span - busy, 1),
                      "kernels": parts}))
