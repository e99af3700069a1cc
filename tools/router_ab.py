"""Router alone (L2 flushed, CUDA events): time and achieved HBM GB/s of X + W_router reads for
Mixtral (d=4096, E=8, k=2) and the Qwen layer (d=2048, 60 routed + shared gate, k=4+4) at several
token counts; saves ids/weights to compare kernels across QMOE_ROUTER_STREAM settings.
    python tools/router_ab.py out.pt"""
import json, os, statistics, sys
sys.path.insert(0, ".")
import torch
from paper_2503_09304_b200 import kernels as K

flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
res, saved = [], {}
for name, d, E, k, S, mode in (("mixtral", 4096, 8, 2, 0, K.ROUTE_TOPK_SOFTMAX),
                               ("qwen", 2048, 60, 4, 4, K.ROUTE_SOFTMAX_TOPK)):
    g = torch.Generator(device="cuda").manual_seed(1)
    wr = (torch.randn((E + (1 if S else 0), d), device="cuda", generator=g) * d ** -0.5).bfloat16()
    for T in [int(t) for t in os.environ.get("ROUTER_AB_T", "256,1024,2048,4096,8192,16384").split(",")]:
        x = torch.randn((T, d), device="cuda", generator=g).bfloat16()
        for _ in range(3):
            ids, w = K.router(x, wr, k, mode, n_shared=S)
        ts = []
        for _ in range(20):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); K.router(x, wr, k, mode, n_shared=S); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        nbytes = 2 * T * d + 2 * wr.numel() + 8 * T * (k + S)
        res.append({"shape": name, "T": T, "us": ms * 1e3, "gbs": nbytes / ms / 1e6})
        saved[f"{name}{T}"] = (ids.cpu(), w.cpu())
        print(json.dumps(res[-1]), flush=True)
torch.save(saved, sys.argv[1])
