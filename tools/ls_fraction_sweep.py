"""BASELINE config 5's LS-fraction axis, measured: one Mixtral-shaped MoE layer (router -> permute ->
grouped SwiGLU -> combine, L2 flushed, CUDA events) on batches of 64 members (prompt rows drawn from
the paper workload's lognormal) whose LS members -- 0, 25, 50, 75, 100% of them -- come first in
the batch, as the QLLM scheduler orders a fresh batch (reference sched.py:305-311).  The member
order only permutes the token rows the kernels see; this measures that it costs nothing.
    python tools/ls_fraction_sweep.py > out.jsonl"""
import json
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2503_09304_b200 import kernels as K  # noqa: E402

d, F, E, k = 4096, 14336, 8, 2
g = torch.Generator(device="cuda").manual_seed(0)
wr = (torch.randn((E, d), device="cuda", generator=g) * d ** -0.5).bfloat16()
gu = (torch.randn((E, 2 * F, d), device="cuda", generator=g) * d ** -0.5).bfloat16()
dn = (torch.randn((E, d, F), device="cuda", generator=g) * F ** -0.5).bfloat16()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
rng = np.random.default_rng(3)
for T_target in (1024, 8192):
    lens = np.clip(rng.lognormal(np.log(T_target / 64), 0.8, 64).astype(int), 4, 2048)
    T = int(lens.sum())
    x_members = [torch.randn((int(n), d), device="cuda", generator=g).bfloat16() for n in lens]
    is_ls = rng.permutation(64)
    for frac in (0.0, 0.25, 0.5, 0.75, 1.0):
        ls = set(is_ls[: int(round(frac * 64))].tolist())
        order = [i for i in range(64) if i in ls] + [i for i in range(64) if i not in ls]  # LS first
        x = torch.cat([x_members[i] for i in order])
        y = torch.empty((T * k, d), dtype=torch.bfloat16, device="cuda")
        act = torch.empty((T * k, F), dtype=torch.bfloat16, device="cuda")

        def layer():
            ids, w = K.router(x, wr, k)
            perm, offsets, xp = K.permute(ids, E, x=x)
            K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, act_ws=act)
            return K.combine(y, w, x)

        for _ in range(3):
            layer()
        ts = []
        for _ in range(10):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            layer()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(a.elapsed_time(b) for a, b in ts)
        print(json.dumps({"tokens": T, "members": 64, "ls_fraction": frac, "layer_ms": ms,
                          "tflops": 6.0 * T * k * d * F / ms / 1e9}), flush=True)
