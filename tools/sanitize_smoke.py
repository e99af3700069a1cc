"""Small kernel workload for compute-sanitizer (memcheck / racecheck / synccheck): router, permute,
every bf16 expert path (swap-AB, swap-AB CTA pair, fused 1-CTA, fused CTA pair), combine, on tiny shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_09304_b200 import kernels as K

torch.manual_seed(0)
for (T, d, F, E, k) in [(16, 256, 512, 8, 2), (400, 256, 512, 4, 2), (600, 256, 256, 2, 2), (1600, 256, 256, 2, 2),
                        (200, 256, 512, 1, 1), (1100, 256, 256, 32, 4)]:
    x = torch.randn((T, d), device="cuda").bfloat16()
    wr = (torch.randn((E, d), device="cuda") / d ** 0.5).bfloat16()
    gu = (torch.randn((E, 2 * F, d), device="cuda") / d ** 0.5).bfloat16()
    dn = (torch.randn((E, d, F), device="cuda") / F ** 0.5).bfloat16()
    ids, w = K.router(x, wr, k)
    perm, offsets, xp = K.permute(ids, E, x=x)
    y = torch.zeros((T * k, d), dtype=torch.bfloat16, device="cuda")
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y)
    out = K.combine(y, w, x)
    torch.cuda.synchronize()
    print(T, "path", K.expert_ffn_path(d, F, E, T * k), "ok", float(out.float().abs().mean()))
