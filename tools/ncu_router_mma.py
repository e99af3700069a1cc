import sys, torch
sys.path.insert(0, ".")
from paper_2503_09304_b200 import kernels as K
d, E, k = 4096, 8, 2
wr = (torch.randn((E, d), device="cuda") / 64).bfloat16()
x = torch.randn((2048, d), device="cuda").bfloat16()
for _ in range(3):
    ids, w = K.router(x, wr, k)
torch.cuda.synchronize()
