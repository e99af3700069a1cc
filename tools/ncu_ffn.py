"""Minimal driver for `ncu --set full` on the grouped expert FFN kernels (Mixtral layer, T tokens)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2503_09304_b200.moe_block import SparseMoeBlock

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
blk = SparseMoeBlock(4096, 14336, 8, 2).init_random(1234)
x = torch.randn((T, 4096), device="cuda").bfloat16()
for _ in range(2):
    blk(x)
torch.cuda.synchronize()
