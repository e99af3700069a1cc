import sys, torch
sys.path.insert(0, ".")
from paper_2503_09304_b200.moe_block import SparseMoeBlock
from paper_2503_09304_b200 import kernels as K
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
blk = SparseMoeBlock(2048, 1408, 60, 4, route_mode=K.ROUTE_SOFTMAX_TOPK).init_random(1)
x = torch.randn((T, 2048), device="cuda").bfloat16()
for _ in range(2):
    blk(x)
torch.cuda.synchronize()
