"""Compare two tools/router_ab.py output files (e.g. QMOE_ROUTER_TC=0 vs the tcgen05 router):
rows whose expert set differs and the max weight difference, per shape and token count.
    python tools/router_tc_cmp.py a.pt b.pt"""
import sys
import torch

a, b = torch.load(sys.argv[1]), torch.load(sys.argv[2])
for key in a:
    (ia, wa), (ib, wb) = a[key], b[key]
    diff = (ia != ib).any(1)
    same = ~diff
    dw = (wa[same] - wb[same]).abs().max().item() if same.any() else 0.0
    print(f"{key}: {int(diff.sum())} of {ia.shape[0]} rows pick another set; max |dw| on the rest {dw:.2e}")
