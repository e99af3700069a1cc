"""Device greedy emission (qmoe_lm_head_argmax) against torch fp32: the
token is the reference's argmax (model.py:166-169, first maximal index) wherever the top-2 margin
exceeds the fp32 accumulation-order band; inside the band the pick is one of the tied maxima.
Shapes: Mixtral's LM head (V=32000, d=4096) and Qwen's (V=151936, d=2048), decode batch sizes."""

import pytest
import torch

from paper_2503_09304_b200 import kernels as K

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("V,d", [(32000, 4096), (151936, 2048), (1000, 512), (37, 128)])
@pytest.mark.parametrize("T", [1, 7, 16, 32, 64])
def test_lm_head_argmax_matches_torch(cuda, V, d, T):
    g = torch.Generator(device="cuda").manual_seed(V + T)
    w = (torch.randn((V, d), device="cuda", generator=g) * d ** -0.5).bfloat16()
    h = torch.randn((T, d), device="cuda", generator=g).bfloat16()
    tok = K.lm_head_argmax(h, w)
    logits = h.float() @ w.float().T
    top2 = logits.topk(2, dim=1)
    margin = top2.values[:, 0] - top2.values[:, 1]
    safe = margin > 1e-3
    ref = logits.argmax(1)
    assert torch.equal(tok[safe].long(), ref[safe])
    picked = logits.gather(1, tok.long()[:, None])[:, 0]
    assert bool((picked >= top2.values[:, 0] - 1e-3).all())


def test_lm_head_argmax_ties_go_to_lowest_id(cuda):
    d, V = 256, 5000
    w = torch.zeros((V, d), device="cuda", dtype=torch.bfloat16)
    w[[17, 4000, 2500]] = 1.0  # three exact maxima
    h = torch.ones((3, d), device="cuda", dtype=torch.bfloat16)
    assert K.lm_head_argmax(h, w).tolist() == [17, 17, 17]
    for _ in range(3):  # the workspace is left zeroed: repeated launches agree
        assert K.lm_head_argmax(h, w).tolist() == [17, 17, 17]
