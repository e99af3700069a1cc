"""INTEGRATION.md section 1 (the reference's model plugin swapped for libqmoe over ctypes) is
executable as written: its code block runs against libqmoe.so with a stand-in for the reference's
MoEModel base class that holds the reference's seeded parameters (oracle ToyParams, model.py:86-102),
and its route_many / expert_forward_many answer exactly what the oracle restatement of
model.py:122-145 answers."""

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _plugin_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    head = "```python\n# moesim/qmoe_plugin.py"
    assert head in text, "INTEGRATION.md lost its plugin code block"
    code = text.split(head, 1)[1].split("```", 1)[0]
    assert "from moesim.model import MoEModel" in code
    return code


def test_integration_plugin_matches_oracle(cuda):
    from oracle import moe_oracle as O
    from paper_2503_09304_b200 import _lib

    class MoEModel:  # the reference base class's parameters, nothing else
        def __init__(self, config):
            p = O.ToyParams(config)
            self.config = config
            self.w_router, self.expert_weight, self.expert_bias = p.w_router, p.expert_weight, p.expert_bias

    code = _plugin_source().replace("from moesim.model import MoEModel", "")
    code = code.replace('"/path/to/paper_2503_09304_b200/libqmoe.so"', repr(str(_lib.LIB_PATH)))
    ns = {"MoEModel": MoEModel}
    exec(compile("# moesim/qmoe_plugin.py" + code, "INTEGRATION.md#plugin", "exec"), ns)
    cfg = O.ToyConfig(num_layers=2, hidden_dim=64, num_experts=8, top_k=2)
    model = ns["QmoeModel"](cfg)
    p = O.ToyParams(cfg)
    H = np.random.default_rng(5).standard_normal((12, cfg.hidden_dim))
    for layer in range(cfg.num_layers):
        got = model.route_many(H, layer)
        ids, w = O.route_many(p.w_router[layer], H, cfg.top_k)
        for t in range(H.shape[0]):
            assert sorted(got[t]) == [int(e) for e in ids[t]]
            np.testing.assert_allclose([got[t][int(e)] for e in ids[t]], w[t], rtol=0, atol=1e-12)
        one = model.route(H[3], layer)
        assert one == got[3]
        for e in (0, 3, cfg.num_experts - 1):
            Y = model.expert_forward_many(e, layer, H)
            ref = O.expert_tanh(p.expert_weight[layer][e], p.expert_bias[layer][e], H)
            np.testing.assert_allclose(Y, ref, rtol=0, atol=1e-12)
