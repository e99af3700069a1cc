"""Golden numbers for the cost-model calibration (reference cli.py:198-255), computed by the
UNMODIFIED reference imported read-only from /root/reference/pkg (builder container only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_calibration.py

Writes tests/golden/calibration.json: calibration_iteration_ms of two (ModelConfig, CostModel)
pairs and the CostModel `calibrate` returns for the reference test's window (test_cli.py:127-132).
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from moesim.cli import calibrate, calibration_iteration_ms  # noqa: E402
from moesim.engine import CostModel  # noqa: E402
from moesim.model import ModelConfig  # noqa: E402

cases = []
for mc, cm in [({"num_layers": 4, "hidden_dim": 8, "num_experts": 4, "top_k": 2, "vocab_size": 32, "seed": 3},
                {"attn_base": 9.0, "router_cost": 4.0, "expert_base": 3.0}),
               ({"num_layers": 2, "hidden_dim": 16, "num_experts": 8, "top_k": 2, "vocab_size": 64, "seed": 0}, {})]:
    ms = calibration_iteration_ms(ModelConfig(**mc), CostModel(**cm))
    tuned = calibrate(ModelConfig(**mc), CostModel(**cm), 300.0, 400.0)
    cases.append({"model": mc, "cost": cm, "iteration_ms": ms, "tuned_300_400": tuned.__dict__,
                  "tuned_iteration_ms": calibration_iteration_ms(ModelConfig(**mc), tuned)})
out = Path(__file__).resolve().parent / "calibration.json"
out.write_text(json.dumps({"source": "reference moesim cli.calibration_iteration_ms / calibrate", "cases": cases},
                          indent=1))
print(json.dumps(cases, indent=1))
