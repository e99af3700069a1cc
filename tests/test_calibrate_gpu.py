"""Cost-model calibration (calibrate.py; reference cli.py:198-255, test_cli.py:127-140).

The virtual canonical decode iteration of the reference's toy model equals the reference's own
number bit for bit (tests/golden/calibration.json, made by tests/golden/gen_calibration.py from
the unmodified reference), and so does the CostModel `calibrate` returns; `b200_cost_model`
charges the virtual iteration of a model at the speed the B200 measured for it."""

import json
from dataclasses import asdict

import pytest

from conftest import GOLDEN


def test_calibrate_rejects_degenerate_targets():
    """test_cli.py:135-140: rejected before anything runs (no GPU needed)."""
    from paper_2503_09304_b200.calibrate import calibrate
    from paper_2503_09304_b200.engine import CostModel
    from paper_2503_09304_b200.model import ModelConfig

    model = ModelConfig(num_layers=2, hidden_dim=8, num_experts=4, top_k=2, vocab_size=32, seed=3)
    with pytest.raises(ValueError):
        calibrate(model, CostModel(), 0.0, 0.0)
    with pytest.raises(ValueError):
        calibrate(model, CostModel(), 400.0, 300.0)


@pytest.mark.gpu
def test_calibration_matches_reference(cuda):
    from paper_2503_09304_b200.calibrate import calibrate, calibration_iteration_ms
    from paper_2503_09304_b200.engine import CostModel
    from paper_2503_09304_b200.model import ModelConfig

    gold = json.loads((GOLDEN / "calibration.json").read_text())["cases"]
    for case in gold:
        mc, cm = ModelConfig(**case["model"]), CostModel(**case["cost"])
        assert calibration_iteration_ms(mc, cm) == case["iteration_ms"]
        tuned = calibrate(mc, cm, 300.0, 400.0)
        assert asdict(tuned) == case["tuned_300_400"]
        assert calibration_iteration_ms(mc, tuned) == case["tuned_iteration_ms"]
        assert 300.0 <= calibration_iteration_ms(mc, tuned) <= 400.0


@pytest.mark.gpu
def test_b200_cost_model_charges_measured_speed(cuda):
    """A 4-layer Mixtral-shaped decoder: the scaled CostModel's virtual canonical iteration equals
    the measured wall time (same routing and token counts), and the scale is positive."""
    from paper_2503_09304_b200.calibrate import _canonical_iteration_ms, b200_cost_model
    from paper_2503_09304_b200.engine import VirtualClock
    from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, DecoderMoEModel

    from dataclasses import replace
    model = DecoderMoEModel(replace(MIXTRAL_8X7B, num_layers=4))
    scaled, info = b200_cost_model(model, repeats=3)
    assert info["wall_ms"] > 0 and info["scale"] > 0
    virt = _canonical_iteration_ms(model, VirtualClock(), scaled, 0, model.config.vocab_size)[0]
    assert virt == pytest.approx(info["wall_ms"], rel=1e-9)
