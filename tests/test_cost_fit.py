"""Per-stage CostModel fit (calibrate.fit_cost_model): recovers the linear terms of the reference's
CostModel (reference engine.py:48-88) from noisy stage samples; non-negative coefficients."""
import numpy as np

from paper_2503_09304_b200.calibrate import fit_cost_model
from paper_2503_09304_b200.engine import CostModel


def test_fit_recovers_linear_stage_costs():
    rng = np.random.default_rng(0)
    true = CostModel(attn_base=0.21, attn_per_token=0.00031, attn_per_cached=0.0000042, router_cost=0.012,
                     expert_base=0.041, expert_per_entry=0.00095, checkpoint_cost=0.02, restore_cost=0.004)
    att = []
    for _ in range(400):
        t, c = int(rng.integers(1, 4000)), int(rng.integers(0, 60000))
        att.append((t, c, true.attention_cost(t, c) * (1 + 0.01 * rng.standard_normal())))
    exp = []
    for _ in range(400):
        n, e = int(rng.integers(1, 9)), int(rng.integers(1, 16000))
        exp.append((n, e, (n * true.expert_base + e * true.expert_per_entry) * (1 + 0.01 * rng.standard_normal())))
    samples = {"attention": att, "experts": exp, "router": list(0.012 + 0.0001 * rng.standard_normal(50)),
               "checkpoint": [0.02] * 5, "restore": [0.004] * 5}
    cm, rep = fit_cost_model(samples)
    for k in ("attn_base", "attn_per_token", "attn_per_cached", "expert_base", "expert_per_entry", "router_cost"):
        assert abs(getattr(cm, k) / getattr(true, k) - 1) < 0.05, (k, getattr(cm, k), getattr(true, k))
    assert rep["attn_base"]["r2"] > 0.99 and rep["expert_base"]["r2"] > 0.99
    cm.validate()


def test_iteration_fit_recovers_the_model_from_whole_iterations():
    """fit_cost_model_iterations: every iteration's wall time = sum over its layers of the linear
    stage costs; the fit recovers the terms (router_cost from the stage median, the layer term
    pays the rest) and predicts iterations."""
    from paper_2503_09304_b200.calibrate import fit_cost_model_iterations

    rng = np.random.default_rng(1)
    true = CostModel(attn_base=0.15, attn_per_token=0.0002, attn_per_cached=0.000003, router_cost=0.012,
                     expert_base=0.03, expert_per_entry=0.0008, checkpoint_cost=0.02, restore_cost=0.004)
    its = []
    for _ in range(300):
        L = int(rng.integers(1, 33))
        T = int(rng.integers(1, 4000))
        cached = int(rng.integers(0, 60000))
        hit, entries = int(rng.integers(L, 8 * L + 1)), 2 * T * L  # non-empty experts vary per layer
        ms = (L * (true.attn_base + true.router_cost) + true.attn_per_token * T * L + true.attn_per_cached * cached
              + true.expert_base * hit + true.expert_per_entry * entries)
        its.append((L, T * L, cached, hit, entries, ms * (1 + 0.001 * rng.standard_normal())))
    samples = {"iterations": its, "router": [0.012] * 20, "checkpoint": [0.02], "restore": [0.004]}
    cm, rep = fit_cost_model_iterations(samples, stage_fit=true)
    for k in ("attn_base", "attn_per_token", "attn_per_cached", "expert_base", "expert_per_entry", "router_cost"):
        assert abs(getattr(cm, k) / getattr(true, k) - 1) < 0.08, (k, getattr(cm, k), getattr(true, k))
    assert rep["r2"] > 0.99 and rep["median_abs_rel_err"] < 0.02
    cm.validate()
    # without a stage fit the whole per-token term is charged to attention: same iteration totals
    cm2, _ = fit_cost_model_iterations(samples)
    assert cm2.expert_per_entry == 0.0
    assert abs(cm2.attn_per_token / (true.attn_per_token + 2 * true.expert_per_entry) - 1) < 0.08
