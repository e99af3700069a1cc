"""Per-stage B200 CostModel fit: measure every engine stage of the
Mixtral-8x7B-shaped decoder on the B200 (CUDA events per stage, virtual-clock run of a paper-workload
trace), least-squares fit the reference's linear CostModel terms (reference engine.py:48-88), and
validate on the canonical decode iteration (reference cli.py:198-236): virtual ms with the fitted
model vs the B200 wall-clock median.

    python tools/fit_cost_model.py profiles/cost_model_b200_r02.json [mixtral|qwen]
"""
import json, statistics, sys
from dataclasses import replace
sys.path.insert(0, ".")
import torch
from paper_2503_09304_b200.calibrate import (_canonical_iteration_ms, fit_cost_model, fit_cost_model_iterations,
                                             measure_stage_samples)
from paper_2503_09304_b200.engine import CostModel, VirtualClock, WallClock
from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, QWEN15_MOE_A27B, DecoderMoEModel
from paper_2503_09304_b200.workload import WorkloadSpec, trace_for_rate

name = sys.argv[2] if len(sys.argv) > 2 else "mixtral"
model = DecoderMoEModel(QWEN15_MOE_A27B if name == "qwen" else MIXTRAL_8X7B)
trace = trace_for_rate(WorkloadSpec(duration_s=6.0, output_bounds=(1, 160)), 7.0, seed=11)
measure_stage_samples(model, trace[:6])  # warm-up (kernels, allocator)
samples = measure_stage_samples(model, trace, wall=True)
cm, rep = fit_cost_model(samples)
cm_it, rep_it = fit_cost_model_iterations(samples, stage_fit=cm)
cm_v, rep_v = fit_cost_model(measure_stage_samples(model, trace, wall=False))
wall = _canonical_iteration_ms(model, WallClock(), CostModel(), 0, model.config.vocab_size, repeats=5)
virt = _canonical_iteration_ms(model, VirtualClock(), cm, 0, model.config.vocab_size)[0]
virt_it = _canonical_iteration_ms(model, VirtualClock(), cm_it, 0, model.config.vocab_size)[0]
virt_v = _canonical_iteration_ms(model, VirtualClock(), cm_v, 0, model.config.vocab_size)[0]
out = {"model": model.config.name, "trace": f"paper workload, 7 req/s, 6 s ({len(trace)} jobs, outputs <= 160)",
       "samples": {k: len(v) for k, v in samples.items()}, "fit": rep, "cost_model": cm.__dict__,
       "virtual_clock_measurement": {"fit": rep_v, "cost_model": cm_v.__dict__,
                                     "canonical_decode_virtual_ms_fitted": virt_v},
       "iteration_fit": {"fit": rep_it, "cost_model": cm_it.__dict__, "canonical_decode_virtual_ms": virt_it,
                         "rel_err": virt_it / statistics.median(wall) - 1.0},
       "reference_cost_model": CostModel().__dict__,
       "validation": {"canonical_decode_wall_ms_median": statistics.median(wall), "wall_ms_all": wall,
                      "canonical_decode_virtual_ms_fitted": virt,
                      "rel_err": virt / statistics.median(wall) - 1.0}}
open(sys.argv[1], "w").write(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
