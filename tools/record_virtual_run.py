"""Record a VIRTUAL-clock run of the full B200 path on the Mixtral-8x7B-shaped decoder (32 layers,
random-init bf16, real tcgen05 kernels) for the big-shape decision-log parity check (SURVEY.md
section 8c, parity matrix row 2): the decision log this run produces, plus the routing (expert ids
per member per layer, in the reference's route/route_many call order) and the emitted tokens.

tests/golden/gen_golden.py then replays exactly these ids and tokens through the UNMODIFIED
reference simulator (a routing-replay stub model) and records the reference's
own decision log; tests/test_decision_log.py checks the two logs are identical, and
tests/test_engine_gpu.py re-runs this recording and checks the B200 path reproduces it.

    python tools/record_virtual_run.py tests/golden/logs/mixtral_b200_run.json.gz [qwen]
"""
from __future__ import annotations

import gzip
import json
import sys
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, QWEN15_MOE_A27B, DecoderMoEModel  # noqa: E402
from paper_2503_09304_b200.sim import Simulation  # noqa: E402
from paper_2503_09304_b200.workload import WorkloadSpec, trace_for_rate  # noqa: E402

# short paper-style workload (Poisson, 20% LS) with small prompts so the reference replays it fast
SPEC = WorkloadSpec(duration_s=3.0, ls_fraction=0.2, prompt_mean=48, prompt_sigma=0.8, prompt_bounds=(4, 256),
                    output_mean=24, output_sigma=0.9, output_bounds=(1, 64))
RATE, SEED, MBS = 6.0, 5, 8


def trace():
    return trace_for_rate(SPEC, RATE, seed=SEED)


def record(model: DecoderMoEModel, scheduler: str = "qllm") -> dict:
    tr = trace()
    sim = Simulation(tr, model=model, scheduler=scheduler, max_batch_size=MBS, record_log=True)
    routes, emits = [], []
    eng = sim.engine
    cur = {}
    init_state = eng._init_state

    def _init_state(seqs):
        st = init_state(seqs)
        cur["members"] = st.members
        return st

    eng._init_state = _init_state
    route_batch, emit_batch = model.route_batch, model.emit_batch

    def route(layer, x):
        ids, w = route_batch(layer, x)
        rows = ids.tolist()
        for mr in cur["members"]:  # the reference routes member by member (engine.py:303-310)
            routes.append([layer, mr.n, [sorted(r) for r in rows[mr.row0:mr.row0 + mr.n]]])
        return ids, w

    def emit(h, rows):
        out = emit_batch(h, rows)
        emits.extend(int(t) for t in out)
        return out

    model.route_batch, model.emit_batch = route, emit
    try:
        res = sim.run()
    finally:
        model.route_batch, model.emit_batch = route_batch, emit_batch
        eng._init_state = init_state
    cfg = model.config  # the engine's view: Qwen's shared sub-experts count as experts 60..63
    return {
        "scheduler": scheduler, "policy": scheduler, "max_batch_size": MBS,
        # the reference replays with a stub of this shape (d only sizes its toy arrays; costs and
        # decisions do not depend on d, engine.py:71-85)
        "model": {"num_layers": cfg.num_layers, "hidden_dim": 8, "num_experts": cfg.num_experts,
                  "top_k": cfg.top_k, "vocab_size": cfg.vocab_size, "seed": 0},
        "source": f"B200 {cfg.name} bf16 random-init (seed 0), virtual clock, trace_for_rate(rate={RATE}, seed={SEED})",
        "trace": [[r.id, r.arrival_ms, r.priority.tag, r.prompt_len, r.max_new_tokens, r.prompt_seed] for r in tr],
        "log": res.log, "routes": routes, "emits": emits,
        "tokens": {str(i): s.generated for i, s in sorted(res.sequences.items())},
        "records": [[r.seq_id, r.first_token_ms, r.finish_ms] for r in res.records],
        "makespan_ms": res.makespan_ms, "preemptions": res.probes.preemptions,
    }


def main():
    out = Path(sys.argv[1])
    model = DecoderMoEModel(QWEN15_MOE_A27B if "qwen" in sys.argv[2:] else MIXTRAL_8X7B)
    rec = record(model)
    out.parent.mkdir(parents=True, exist_ok=True)
    with gzip.open(out, "wt", encoding="utf-8") as fh:
        json.dump(rec, fh, separators=(",", ":"))
    print(json.dumps({"events": len(rec["log"]), "routes": len(rec["routes"]), "emits": len(rec["emits"]),
                      "preemptions": rec["preemptions"], "makespan_ms": rec["makespan_ms"], "jobs": len(rec["trace"])}))


if __name__ == "__main__":
    main()
