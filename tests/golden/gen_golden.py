"""Generate golden fixtures from the UNMODIFIED reference (moesim), imported read-only from
/root/reference/pkg.  Run in the builder container (the reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden.py

Outputs (committed):
  tiny_layer.npz         one MoE layer of ModelConfig(2,256,8,2,256,seed=0) on real attention
                         outputs captured from trace A: router ids/weights, per-expert queue order,
                         expert outputs (slot order), combine output, plus a resume case
  toy_params_digest.json sha256 of every parameter array of three seeded configs (pins the
                         oracle's draw order, model.py:86-102)
  logs/*.json.gz         decision logs (selections, trims, reports with virtual timestamps and
                         directives, per-expert queue contents, preemptions, tokens) for traces
                         A, B, P under qllm / baseline / never-preempt and for the reference's
                         random-preemption transparency traces, with the routing/emit call
                         records a replay backend needs.
Hooks are instance-attribute wraps and the constructor's policy= argument, exactly as in
SURVEY.md Appendix A; the reference source is never modified or copied.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
sys.dont_write_bytecode = True

from moesim.cli import ExperimentConfig, trace_for_rate  # noqa: E402
from moesim.core import Phase, Priority, SchedulerDirective  # noqa: E402
from moesim.engine import CostModel  # noqa: E402
from moesim.model import ModelConfig, MoEModel  # noqa: E402
from moesim.sched import POLICIES  # noqa: E402
from moesim.sim import Simulation  # noqa: E402
from moesim.workload import WorkloadSpec, generate  # noqa: E402

OUT = Path(__file__).resolve().parent
TINY = ModelConfig(num_layers=2, hidden_dim=256, num_experts=8, top_k=2, vocab_size=256, seed=0)


def trace_a(seed=2, rate=16.0):
    cfg = ExperimentConfig(
        model=TINY,
        workload=WorkloadSpec(ls_fraction=0.25, prompt_mean=32, prompt_sigma=0.8, prompt_bounds=(4, 128),
                              output_mean=16, output_sigma=0.9, output_bounds=(1, 48)),
        jobs_per_run=16, seed=seed, max_batch_size=8)
    return trace_for_rate(cfg, rate)


def trace_p():
    return generate(WorkloadSpec(arrival_rate=4.0, ls_fraction=0.2, duration_s=60, seed=1, prompt_mean=64,
                                 prompt_sigma=0.8, prompt_bounds=(4, 256), output_mean=32, output_sigma=0.9,
                                 output_bounds=(1, 64)))[:16]


def small_trace(seed):
    """reference tests/test_sim.py:31-37"""
    return generate(WorkloadSpec(arrival_rate=40.0, duration_s=0.3, seed=seed, ls_fraction=0.3, prompt_mean=6,
                                 prompt_sigma=0.6, prompt_bounds=(2, 16), output_mean=3, output_sigma=0.5,
                                 output_bounds=(1, 6)))


class RandomPreempt:
    """Seeded coin per report (reference tests/test_sim.py:18-28)."""

    def __init__(self, seed, p=0.3):
        self.rng = np.random.default_rng(seed)
        self.p = p

    def __call__(self, report, queues):
        return (SchedulerDirective.PREEMPT_AT_NEXT_BOUNDARY if self.rng.random() < self.p
                else SchedulerDirective.CONTINUE)


def record_run(trace, model_config, scheduler, mbs, policy=None, policy_spec=None, model_factory=None):
    """Run the reference with logging hooks; returns a JSON-able dict.  model_factory (optional)
    swaps in a routing-replay stub after construction."""
    log = []
    base_policy = policy if policy is not None else (POLICIES[scheduler] if scheduler in POLICIES else None)

    def logged_policy(r, snap):
        d = base_policy(r, snap)
        log.append(["R", r.batch_id, r.stage.name, r.layer_index, r.expert_id, r.timestamp, d.name])
        return d

    kwargs = {}
    if scheduler != "baseline":
        kwargs["policy"] = logged_policy
    sim = Simulation(trace, model_config=model_config, scheduler=scheduler, max_batch_size=mbs, **kwargs)
    if model_factory is not None:
        sim.model = sim.engine.model = model_factory(model_config)
    sch = sim.scheduler
    g = sch.get_next_batch

    def get_next_batch(decode_only=False):
        s = g(decode_only)
        if s is not None:
            log.append(["S", list(s.seq_ids), s.phase.name, bool(s.resume), bool(decode_only)])
        return s

    sch.get_next_batch = get_next_batch
    rq = sch.requeue_front

    def requeue_front(ids):
        log.append(["T", list(ids)])
        return rq(ids)

    sch.requeue_front = requeue_front
    op = sch.on_preempted

    def on_preempted(ckpts):
        log.append(["P", [int(i) for i in ckpts], [[c.layer_index, c.stage.name] for c in ckpts.values()]])
        return op(ckpts)

    sch.on_preempted = on_preempted
    ro = sch.route_output

    def route_output(seq, token, now):
        log.append(["K", seq.id, int(token), now])
        return ro(seq, token, now)

    sch.route_output = route_output
    if scheduler == "baseline":
        oer = sch.on_engine_report

        def on_engine_report(r):
            d = oer(r)
            log.append(["R", r.batch_id, r.stage.name, r.layer_index, r.expert_id, r.timestamp, d.name])
            return d

        sch.on_engine_report = on_engine_report
    dr = sim.engine.queues.drain

    def drain(e, l):
        q = dr(e, l)
        log.append(["Q", l, e, [[x.seq_id, x.token_index] for x in q]])
        return q

    sim.engine.queues.drain = drain
    # routing / emit call records for replay backends (keyed by call order)
    routes, emits = [], []
    m = sim.model
    r1, rm, em = m.route, m.route_many, m.emit_token

    def route(h, layer):
        out = r1(h, layer)
        routes.append([layer, 1, [sorted(out)]])
        return out

    def route_many(H, layer):
        out = rm(H, layer)
        routes.append([layer, len(out), [sorted(o) for o in out]])
        return out

    def emit(h):
        t = em(h)
        emits.append(int(t))
        return t

    m.route, m.route_many, m.emit_token = route, route_many, emit
    res = sim.run()
    return {
        "scheduler": scheduler,
        "policy": policy_spec or scheduler,
        "max_batch_size": mbs,
        "model": model_config.__dict__,
        "trace": [[r.id, r.arrival_ms, r.priority.tag, r.prompt_len, r.max_new_tokens, r.prompt_seed] for r in trace],
        "log": log,
        "routes": routes,
        "emits": emits,
        "tokens": {str(i): s.generated for i, s in sorted(res.sequences.items())},
        "records": [[r.seq_id, r.first_token_ms, r.finish_ms] for r in res.records],
        "makespan_ms": res.makespan_ms,
        "preemptions": res.probes.preemptions,
    }


def write_json_gz(obj, path):
    path.parent.mkdir(parents=True, exist_ok=True)
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(obj, fh, separators=(",", ":"))


def gen_logs():
    runs = []
    for name, trace, mbs in (("A", trace_a(), 8), ("B", trace_a(seed=1, rate=4.0), 8), ("P", trace_p(), 32)):
        for sched in ("qllm", "baseline", "never-preempt"):
            rec = record_run(trace, TINY, sched, mbs)
            write_json_gz(rec, OUT / "logs" / f"trace{name}_{sched}.json.gz")
            runs.append((name, sched, len(rec["log"]), rec["preemptions"], rec["makespan_ms"]))
    small = ModelConfig(num_layers=2, hidden_dim=8, num_experts=4, top_k=2, vocab_size=32, seed=2)
    for seed in range(8):
        trace = small_trace(seed)
        if not trace:
            continue
        rec = record_run(trace, small, "qllm", 32, policy=RandomPreempt(seed), policy_spec=f"random:{seed}:0.3")
        write_json_gz(rec, OUT / "logs" / f"random{seed}_qllm.json.gz")
        runs.append((f"random{seed}", "qllm", len(rec["log"]), rec["preemptions"], rec["makespan_ms"]))
    for r in runs:
        print("log", *r)


class ReplayStub(MoEModel):
    """Reference-side routing-replay stub: the reference's own
    engine, scheduler, driver and virtual clock run unchanged; route / route_many / emit_token
    return the B200 run's recorded expert ids and tokens in call order and assert the call
    (layer, token count) matches, so any schedule divergence surfaces at once."""

    def __init__(self, cfg, routes, emits):
        super().__init__(cfg)
        self._routes, self._emits = list(routes), list(emits)
        self._r = self._e = 0

    def _next(self, layer, n):
        rl, rn, ids = self._routes[self._r]
        self._r += 1
        assert (rl, rn) == (layer, n), f"replay diverged at route call {self._r - 1}: {(rl, rn)} vs {(layer, n)}"
        return [{e: 1.0 / len(row) for e in row} for row in ids]

    def route(self, h, layer):
        return self._next(layer, 1)[0]

    def route_many(self, H, layer):
        return self._next(layer, len(H))

    def emit_token(self, h):
        t = self._emits[self._e]
        self._e += 1
        return t


def gen_b200_ref(name="mixtral"):
    """The reference's decision log for a B200 virtual-clock run recorded by
    tools/record_virtual_run.py (logs/<name>_b200_run.json.gz, Mixtral- or Qwen-shaped): same
    trace, same expert ids and tokens replayed through the unmodified reference ->
    logs/<name>_b200_ref.json.gz."""
    from moesim.workload import TraceRecord

    src = OUT / "logs" / f"{name}_b200_run.json.gz"
    with gzip.open(src, "rt") as fh:
        run = json.load(fh)
    cfg = ModelConfig(**run["model"])
    trace = [TraceRecord(i, a, Priority.from_tag(p), pl, mn, sd) for i, a, p, pl, mn, sd in run["trace"]]
    rec = record_run(trace, cfg, run["scheduler"], run["max_batch_size"],
                     model_factory=lambda c: ReplayStub(c, run["routes"], run["emits"]))
    rec["source"] = "reference moesim replaying " + run["source"]
    del rec["routes"], rec["emits"]  # identical to the run's by construction
    write_json_gz(rec, OUT / "logs" / f"{name}_b200_ref.json.gz")
    print(name, "b200 ref log", len(rec["log"]), "events", rec["preemptions"], "preemptions", rec["makespan_ms"])


def gen_tiny_layer():
    """Capture real router inputs of trace A's first prefill batch, then run the reference's
    router / queues / experts / combine on them."""
    from moesim.engine import InferenceEngine, _MemberState  # noqa: F401

    captured = {}
    sim = Simulation(trace_a(), model_config=TINY, scheduler="qllm", max_batch_size=8)
    eng = sim.engine
    orig = eng._router_stage

    def grab(states, layer):
        if layer not in captured and sum(st.num_tokens for st in states) > 64:
            captured[layer] = ([st.seq.id for st in states], [st.hidden.copy() for st in states])
        return orig(states, layer)

    eng._router_stage = grab
    sim.run()
    model = MoEModel(TINY)
    out = {}
    for layer in (0, 1):
        ids_members, hs = captured[layer]
        H = np.concatenate(hs)
        routing = model.route_many(H, layer)
        T, k = H.shape[0], TINY.top_k
        ids = np.array([sorted(r) for r in routing], dtype=np.int64)
        w = np.array([[r[e] for e in sorted(r)] for r in routing])
        # per-expert FIFO (ExpertQueues semantics) and expert outputs in slot order
        from moesim.model import ExpertQueueEntry, ExpertQueues
        q = ExpertQueues(TINY.num_experts, TINY.num_layers)
        for t in range(T):
            for e in sorted(routing[t]):
                q.enqueue(ExpertQueueEntry(0, t, layer, e, routing[t][e]))
        perm, offsets = [], [0]
        Y = np.zeros((T * k, TINY.hidden_dim))
        for e in q.pending_experts(layer):
            entries = q.drain(e, layer)
            X = np.stack([H[x.token_index] for x in entries])
            Yo = model.expert_forward_many(e, layer, X)
            for row, x in enumerate(entries):
                j = sorted(routing[x.token_index]).index(e)
                Y[x.token_index * k + j] = Yo[row]
                perm.append(x.token_index * k + j)
        counts = [sum(1 for t in range(T) for e2 in ids[t] if e2 == e) for e in range(TINY.num_experts)]
        offsets = np.concatenate([[0], np.cumsum(counts)])
        combined = np.stack([model.combine(H[t], routing[t], {e: Y[t * k + j] for j, e in enumerate(ids[t])}, set())
                             for t in range(T)])
        # resume case: pretend experts < 4 were drained before a preemption
        cursor = np.full(T, 4, dtype=np.int64)
        q2 = ExpertQueues(TINY.num_experts, TINY.num_layers)
        for t in range(T):
            for e in sorted(x for x in routing[t] if x >= 4):
                q2.enqueue(ExpertQueueEntry(0, t, layer, e, routing[t][e]))
        perm_resume = []
        for e in q2.pending_experts(layer):
            for x in q2.drain(e, layer):
                perm_resume.append(x.token_index * k + sorted(routing[x.token_index]).index(e))
        out.update({
            f"H{layer}": H, f"ids{layer}": ids, f"w{layer}": w, f"perm{layer}": np.array(perm),
            f"offsets{layer}": offsets, f"Y{layer}": Y, f"out{layer}": combined,
            f"cursor{layer}": cursor, f"perm_resume{layer}": np.array(perm_resume),
            f"members{layer}": np.array(ids_members),
        })
        print("tiny layer", layer, "T", T, "counts", counts)
    np.savez_compressed(OUT / "tiny_layer.npz", **out)


def gen_param_digests():
    digests = {}
    for cfg in (TINY, ModelConfig(num_layers=2, hidden_dim=4, num_experts=4, top_k=2, vocab_size=16, seed=42),
                ModelConfig(num_layers=2, hidden_dim=8, num_experts=4, top_k=2, vocab_size=32, seed=2)):
        m = MoEModel(cfg)
        arrays = {"embedding": m.embedding, "w_out": m.w_out, "b_out": m.b_out}
        for l in range(cfg.num_layers):
            arrays[f"w_key{l}"] = m.w_key[l]
            arrays[f"w_value{l}"] = m.w_value[l]
            arrays[f"w_router{l}"] = m.w_router[l]
            arrays[f"expert_weight{l}"] = m.expert_weight[l]
            arrays[f"expert_bias{l}"] = m.expert_bias[l]
        key = json.dumps(cfg.__dict__, sort_keys=True)
        digests[key] = {n: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest() for n, a in arrays.items()}
    (OUT / "toy_params_digest.json").write_text(json.dumps(digests, indent=1, sort_keys=True))


if __name__ == "__main__":
    if sys.argv[1:2] == ["b200"]:  # only the reference replay of committed B200 runs
        for name in sys.argv[2:] or ["mixtral", "qwen"]:
            gen_b200_ref(name)
        sys.exit(0)
    gen_param_digests()
    gen_tiny_layer()
    gen_logs()
    for name in ("mixtral", "qwen"):
        if (OUT / "logs" / f"{name}_b200_run.json.gz").exists():
            gen_b200_ref(name)
