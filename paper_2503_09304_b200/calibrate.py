"""Virtual cost-model calibration.

`calibration_iteration_ms` and `calibrate` restate the reference's closed-loop rescaling
(reference cli.py:198-255): run one canonical decode iteration (32 members, 32 layers, 180-token
contexts, after a prefill that fills the caches) through the engine on a virtual clock, then scale
every CostModel parameter by target / measured.  The virtual charges depend only on the routing and
the token counts, so on the reference's own toy model (f64 kernels) this engine returns the
reference's number exactly (tests/test_calibrate_gpu.py).

`b200_cost_model` is what the reference cannot do: it runs the same canonical iteration of a real
model (e.g. the Mixtral-shaped decoder) on a wall clock on the B200 and returns the CostModel
scaled so that the virtual iteration of that model lasts exactly what the B200 measured, so
virtual-clock studies (decision logs, SLO sweeps) are charged at B200 speed.
"""
from __future__ import annotations

import functools
import statistics
from dataclasses import replace
from typing import Optional

import numpy as np
import torch

from .core import EOS_TOKEN, Phase, Priority, SchedulerDirective, batch_form, sequence_new
from .engine import Completed, CostModel, InferenceEngine, VirtualClock, WallClock
from .kvcache import UnifiedDynamicCache
from .model import ModelConfig, MoEModel

# reference cli.py:41-43
CANONICAL_CONTEXT = 180
CALIBRATION_BATCH = 32
CALIBRATION_LAYERS = 32


def _canonical_iteration_ms(model, clock, cost_model: CostModel, seed: int, vocab_size: int,
                            repeats: int = 1) -> list[float]:
    """Prefill CALIBRATION_BATCH sequences of CANONICAL_CONTEXT random tokens, then time decode
    iterations of the whole batch (reference cli.py:209-236).  Returns one duration per repeat
    (the reference takes one)."""
    cache = UnifiedDynamicCache(model.config.num_layers, model.kv_row_shape(), model.kv_dtype, model.device,
                                model.kv_entry_bytes(), **getattr(model, "kv_page_kwargs", {}))
    engine = InferenceEngine(model, cache, clock, cost_model, CALIBRATION_BATCH)
    rng = np.random.default_rng(seed + 1)
    seqs = []
    for i in range(CALIBRATION_BATCH):
        prompt = [int(t) for t in rng.integers(1, vocab_size, size=CANONICAL_CONTEXT)]
        seq = sequence_new(prompt, priority=Priority.BEST_EFFORT, max_new_tokens=max(4, 2 + repeats), arrival=0.0,
                           seq_id=i)
        seq.cache_handle = i
        cache.register(i)
        seqs.append(seq)

    def cont(report):
        return SchedulerDirective.CONTINUE

    outcome = engine.execute(batch_form(seqs, Phase.PREFILL, CALIBRATION_BATCH, engine.next_batch_id()), seqs, cont)
    assert isinstance(outcome, Completed)
    for seq in seqs:
        seq.generated.append(outcome.tokens[seq.id])
        seq.advance_phase(Phase.DECODE)
    out = []
    for r in range(repeats):
        # the reference's single timed iteration decodes every member; later repeats drop members
        # that emitted EOS (a random-init model may)
        live = seqs if r == 0 else [q for q in seqs if q.generated[-1] != EOS_TOKEN]
        if not live:
            break
        decode = batch_form(live, Phase.DECODE, CALIBRATION_BATCH, engine.next_batch_id())
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        start = clock.now
        outcome = engine.execute(decode, live, cont)
        assert isinstance(outcome, Completed)
        if torch.cuda.is_available():
            torch.cuda.synchronize()
        out.append(clock.now - start)
        for seq in live:
            seq.generated.append(outcome.tokens[seq.id])
    return out


@functools.lru_cache(maxsize=32)
def calibration_iteration_ms(model_config: ModelConfig, cost_model: CostModel) -> float:
    """Virtual ms of one canonical decode iteration of the reference's toy model (f64) with
    `cost_model` (reference cli.py:198-236; memoized like the reference, both configs frozen)."""
    config = replace(model_config, num_layers=CALIBRATION_LAYERS)
    model = MoEModel(config)
    return _canonical_iteration_ms(model, VirtualClock(), cost_model, config.seed, config.vocab_size)[0]


def calibrate(model_config: ModelConfig, cost_model: CostModel, target_lo: float, target_hi: float) -> CostModel:
    """Rescale `cost_model` so the canonical decode iteration lands in [target_lo, target_hi]
    (reference cli.py:238-255): every parameter times midpoint / measured, then re-measured as a
    closed-loop check.  ValueError on an infeasible window or a landing outside it."""
    if target_hi <= 0 or target_lo < 0 or target_lo > target_hi:
        raise ValueError(f"infeasible target range [{target_lo}, {target_hi}]")
    measured = calibration_iteration_ms(model_config, cost_model)
    if measured <= 0:
        raise ValueError("cost model charges nothing; cannot calibrate")
    mid = 0.5 * (target_lo + target_hi)
    scaled = cost_model.scaled(mid / measured)
    check = calibration_iteration_ms(model_config, scaled)
    if not (target_lo <= check <= target_hi):
        raise ValueError(f"calibration landed at {check:.3f} ms, outside [{target_lo}, {target_hi}]")
    return scaled


def b200_cost_model(model, cost_model: CostModel = CostModel(), repeats: int = 5,
                    seed: Optional[int] = None) -> tuple[CostModel, dict]:
    """CostModel whose virtual canonical decode iteration of `model` equals the B200's wall time.

    The canonical iteration (CALIBRATION_BATCH members, CANONICAL_CONTEXT-token contexts, all of
    `model`'s layers) runs `repeats` times on a WallClock (median taken; the first prefill warms
    the kernels up) and once on a VirtualClock with `cost_model`; every parameter is scaled by
    wall / virtual, the reference's one-factor rescaling (cli.py:250-251) with the B200 as the
    target.  Returns (scaled model, {"wall_ms", "virtual_ms", "scale"})."""
    cfg = model.config
    seed = getattr(cfg, "seed", 0) if seed is None else seed
    wall = _canonical_iteration_ms(model, WallClock(), cost_model, seed, cfg.vocab_size, repeats=repeats)
    virt = _canonical_iteration_ms(model, VirtualClock(), cost_model, seed, cfg.vocab_size)[0]
    if virt <= 0:
        raise ValueError("cost model charges nothing; cannot calibrate")
    wall_ms = statistics.median(wall)
    scale = wall_ms / virt
    return cost_model.scaled(scale), {"wall_ms": wall_ms, "wall_ms_all": wall, "virtual_ms": virt, "scale": scale}


# ---------------------------------------------------------------------------------------------
# Per-stage fit: every CostModel term from measured B200 stage times (reference engine.py:48-88
# charges attention a0 + a1*tokens + a2*cached, router r0, each non-empty expert e0 + e1*entries,
# checkpoint c0 per preemption, restore c1 per member).

def fit_cost_model(samples: dict) -> tuple[CostModel, dict]:
    """Non-negative least squares of each stage's linear form on measured samples (ms):
      attention: [(tokens, cached_entries, ms)]        -> attn_base, attn_per_token, attn_per_cached
      router:    [ms]                                  -> router_cost (median)
      experts:   [(non_empty_experts, entries, ms)]    -> expert_base, expert_per_entry
                 (one grouped launch covers all experts of a layer, so its time is fitted as
                 n_experts * e0 + entries * e1: the reference's per-expert charges summed)
      checkpoint: [ms per preemption], restore: [ms per member]  -> medians
    Returns (CostModel, fit report with R^2 and the worst relative error per stage)."""
    from scipy.optimize import nnls

    rep = {}

    def lin(rows, names):
        a = np.array([r[:-1] for r in rows], dtype=np.float64)
        y = np.array([r[-1] for r in rows], dtype=np.float64)
        coef, _ = nnls(a, y)
        pred = a @ coef
        ss = float(((y - y.mean()) ** 2).sum())
        rep[names[0]] = {"n": len(rows), "r2": 1.0 - float(((y - pred) ** 2).sum()) / ss if ss > 0 else 1.0,
                         "max_rel_err": float(np.max(np.abs(pred - y) / np.maximum(y, 1e-9))),
                         "coef": dict(zip(names, coef.tolist()))}
        return coef

    att = lin([(1.0, t, c, ms) for t, c, ms in samples["attention"]], ["attn_base", "attn_per_token", "attn_per_cached"])
    exp = lin([(n, e, ms) for n, e, ms in samples["experts"]], ["expert_base", "expert_per_entry"])
    med = lambda v: float(statistics.median(v)) if v else 0.0  # noqa: E731
    cm = CostModel(attn_base=float(att[0]), attn_per_token=float(att[1]), attn_per_cached=float(att[2]),
                   router_cost=med(samples["router"]), expert_base=float(exp[0]), expert_per_entry=float(exp[1]),
                   checkpoint_cost=med(samples.get("checkpoint", [])), restore_cost=med(samples.get("restore", [])))
    rep["router"] = {"n": len(samples["router"]), "median_ms": cm.router_cost}
    return cm, rep


def fit_cost_model_iterations(samples: dict, stage_fit: Optional[CostModel] = None) -> tuple[CostModel, dict]:
    """The CostModel whose virtual iterations match measured whole-iteration wall times: non-negative
    least squares of each completed iteration's wall ms on per-iteration sums of the linear model's
    features -- layers (attention base + router), tokens x layers, cached entries scanned and
    non-empty experts (reference engine.py:48-88).  Expert entries are k x tokens x layers in a
    whole iteration, so the per-token term is one coefficient; it is split between attn_per_token
    and expert_per_entry in the proportion of the stage-level fit (stage_fit; all to attention when
    absent).  router_cost keeps its measured stage median and the layer term pays the rest;
    checkpoint / restore keep the stage medians.  Stage-level event brackets overstate an iteration
    (overlapping launches, host run-ahead); this is the fit a virtual-clock study needs.
    samples: measure_stage_samples(...) output (its "iterations" rows: layers, tokens x layers,
    cached, non-empty experts, entries, wall ms)."""
    from scipy.optimize import nnls

    rows = samples["iterations"]
    a = np.array([r[:4] for r in rows], dtype=np.float64)
    y = np.array([r[5] for r in rows], dtype=np.float64)
    coef, _ = nnls(a, y)
    pred = a @ coef
    ss = float(((y - y.mean()) ** 2).sum())
    med = lambda v: float(statistics.median(v)) if v else 0.0  # noqa: E731
    router = min(med(samples["router"]), float(coef[0]))
    tl = sum(r[1] for r in rows)
    k_eff = (sum(r[4] for r in rows) / tl) if tl else 1.0  # expert entries per token-layer
    share = 0.0
    if stage_fit is not None:
        te = stage_fit.expert_per_entry * k_eff
        share = te / (te + stage_fit.attn_per_token) if te + stage_fit.attn_per_token > 0 else 0.0
    cm = CostModel(attn_base=float(coef[0]) - router, attn_per_token=float(coef[1]) * (1.0 - share),
                   attn_per_cached=float(coef[2]), router_cost=router, expert_base=float(coef[3]),
                   expert_per_entry=float(coef[1]) * share / k_eff if k_eff > 0 else 0.0,
                   checkpoint_cost=med(samples.get("checkpoint", [])), restore_cost=med(samples.get("restore", [])))
    rep = {"n": len(rows), "r2": 1.0 - float(((y - pred) ** 2).sum()) / ss if ss > 0 else 1.0,
           "median_abs_rel_err": float(np.median(np.abs(pred - y) / np.maximum(y, 1e-9))),
           "entries_per_token_layer": k_eff, "per_token_split_to_experts": share,
           "coef": dict(zip(["per_layer", "per_token_layer", "per_cached", "per_expert"], coef.tolist()))}
    return cm, rep


def measure_stage_samples(model, trace, max_batch_size: int = 32, scheduler: str = "qllm",
                          wall: bool = True) -> dict:
    """Run `trace` through the engine with CUDA events around every stage of `model`; returns the
    samples fit_cost_model takes.  wall=True: the serving configuration (WallClock, device-preempt
    expert stage: the host runs ahead, so an event pair brackets the stage's device time);
    wall=False: virtual clock (host-boundary expert stage, one host sync per layer, whose report
    loop then shows up in the expert stage).  Checkpoint / restore are the host time of the
    engine's _preempt and the device time of the restore gather."""
    import time as _time

    from .sim import Simulation

    sim = Simulation(trace, model=model, scheduler=scheduler, max_batch_size=max_batch_size,
                     clock=WallClock() if wall else None)
    eng = sim.engine
    out = {"attention": [], "router": [], "experts": [], "checkpoint": [], "restore": []}
    pending = []  # (kind, start event, end event, extra) resolved after the run

    def timed(kind, fn, extra):
        def wrap(*a, **kw):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            r = fn(*a, **kw)
            e.record()
            pending.append((kind, s, e, extra(a, r)))
            return r
        return wrap

    cache = sim.cache
    att, route, perm, run, comb = (model.attention_batch, model.route_batch, model.permute, model.run_experts,
                                   model.combine_batch)
    # per-iteration feature sums of the reference's linear model (engine.py:48-88) and the
    # iteration's wall time, for the iteration-level fit
    it = {"f": None}
    out["iterations"] = []

    def att_extra(a, r):
        T, cached = sum(m.n for m in a[2]), sum(cache.count(m.seq.cache_handle, a[0]) for m in a[2])
        if it["f"] is not None:
            f = it["f"]
            f[0] += 1
            f[1] += T
            f[2] += cached
        return T, cached

    model.attention_batch = timed("attention", att, att_extra)
    model.route_batch = timed("router", route, lambda a, r: None)
    state = {}

    def perm_hook(*a, **kw):
        s = torch.cuda.Event(enable_timing=True)
        s.record()
        r = perm(*a, **kw)
        state["start"] = s
        state["offsets"] = r[1]
        return r

    def comb_hook(*a, **kw):
        r = comb(*a, **kw)
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        off = state["offsets"].tolist()
        counts = [off[i + 1] - off[i] for i in range(len(off) - 1)]
        pending.append(("experts", state["start"], e, (sum(1 for c in counts if c), sum(counts))))
        if it["f"] is not None:
            it["f"][3] += sum(1 for c in counts if c)
            it["f"][4] += sum(counts)
        return r

    model.permute, model.combine_batch = perm_hook, comb_hook
    pre, init = eng._preempt, eng._init_state

    def pre_hook(*a, **kw):
        t = _time.perf_counter()
        r = pre(*a, **kw)
        out["checkpoint"].append((_time.perf_counter() - t) * 1e3)
        return r

    def init_hook(seqs):
        resumed = seqs[0].checkpoint is not None
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = init(seqs)
        e.record()
        if resumed:
            pending.append(("restore", s, e, len(seqs)))
        return r

    execute = eng.execute

    def exec_hook(*a, **kw):
        it["f"] = [0, 0, 0, 0, 0]
        torch.cuda.synchronize()
        t = _time.perf_counter()
        r = execute(*a, **kw)
        torch.cuda.synchronize()
        if r.__class__.__name__ == "Completed":  # whole iterations only
            out["iterations"].append(tuple(it["f"]) + ((_time.perf_counter() - t) * 1e3,))
        it["f"] = None
        return r

    eng._preempt, eng._init_state, eng.execute = pre_hook, init_hook, exec_hook
    try:
        sim.run()
    finally:
        model.attention_batch, model.route_batch, model.permute, model.run_experts, model.combine_batch = (
            att, route, perm, run, comb)
        eng._preempt, eng._init_state, eng.execute = pre, init, execute
    torch.cuda.synchronize()
    for kind, s, e, extra in pending:
        ms = s.elapsed_time(e)
        if kind == "attention":
            out["attention"].append((extra[0], extra[1], ms))
        elif kind == "router":
            out["router"].append(ms)
        elif kind == "experts":
            out["experts"].append((extra[0], extra[1], ms))
        else:
            out["restore"].append(ms / max(1, extra))
    return out


def main(argv=None) -> int:
    """python -m paper_2503_09304_b200.calibrate [--model mixtral|qwen] [--repeats N] [--out F]:
    the B200-calibrated CostModel of a random-init bf16 decoder (JSON)."""
    import argparse
    import json

    from .mixtral import MIXTRAL_8X7B, QWEN15_MOE_A27B, DecoderMoEModel

    ap = argparse.ArgumentParser(description=main.__doc__)
    ap.add_argument("--model", choices=("mixtral", "qwen"), default="mixtral")
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args(argv)
    model = DecoderMoEModel(QWEN15_MOE_A27B if args.model == "qwen" else MIXTRAL_8X7B)
    scaled, info = b200_cost_model(model, repeats=args.repeats)
    rec = {"model": model.config.name, "canonical_iteration": {"members": CALIBRATION_BATCH,
                                                                "context_tokens": CANONICAL_CONTEXT,
                                                                "layers": model.config.num_layers},
           "wall_ms": info["wall_ms"], "wall_ms_all": info["wall_ms_all"],
           "virtual_ms_default_cost_model": info["virtual_ms"], "scale": info["scale"],
           "cost_model": scaled.__dict__}
    text = json.dumps(rec, indent=1)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text + "\n")
    print(text)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
