"""Wall-clock serving runs (QLLM vs FCFS on the same kernels) and their summary metrics.

Used by tools/serve.py (rate sweeps) and bench.py (the LS TTFT / BE tokens/s half of the
headline metric).  The trace is the paper workload (reference workload.py defaults, Poisson
arrivals, 20% LS) seeded per rate exactly like the reference runner (cli.py:172-190)."""

from __future__ import annotations

import gc
import time
from dataclasses import replace
from typing import Optional

import torch

from .engine import WallClock
from .metrics import aggregate
from .sim import Simulation
from .workload import WorkloadSpec, trace_for_rate


def kv_pages_for(model, capacity_bytes: float, max_batch_size: int) -> dict:
    """Page-pool kwargs sized for the admission ledger's capacity up front (one allocation, no
    grow-and-copy next to the model): capacity / (page tokens x layers x entry bytes) full pages
    plus partially filled pages for 8x the batch size of resident sequences (more resident
    sequences than that -- the ledger admits up to capacity / lifetime footprint of them -- grow
    the pool by at most half its size, clamped to max_pages, kvcache._ensure_pages)."""
    kw = dict(getattr(model, "kv_page_kwargs", {}))
    page = kw.get("page_size", 16)
    per_token = model.config.num_layers * model.kv_entry_bytes()
    full = int(-(-capacity_bytes // (page * per_token)))
    partial = min(int(capacity_bytes // per_token), 8 * max_batch_size)
    kw["initial_pages"] = full + partial
    return kw


def serve_once(model, trace, scheduler: str, max_batch_size: int = 32, slo_ms: float = 3000.0,
               kv_capacity_bytes: Optional[float] = None, clock_factory=WallClock) -> dict:
    """clock_factory: WallClock (one GPU) or, for expert-parallel serving, a LockstepClock shared
    by the ranks (ep_serving.py); every rank then runs this same call."""
    torch.cuda.synchronize()
    extra = {}
    if kv_capacity_bytes is not None:
        extra = {"cache_capacity_bytes": kv_capacity_bytes,
                 "kv_page_kwargs": kv_pages_for(model, kv_capacity_bytes, max_batch_size)}
    sim = Simulation(trace, model=model, scheduler=scheduler, max_batch_size=max_batch_size, clock=clock_factory(),
                     **extra)
    # the engine's per-layer host objects are short-lived and acyclic; the cyclic collector's
    # generation-0 passes (triggered by allocation counts, i.e. every few layers) only add latency
    # to the host path that feeds the GPU, so it is paused for the run and run once after it
    gc.collect()
    gc_was = gc.isenabled()
    gc.disable()
    t0 = time.perf_counter()
    try:
        res = sim.run()
    finally:
        if gc_was:
            gc.enable()
    wall = time.perf_counter() - t0
    rep = aggregate(res.records, slo_ms, res.makespan_ms)
    dec = sorted(r.duration_ms for r in res.probes.iterations if not r.preempted and r.phase.name == "DECODE")
    ls, be = rep.ls, rep.be
    out = {
        "scheduler": scheduler, "jobs": rep.jobs, "makespan_ms": res.makespan_ms, "wall_s": wall,
        "ls_jobs": ls.jobs if ls else 0,
        "ls_ttft_p50_ms": ls.median_ttft_ms if ls else None, "ls_ttft_p99_ms": ls.p99_ttft_ms if ls else None,
        "ls_mean_turnaround_ms": ls.mean_turnaround_ms if ls else None,
        "ls_slo_attainment": ls.slo_attainment if ls else None,
        "be_ttft_p50_ms": be.median_ttft_ms if be else None,
        "be_mean_turnaround_ms": be.mean_turnaround_ms if be else None,
        "be_tokens_per_s": rep.be_tokens_per_s, "ls_tokens_per_s": rep.ls_tokens_per_s,
        "completion_rate_jps": rep.completion_rate_jps, "preemptions": res.probes.preemptions,
        "decode_iter_ms_median": dec[len(dec) // 2] if dec else None,
        "engine": res.engine_stats,
        "preempt_positions": sim.engine.preemption_positions(),
    }
    # where the time went: busy time per phase, decode batch sizes, idle time (no work queued)
    its = res.probes.iterations
    dit = [r for r in its if r.phase.name == "DECODE"]
    pit = [r for r in its if r.phase.name == "PREFILL"]
    busy = sum(r.duration_ms for r in its)
    out["iterations"] = {
        "decode": len(dit), "decode_ms": sum(r.duration_ms for r in dit),
        "decode_members_mean": sum(r.size for r in dit) / len(dit) if dit else 0.0,
        "prefill": len(pit), "prefill_ms": sum(r.duration_ms for r in pit),
        "preempted": sum(1 for r in its if r.preempted), "idle_ms": res.makespan_ms - busy,
    }
    if dec and ls:
        # the paper's SLO is 10x an A100 decode iteration; the B200 analogue is 10x
        # this run's measured median decode iteration
        scaled = 10.0 * dec[len(dec) // 2]
        out["scaled_slo_ms"] = scaled
        out["ls_scaled_slo_attainment"] = aggregate(res.records, scaled, res.makespan_ms).ls.slo_attainment
    del sim, res
    gc.collect()  # the run's KV page pools sit in reference cycles; free them before the next run
    torch.cuda.empty_cache()
    return out


def warm_up(model, max_batch_size: int = 32, clock_factory=WallClock) -> None:
    """Short run through prefill, decode and preemption so later timings exclude one-time init."""
    warm = trace_for_rate(WorkloadSpec(duration_s=2.0, prompt_mean=64, output_mean=8), 4.0, seed=99)
    serve_once(model, warm, "qllm", max_batch_size, clock_factory=clock_factory)


def compare(model, rate: float, duration_s: float, seed: int = 0, max_batch_size: int = 32,
            slo_ms: float = 3000.0, schedulers=("baseline", "qllm"), workload: Optional[WorkloadSpec] = None,
            kv_capacity_bytes: Optional[float] = None, clock_factory=WallClock) -> dict:
    trace = trace_for_rate(replace(workload or WorkloadSpec(), duration_s=duration_s), rate, seed=seed)
    out = {"rate": rate, "duration_s": duration_s, "jobs": len(trace), "slo_ms": slo_ms,
           "kv_capacity_gib": (kv_capacity_bytes or 8 * 1024**3) / 1024**3}
    for s in schedulers:
        out["fcfs" if s == "baseline" else s] = serve_once(model, trace, s, max_batch_size, slo_ms, kv_capacity_bytes,
                                                            clock_factory)
    return out
