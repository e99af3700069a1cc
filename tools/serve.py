"""Wall-clock serving run of a Mixtral/Qwen-shaped model on one B200: QLLM vs FCFS baseline on the
paper workload (Poisson arrivals, 20% LS, lognormal lengths; reference workload.py defaults,
trace seeding of reference cli.py:172-190).  Prints one JSON object per (scheduler, rate)."""
import argparse, json, sys, time
sys.path.insert(0, ".")
import torch
from dataclasses import replace
from paper_2503_09304_b200.engine import WallClock, CostModel
from paper_2503_09304_b200.metrics import aggregate
from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, QWEN15_MOE_A27B, DecoderMoEModel
from paper_2503_09304_b200.sim import Simulation
from paper_2503_09304_b200.workload import WorkloadSpec, trace_for_rate


def run(model, trace, sched, mbs, slo_ms):
    torch.cuda.synchronize()
    sim = Simulation(trace, model=model, scheduler=sched, max_batch_size=mbs, clock=WallClock())
    t0 = time.perf_counter()
    res = sim.run()
    wall = time.perf_counter() - t0
    rep = aggregate(res.records, slo_ms, res.makespan_ms)
    it = [r for r in res.probes.iterations if not r.preempted and r.phase.name == "DECODE"]
    out = {"scheduler": sched, "jobs": rep.jobs, "makespan_ms": res.makespan_ms, "wall_s": wall,
           "ls_jobs": rep.ls.jobs if rep.ls else 0,
           "ls_ttft_p50_ms": rep.ls.median_ttft_ms if rep.ls else None,
           "ls_ttft_p99_ms": rep.ls.p99_ttft_ms if rep.ls else None,
           "ls_mean_turnaround_ms": rep.ls.mean_turnaround_ms if rep.ls else None,
           "ls_slo_attainment": rep.ls.slo_attainment if rep.ls else None,
           "be_ttft_p50_ms": rep.be.median_ttft_ms if rep.be else None,
           "be_mean_turnaround_ms": rep.be.mean_turnaround_ms if rep.be else None,
           "be_tokens_per_s": rep.be_tokens_per_s, "ls_tokens_per_s": rep.ls_tokens_per_s,
           "completion_rate_jps": rep.completion_rate_jps, "preemptions": res.probes.preemptions,
           "decode_iter_ms_median": sorted(r.duration_ms for r in it)[len(it) // 2] if it else None,
           "engine": res.engine_stats}
    del sim
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="mixtral", choices=["mixtral", "qwen"])
    ap.add_argument("--rates", default="7")
    ap.add_argument("--duration", type=float, default=20.0)
    ap.add_argument("--schedulers", default="baseline,qllm")
    ap.add_argument("--mbs", type=int, default=32)
    ap.add_argument("--slo-ms", type=float, default=3000.0)
    ap.add_argument("--layers", type=int, default=0, help="debug only: fewer layers")
    args = ap.parse_args()
    cfg = MIXTRAL_8X7B if args.model == "mixtral" else QWEN15_MOE_A27B
    if args.layers:
        cfg = replace(cfg, num_layers=args.layers)
    t = time.perf_counter()
    model = DecoderMoEModel(cfg)
    torch.cuda.synchronize()
    print(json.dumps({"init_s": time.perf_counter() - t, "model": cfg.name, "mem_gb": torch.cuda.memory_allocated() / 1e9}), flush=True)
    wl = WorkloadSpec(duration_s=args.duration)
    # warm-up: a few short jobs through every code path (prefill, decode, preemption)
    warm = trace_for_rate(replace(wl, duration_s=2.0, prompt_mean=64, output_mean=8), 4.0, seed=99)
    run(model, warm, "qllm", args.mbs, args.slo_ms)
    for rate in [float(r) for r in args.rates.split(",")]:
        trace = trace_for_rate(wl, rate, seed=0)
        for sched in args.schedulers.split(","):
            out = run(model, trace, sched, args.mbs, args.slo_ms)
            out.update({"rate": rate, "model": cfg.name, "trace_jobs": len(trace), "duration_s": args.duration})
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
