"""Serving-time breakdown (Mixtral plugin, or Qwen with --qwen; paper workload, wall clock): a short run under torch.profiler
(CUPTI kernel timeline -> GPU busy vs span, per decode iteration) and a second one under cProfile (host
hot spots).  python tools/serve_profile.py [rate] [seconds] [scheduler] > out.txt"""
import cProfile
import io
import json
import pstats
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, QWEN15_MOE_A27B, DecoderMoEModel  # noqa: E402
from paper_2503_09304_b200.serving import compare, warm_up  # noqa: E402

rate = float(sys.argv[1]) if len(sys.argv) > 1 else 7.0
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
sched = sys.argv[3] if len(sys.argv) > 3 else "baseline"
m = DecoderMoEModel(QWEN15_MOE_A27B if "--qwen" in sys.argv else MIXTRAL_8X7B)
warm_up(m)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    out = compare(m, rate, secs, schedulers=(sched,), kv_capacity_bytes=40 * 1024**3)
r = out["fcfs" if sched == "baseline" else sched]
ev = sorted((e.time_range.start, e.time_range.end) for e in prof.events()
            if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0)
busy, cs, ce = 0.0, None, None
for s, e in ev:
    if ce is None or s > ce:
        if ce is not None:
            busy += ce - cs
        cs, ce = s, e
    else:
        ce = max(ce, e)
if ce is not None:
    busy += ce - cs
span = ev[-1][1] - ev[0][0]
# idle gaps of the GPU timeline by size: short ones inside an iteration (host enqueue behind the GPU),
# long ones at iteration boundaries (token sync -> scheduler -> next iteration's first launch)
gaps, ce = [], None
for s, e in ev:
    if ce is not None and s > ce:
        gaps.append(s - ce)
    ce = e if ce is None else max(ce, e)
bins = {"<20us": 0.0, "20-100us": 0.0, "100-500us": 0.0, "0.5-2ms": 0.0, ">2ms": 0.0}
cnt = dict.fromkeys(bins, 0)
for g in gaps:
    k = ("<20us" if g < 20 else "20-100us" if g < 100 else "100-500us" if g < 500 else "0.5-2ms" if g < 2000
         else ">2ms")
    bins[k] += g / 1e3
    cnt[k] += 1
print(json.dumps({"rate": rate, "seconds": secs, "scheduler": sched, "gpu_busy_ms": busy / 1e3, "gpu_span_ms": span / 1e3,
                  "busy_frac": busy / span, "idle_ms_by_gap_size": bins, "gaps_by_size": cnt,
                  "decode_iter_ms_median": r["decode_iter_ms_median"],
                  "iterations": r["iterations"], "be_tokens_per_s": r["be_tokens_per_s"]}), flush=True)
if "--no-cprofile" in sys.argv:
    sys.exit(0)
pr = cProfile.Profile()
pr.enable()
compare(m, rate, secs, schedulers=(sched,), kv_capacity_bytes=40 * 1024**3)
pr.disable()
buf = io.StringIO()
pstats.Stats(pr, stream=buf).sort_stats("tottime").print_stats(30)
print(buf.getvalue()[:9000])
