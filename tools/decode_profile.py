"""Where a serving decode iteration's time goes (32-layer Mixtral / 24-layer Qwen plugin, 32 members with
180-token contexts, wall-clock engine with device preemption): torch.profiler (CUPTI) kernel timeline of
a few iterations -> wall ms per iteration, GPU-busy ms (union of kernel intervals), and the per-kernel
totals.  python tools/decode_profile.py [qwen] > out.json"""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2503_09304_b200.core import Phase, Priority, SchedulerDirective, batch_form, sequence_new  # noqa: E402
from paper_2503_09304_b200.engine import InferenceEngine, WallClock  # noqa: E402
from paper_2503_09304_b200.kvcache import UnifiedDynamicCache  # noqa: E402
from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, QWEN15_MOE_A27B, DecoderMoEModel  # noqa: E402

cfg = QWEN15_MOE_A27B if "qwen" in sys.argv[1:] else MIXTRAL_8X7B
m = DecoderMoEModel(cfg)
cache = UnifiedDynamicCache(cfg.num_layers, m.kv_row_shape(), m.kv_dtype, m.device, m.kv_entry_bytes(), 64e9,
                            **m.kv_page_kwargs)
eng = InferenceEngine(m, cache, WallClock(), max_batch_size=32)
seqs = []
for i in range(32):
    s = sequence_new(list(range(1, 181)), Priority.BEST_EFFORT, 64, 0.0, seq_id=i)
    s.cache_handle = i
    cache.register(i)
    seqs.append(s)


def cont(r):
    return SchedulerDirective.CONTINUE


out = eng.execute(batch_form(seqs, Phase.PREFILL, 32, eng.next_batch_id()), seqs, cont)
for s in seqs:
    s.generated.append(out.tokens[s.id])
    s.advance_phase(Phase.DECODE)


def step():
    o = eng.execute(batch_form(seqs, Phase.DECODE, 32, eng.next_batch_id()), seqs, cont)
    for s in seqs:
        s.generated.append(o.tokens[s.id])


for _ in range(4):
    step()
torch.cuda.synchronize()
N = 5
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t = time.perf_counter()
    for _ in range(N):
        step()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) * 1e3 / N
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
iv = sorted((e.time_range.start, e.time_range.end) for e in ev)
busy, cur_s, cur_e = 0.0, None, None
for s, e in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
if cur_e is not None:
    busy += cur_e - cur_s
span = (iv[-1][1] - iv[0][0]) if iv else 0.0
agg = {}
for e in ev:
    name = e.name.split("(")[0].replace("void ", "")[:80]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += e.time_range.elapsed_us()
top = sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]
print(json.dumps({"model": cfg.name, "members": 32, "context": 180, "iterations": N,
                  "wall_ms_per_iteration": wall, "gpu_busy_ms_per_iteration": busy / 1e3 / N,
                  "gpu_span_ms_per_iteration": span / 1e3 / N,
                  "kernels_per_iteration": len(ev) / N,
                  "top_kernels_ms_per_iteration": {k: {"launches": v[0] / N, "ms": v[1] / 1e3 / N} for k, v in top}},
                 indent=1))
