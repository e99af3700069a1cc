"""Time decode iterations of the 32-layer Mixtral plugin through the engine (dev diagnostic)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2503_09304_b200.core import Phase, Priority, SchedulerDirective, batch_form, sequence_new
from paper_2503_09304_b200.engine import InferenceEngine, VirtualClock, WallClock
from paper_2503_09304_b200.kvcache import UnifiedDynamicCache
from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, QWEN15_MOE_A27B, DecoderMoEModel

cfg = QWEN15_MOE_A27B if "qwen" in sys.argv[1:] else MIXTRAL_8X7B
m = DecoderMoEModel(cfg)
for dp in (False, True):
    cache = UnifiedDynamicCache(cfg.num_layers, m.kv_row_shape(), m.kv_dtype, m.device, m.kv_entry_bytes(), 64e9, **m.kv_page_kwargs)
    eng = InferenceEngine(m, cache, WallClock(), max_batch_size=32, device_preempt=dp)
    seqs = []
    for i in range(32):
        s = sequence_new(list(range(1, 181)), Priority.BEST_EFFORT, 64, 0.0, seq_id=i)
        s.cache_handle = i
        cache.register(i)
        seqs.append(s)
    cont = lambda r: SchedulerDirective.CONTINUE
    out = eng.execute(batch_form(seqs, Phase.PREFILL, 32, eng.next_batch_id()), seqs, cont)
    for s in seqs:
        s.generated.append(out.tokens[s.id]); s.advance_phase(Phase.DECODE)
    ts, gs = [], []
    import os, cProfile, pstats, io
    prof = cProfile.Profile() if os.environ.get("PROF") and dp else None
    for it in range(12):
        if prof is not None and it == 2:
            prof.enable()
        torch.cuda.synchronize(); t = time.perf_counter()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = eng.execute(batch_form(seqs, Phase.DECODE, 32, eng.next_batch_id()), seqs, cont)
        b.record(); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3); gs.append(a.elapsed_time(b))
        for s in seqs:
            s.generated.append(out.tokens[s.id])
    if prof is not None:
        prof.disable()
        buf = io.StringIO()
        pstats.Stats(prof, stream=buf).sort_stats("tottime").print_stats(30)
        print(buf.getvalue()[:7000])
    print(f"{cfg.name} device_preempt={dp}: decode iteration ms {sorted(ts)[len(ts)//2]:.2f} "
          f"(GPU span {sorted(gs)[len(gs)//2]:.2f})", flush=True)
