import sys, time
sys.path.insert(0, ".")
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2503_09304_b200.engine import WallClock
from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, DecoderMoEModel
from paper_2503_09304_b200.sim import Simulation
from paper_2503_09304_b200.workload import WorkloadSpec, trace_for_rate
m = DecoderMoEModel(MIXTRAL_8X7B)
tr = trace_for_rate(WorkloadSpec(duration_s=3.0, output_mean=40), 7.0, seed=0)
for dp in (False, True):
    sim = Simulation(tr, model=m, scheduler="baseline", max_batch_size=32, clock=WallClock())
    sim.engine._device_preempt = dp
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t = time.time(); res = sim.run(); wall = time.time() - t
    dec = sorted(r.duration_ms for r in res.probes.iterations if r.phase.name == "DECODE")
    print(f"=== dp={dp} wall {wall:.1f}s decode median {dec[len(dec)//2]:.1f} ms, iters {len(dec)}")
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=50))
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12, max_name_column_width=50))
    del sim
