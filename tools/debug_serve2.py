import sys, time, statistics
sys.path.insert(0, ".")
import torch
from paper_2503_09304_b200.engine import WallClock
from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, DecoderMoEModel
from paper_2503_09304_b200.sim import Simulation
from paper_2503_09304_b200.workload import WorkloadSpec, trace_for_rate
m = DecoderMoEModel(MIXTRAL_8X7B)
tr = trace_for_rate(WorkloadSpec(duration_s=8.0), 7.0, seed=0)
for dp in (False, True):
    sim = Simulation(tr, model=m, scheduler="baseline", max_batch_size=32, clock=WallClock())
    sim.engine._device_preempt = dp
    t = time.time(); res = sim.run(); wall = time.time() - t
    dec = [(r.size, r.duration_ms) for r in res.probes.iterations if r.phase.name == "DECODE"]
    pre = [(r.size, r.duration_ms) for r in res.probes.iterations if r.phase.name == "PREFILL"]
    by = {}
    for n, d in dec: by.setdefault(n // 8 * 8, []).append(d)
    print(f"dp={dp} wall {wall:.1f}s decode iters {len(dec)} median {statistics.median(d for _, d in dec):.1f} ms; by size {[(k, round(statistics.median(v),1), len(v)) for k, v in sorted(by.items())]}; prefill {len(pre)} median {statistics.median(d for _, d in pre):.1f}", flush=True)
    del sim
