"""Device-resident preemption without a host round trip (north_star item 4): an LS arrival raises
the running iteration's preempt flag from another thread; the grouped expert launch stops at its
next expert boundary; everything the run-ahead host already enqueued behind that boundary is void
(later launches claim nothing, guarded K/V appends skip); the host rolls the iteration back to the
boundary one layer later.  Tokens must stay identical to an undisturbed run (preemption
transparency, reference tests/test_engine.py:249-300, tests/test_sim.py:40-52)."""

import threading
import time
from dataclasses import replace

import pytest
import torch

from replay import load_log, trace_of
from paper_2503_09304_b200 import kernels as K
from paper_2503_09304_b200.engine import WallClock
from paper_2503_09304_b200.model import ModelConfig
from paper_2503_09304_b200.sim import Simulation

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("T,d,F,E,k", [(32, 1024, 2048, 8, 2), (1200, 1024, 2048, 8, 2), (3000, 1024, 1408, 60, 4)])
def test_early_stop_voids_the_flag_and_later_launches(cuda, T, d, F, E, k):
    g = torch.Generator(device="cuda").manual_seed(T)
    x = torch.randn((T, d), device="cuda", generator=g).bfloat16()
    gu = (torch.randn((E, 2 * F, d), device="cuda", generator=g) * d ** -0.5).bfloat16()
    dn = (torch.randn((E, d, F), device="cuda", generator=g) * F ** -0.5).bfloat16()
    ids = torch.stack([torch.randperm(E, device="cuda", generator=g)[:k].sort().values for _ in range(T)]).int()
    perm, offsets, xp = K.permute(ids, E, x=x)
    y = torch.zeros((T * k, d), dtype=torch.bfloat16, device="cuda")
    flag = torch.full((1,), 2, dtype=torch.int32, device="cuda")  # stop at the first boundary >= 2
    cur = torch.zeros(1, dtype=torch.int32, device="cuda")
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, preempt_flag=flag, cursor_out=cur)
    torch.cuda.synchronize()
    stop = int(cur)
    assert 2 <= stop < E
    assert int(flag) == -1  # the launch stopped early: the iteration is void from here
    before = y.clone()
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, e_begin=stop, preempt_flag=flag, cursor_out=cur)
    torch.cuda.synchronize()
    assert int(cur) == stop and torch.equal(y, before)  # a voided launch claims nothing
    # resuming under a fresh flag completes the layer
    flag.zero_()
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, y, e_begin=stop, preempt_flag=flag, cursor_out=cur)
    full = torch.zeros_like(y)
    K.expert_ffn(K.EXPERT_SWIGLU, xp, offsets, perm, gu, dn, full)
    torch.cuda.synchronize()
    assert int(cur) == E and int(flag) == 0
    R = int(offsets[-1])
    assert torch.equal(y[perm[:R].long()], full[perm[:R].long()])


def test_guarded_kv_append(cuda):
    pool = torch.zeros((64, 8), dtype=torch.bfloat16, device="cuda")
    rows = torch.randn((5, 8), device="cuda").bfloat16()
    slots = torch.tensor([3, 9, 17, 40, 63], dtype=torch.int32, device="cuda")
    guard = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    K.kv_append(pool, slots, rows, guard=guard)
    assert not pool.any()
    guard.fill_(1)  # a raised (not yet void) flag still appends: attention precedes the boundary
    K.kv_append(pool, slots, rows, guard=guard)
    assert torch.equal(pool[slots.long()], rows)


class _Flagger:
    """Raises the engine's arrival flag at random moments (every 0.1-1.5 ms) while a run goes on:
    far more often than LS requests arrive, so the rollback path runs at every layer position."""

    def __init__(self, engine, seed=0):
        self.engine, self.stop = engine, threading.Event()
        self.rng = torch.Generator().manual_seed(seed)
        self.t = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self.stop.is_set():
            time.sleep(0.0001 + 0.0014 * float(torch.rand(1, generator=self.rng)))
            self.engine.raise_arrival_flag()

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join()


@pytest.mark.parametrize("name", ["traceA_qllm", "traceB_qllm"])
def test_arrival_flags_are_transparent_on_the_reference_traces(cuda, name):
    """f64 toy model (reference parameters), wall clock, QLLM policy with its arrival watcher plus
    spurious flags: every sequence's tokens equal the reference's."""
    rec = load_log(name)
    sim = Simulation(trace_of(rec), model_config=ModelConfig(**rec["model"]), scheduler="qllm",
                     max_batch_size=rec["max_batch_size"], clock=WallClock())
    with _Flagger(sim.engine):
        res = sim.run()
    pos = sim.engine.preemption_positions()
    print(name, pos, sim.engine.stats)
    assert pos.get("EXPERT_DEVICE_FLAG", 0) > 0
    # report elision was on (wall clock, built-in policy, arrival watcher, no log): the reports after
    # each iteration's first CONTINUE were answered without the callback, and the rollback reports
    # of the flag-stopped launches still reached the scheduler
    assert sim.engine.elide_reports and sim.engine.stats["reports_elided"] > 0
    assert {str(k): s.generated for k, s in sorted(res.sequences.items())} == rec["tokens"]


def test_arrival_flags_are_transparent_on_the_bf16_decoder(cuda):
    """bf16 Mixtral-shaped 4-layer decoder (paged KV with guarded appends, tcgen05 experts, flash
    attention): greedy tokens under spurious arrival flags equal an undisturbed run's.  Batches of
    one sequence keep every GEMM's row count independent of the schedule (cuBLAS and the K-split
    decode path may round differently at other batch sizes), so tokens are comparable bit for bit."""
    from paper_2503_09304_b200.mixtral import MIXTRAL_8X7B, DecoderMoEModel
    from paper_2503_09304_b200.workload import WorkloadSpec, trace_for_rate

    cfg = replace(MIXTRAL_8X7B, name="mixtral-small", num_layers=4, hidden_dim=1024, ffn_dim=2048, n_heads=8,
                  n_kv_heads=2, head_dim=128, vocab_size=1000, max_position=2048)
    model = DecoderMoEModel(cfg, seed=5)
    trace = trace_for_rate(WorkloadSpec(duration_s=1.5, prompt_mean=40, prompt_bounds=(4, 200), output_mean=12,
                                        output_bounds=(1, 24)), 12.0, seed=3)

    def run(flagged):
        sim = Simulation(trace, model=model, scheduler="qllm", max_batch_size=1, clock=WallClock())
        if flagged:
            with _Flagger(sim.engine, seed=1):
                res = sim.run()
        else:
            res = sim.run()
        return {k: s.generated for k, s in res.sequences.items()}, sim.engine

    base, _ = run(False)
    got, eng = run(True)
    pos = eng.preemption_positions()
    print(pos, eng.stats)
    assert pos.get("EXPERT_DEVICE_FLAG", 0) > 0
    assert got == base
