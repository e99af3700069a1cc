"""Scheduler semantics (restating the reference's tests/test_sched.py intent on this module):
policy rules, exhaustive Algorithm-1 selection against a literal transcription, resume groups,
and the FCFS baseline."""

import itertools

import pytest

from paper_2503_09304_b200.core import (AdmissionError, Checkpoint, EngineReport, MemberProgress, Phase, Priority,
                                        SchedulerDirective, Stage, sequence_new)
from paper_2503_09304_b200.kvcache import UnifiedDynamicCache
from paper_2503_09304_b200.sched import BaselineScheduler, QllmScheduler, never_preempt_policy, qllm_policy

LS, BE = Priority.LATENCY_SENSITIVE, Priority.BEST_EFFORT
PREEMPT, CONT = SchedulerDirective.PREEMPT_AT_NEXT_BOUNDARY, SchedulerDirective.CONTINUE


def cache():
    import torch

    return UnifiedDynamicCache(2, (1,), torch.float32, torch.device("cpu"), entry_bytes=64, initial_pages=1)


def sched(max_batch=32, policy=qllm_policy):
    return QllmScheduler(cache(), max_batch, policy)


def arrive(s, sid, pri):
    seq = sequence_new([1, 2], pri, 4, arrival=float(sid), seq_id=sid)
    seq.cache_handle = sid
    s.cache.register(sid)
    s.dispatch_arrival(seq)
    return seq


def as_decode(s, sid, pri):
    seq = sequence_new([1, 2], pri, 4, arrival=float(sid), seq_id=sid)
    seq.cache_handle = sid
    seq.generated.append(7)
    seq.advance_phase(Phase.DECODE)
    s.sequences[sid] = seq
    s._q[(pri, Phase.DECODE)].fresh.append(sid)
    s._snap = None
    return seq


def report(priorities, stage=Stage.ATTENTION):
    prog = tuple(MemberProgress(i, p, Phase.DECODE, 1) for i, p in enumerate(priorities))
    return EngineReport(1, stage, 0, 0.0, prog)


def ckpt(layer, stage):
    import torch

    z = torch.zeros((1, 1))
    if stage is Stage.EXPERTS:
        return Checkpoint(layer, stage, z, z, torch.zeros((1, 2), dtype=torch.int32), torch.zeros((1, 2)),
                          torch.zeros((2, 1)), torch.zeros(1, dtype=torch.int32))
    return Checkpoint(layer, stage, z, z)


# ------------------------------------------------------------------------------------ policy

def test_policy_rules():
    s = sched()
    assert qllm_policy(report([BE]), s.snapshot()) is CONT
    as_decode(s, 1, LS)
    assert qllm_policy(report([BE, BE]), s.snapshot()) is PREEMPT       # LS waits, batch has no LS
    assert qllm_policy(report([BE, LS]), s.snapshot()) is CONT          # batch already serves LS
    arrive(s, 2, LS)
    assert qllm_policy(report([LS]), s.snapshot()) is PREEMPT           # fresh LS prefill always
    assert never_preempt_policy(report([BE]), s.snapshot()) is CONT


def test_arrival_policy_holds_while_admission_is_blocked():
    """Serving variant: a fresh LS prefill preempts -- unless the KV ledger just refused a prefill
    (the driver fell back to decode-only work): preempting then only drops the decode batch at its
    first report and selects it again (a preemption livelock under KV saturation)."""
    from paper_2503_09304_b200.sched import arrival_policy

    s = sched(policy=arrival_policy)
    arrive(s, 2, LS)
    assert arrival_policy(report([BE]), s.snapshot()) is PREEMPT
    snap = s.snapshot()
    s.admission_blocked = True
    assert s.snapshot() is not snap and s.snapshot().admission_blocked
    assert arrival_policy(report([BE]), s.snapshot()) is CONT
    s.admission_blocked = False
    assert arrival_policy(report([BE]), s.snapshot()) is PREEMPT
    assert qllm_policy(report([BE]), s.snapshot()) is PREEMPT  # the reference policy is unchanged


def test_snapshot_is_rebuilt_after_mutation():
    s = sched()
    snap = s.snapshot()
    assert s.snapshot() is snap
    arrive(s, 0, LS)
    assert s.snapshot() is not snap and s.snapshot().ls_prefill.fresh == (0,)


def test_dispatch_validation_and_route_output():
    s = sched()
    seq = arrive(s, 0, BE)
    with pytest.raises(AdmissionError):
        s.dispatch_arrival(seq)
    assert s.route_output(seq, 5, 10.0) is False
    assert seq.first_token_time == 10.0 and seq.phase is Phase.DECODE
    assert s.be_decode.fresh[-1] == 0
    s.be_decode.fresh.clear()
    assert s.route_output(seq, 0, 12.0) is True  # EOS finishes
    assert seq.finish_time == 12.0 and 0 in s.finished and not s.cache.has_handle(0)


# ------------------------------------------------------------------------------------ Algorithm 1

def transcription(ls_d, ls_p, be_d, be_p, cap):
    """Literal transcription of the published batch selection (paper Algorithm 1)."""
    if len(ls_d) >= cap:
        return Phase.DECODE, ls_d[:cap]
    if ls_p:
        main = ls_p[:cap]
        return Phase.PREFILL, main + be_p[: cap - len(main)]
    if ls_d:
        main = ls_d[:cap]
        return Phase.DECODE, main + be_d[: cap - len(main)]
    if be_d:
        return Phase.DECODE, be_d[:cap]
    if be_p:
        return Phase.PREFILL, be_p[:cap]
    return None


def test_algorithm_one_exhaustively():
    cap = 32
    sizes = [0, 1, cap - 1, cap, cap + 1]
    for n in itertools.product(sizes, repeat=4):
        s = sched(cap)
        nid = 0
        buckets = {}
        for (pri, ph), cnt in zip(((LS, Phase.DECODE), (LS, Phase.PREFILL), (BE, Phase.DECODE), (BE, Phase.PREFILL)), n):
            ids = []
            for _ in range(cnt):
                if ph is Phase.DECODE:
                    as_decode(s, nid, pri)
                else:
                    arrive(s, nid, pri)
                ids.append(nid)
                nid += 1
            buckets[(pri, ph)] = ids
        want = transcription(buckets[(LS, Phase.DECODE)], buckets[(LS, Phase.PREFILL)], buckets[(BE, Phase.DECODE)],
                             buckets[(BE, Phase.PREFILL)], cap)
        got = s.get_next_batch()
        if want is None:
            assert got is None
            continue
        assert (got.phase, got.seq_ids) == want, n
        if n[0] or n[1]:
            assert any(s.sequences[i].priority is LS for i in got.seq_ids)


# ------------------------------------------------------------------------------------ resume groups

def test_resume_groups_merge_matching_positions_and_sort_by_admission():
    s = sched()
    be = [as_decode(s, i, BE) for i in (0, 1)]
    ls = [as_decode(s, 2, LS)]
    for q in (s.be_decode, s.ls_decode):
        q.fresh.clear()
    for seq in be + ls:
        seq.checkpoint = ckpt(1, Stage.EXPERTS)
    s.on_preempted({0: be[0].checkpoint, 1: be[1].checkpoint, 2: ls[0].checkpoint})
    sel = s.get_next_batch()
    assert sel.resume and sel.phase is Phase.DECODE and sel.seq_ids == [0, 1, 2]


def test_mismatched_positions_do_not_merge():
    s = sched()
    a, b = as_decode(s, 0, LS), as_decode(s, 1, BE)
    s.ls_decode.fresh.clear()
    s.be_decode.fresh.clear()
    a.checkpoint, b.checkpoint = ckpt(1, Stage.EXPERTS), ckpt(2, Stage.ROUTER)
    s.on_preempted({0: a.checkpoint, 1: b.checkpoint})
    assert s.get_next_batch().seq_ids == [0]
    assert s.get_next_batch().seq_ids == [1]


def test_pre_attention_checkpoint_rejoins_fresh_queue_head():
    s = sched()
    arrive(s, 0, BE)
    seq = arrive(s, 1, BE)
    s.be_prefill.fresh.remove(1)
    seq.checkpoint = ckpt(0, Stage.ATTENTION)
    s.on_preempted({1: seq.checkpoint})
    assert list(s.be_prefill.fresh) == [1, 0] and seq.checkpoint is None


def test_fresh_ls_prefill_precedes_ls_resume_group():
    s = sched()
    old = arrive(s, 0, LS)
    s.ls_prefill.fresh.clear()
    old.checkpoint = ckpt(0, Stage.ROUTER)
    s.on_preempted({0: old.checkpoint})
    arrive(s, 1, LS)
    sel = s.get_next_batch()
    assert sel.seq_ids == [1] and not sel.resume


def test_requeue_front_keeps_order():
    s = sched()
    for i in range(4):
        arrive(s, i, BE)
    sel = s.get_next_batch()
    s.requeue_front(sel.seq_ids[2:])
    assert list(s.be_prefill.fresh) == [2, 3]


# ------------------------------------------------------------------------------------ baseline

def test_baseline_fcfs_ignores_priority_and_waits_for_finishers():
    b = BaselineScheduler(cache(), max_batch_size=2)
    seqs = []
    for i, pri in enumerate((BE, LS, LS)):
        seq = sequence_new([1], pri, 3, float(i), seq_id=i)
        seq.cache_handle = i
        b.cache.register(i)
        b.dispatch_arrival(seq)
        seqs.append(seq)
    sel = b.get_next_batch()
    assert sel.phase is Phase.PREFILL and sel.seq_ids == [0, 1]
    for s in seqs[:2]:
        b.route_output(s, 5, 1.0)
    sel = b.get_next_batch()
    assert sel.phase is Phase.DECODE and sel.seq_ids == [0, 1]  # batch full: 2 waits
    b.route_output(seqs[0], 0, 2.0)  # EOS frees a slot
    assert b.get_next_batch().seq_ids == [2]
    assert b.on_engine_report(report([BE])) is CONT
    with pytest.raises(AdmissionError):
        b.on_preempted({})


def test_serving_knob_be_prefill_into_free_slots():
    """Off (reference Algorithm 1): fresh BE prefills wait behind BE decodes.  On: they run as soon
    as the decode population leaves batch slots free, capped at the free slots."""
    for knob in (False, True):
        s = QllmScheduler(cache(), 4, qllm_policy, be_prefill_into_free_slots=knob)
        for i in range(2):
            as_decode(s, i, BE)
        for i in range(10, 15):
            arrive(s, i, BE)
        sel = s.get_next_batch()
        if knob:
            assert sel.phase is Phase.PREFILL and sel.seq_ids == [10, 11]
            assert s.get_next_batch(decode_only=True).seq_ids == [0, 1]  # decode-only never takes prefills
        else:
            assert sel.phase is Phase.DECODE and sel.seq_ids == [0, 1]


def test_serving_knob_fill_ls_prefill():
    for fill in (True, False):
        s = QllmScheduler(cache(), 8, qllm_policy, fill_ls_prefill=fill)
        arrive(s, 1, BE)
        arrive(s, 2, LS)
        arrive(s, 3, BE)
        sel = s.get_next_batch()
        assert sel.seq_ids == ([2, 1, 3] if fill else [2])
