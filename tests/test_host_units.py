"""Workload, metrics, core types and the paged-cache ledger (CPU): the reference's unit-test
intent (tests/test_workload.py, test_metrics.py, test_core.py, test_model.py cache tests)
restated against this package, plus trace parity with the reference's generator."""

import json
import math

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2503_09304_b200.core import (CacheCapacityError, Phase, Priority, Stage, StateCorruptionError, batch_form,
                                        sequence_new)
from paper_2503_09304_b200.kvcache import UnifiedDynamicCache
from paper_2503_09304_b200.metrics import (JOBS_CSV_HEADER, MetricsRecorder, aggregate, jobs_csv_lines,
                                           nearest_rank, summary_row, SUMMARY_FIELDS)
from paper_2503_09304_b200.workload import WorkloadSpec, generate, load_trace, save_trace, trace_for_rate


def test_traces_equal_the_reference_generator():
    """Every golden log embeds the reference-generated trace; regenerate it here."""
    import gzip

    with gzip.open(GOLDEN / "logs" / "traceA_qllm.json.gz", "rt") as fh:
        want = json.load(fh)["trace"]
    got = trace_for_rate(WorkloadSpec(ls_fraction=0.25, prompt_mean=32, prompt_sigma=0.8, prompt_bounds=(4, 128),
                                      output_mean=16, output_sigma=0.9, output_bounds=(1, 48)), 16.0, seed=2,
                         jobs_per_run=16)
    assert [[r.id, r.arrival_ms, r.priority.tag, r.prompt_len, r.max_new_tokens, r.prompt_seed] for r in got] == want
    for seed in range(3):
        with gzip.open(GOLDEN / "logs" / f"random{seed}_qllm.json.gz", "rt") as fh:
            want = json.load(fh)["trace"]
        got = generate(WorkloadSpec(arrival_rate=40.0, duration_s=0.3, seed=seed, ls_fraction=0.3, prompt_mean=6,
                                    prompt_sigma=0.6, prompt_bounds=(2, 16), output_mean=3, output_sigma=0.5,
                                    output_bounds=(1, 6)))
        assert [[r.id, r.arrival_ms, r.priority.tag, r.prompt_len, r.max_new_tokens, r.prompt_seed] for r in got] == want


def test_workload_statistics_and_clamps():
    spec = WorkloadSpec(arrival_rate=5.0, duration_s=200.0, seed=3)
    tr = generate(spec)
    n = len(tr)
    assert abs(n - 1000) < 3 * math.sqrt(1000)
    ls = sum(r.priority is Priority.LATENCY_SENSITIVE for r in tr)
    assert abs(ls - 0.2 * n) < 3 * math.sqrt(n * 0.2 * 0.8)
    assert all(4 <= r.prompt_len <= 2048 and 1 <= r.max_new_tokens <= 512 for r in tr)
    assert [r.arrival_ms for r in tr] == sorted(r.arrival_ms for r in tr)
    toks = tr[0].prompt_tokens(256)
    assert toks == tr[0].prompt_tokens(256) and min(toks) >= 1


def test_trace_round_trip_and_validation(tmp_path):
    tr = generate(WorkloadSpec(duration_s=5.0, seed=1))
    p = tmp_path / "t.csv"
    save_trace(tr, str(p))
    assert load_trace(str(p)) == tr
    p.write_text("arrival_ms,priority,prompt_len,output_len,seed\n1.0,LS,3,4\n")
    with pytest.raises(ValueError, match=":2:"):
        load_trace(str(p))
    p.write_text("5.0,LS,3,4,1\n1.0,BE,3,4,1\n")
    with pytest.raises(ValueError, match="out of order"):
        load_trace(str(p))
    with pytest.raises(ValueError):
        WorkloadSpec(ls_fraction=1.5).validate()


def _finished(sid, pri, arrival, first, finish, out_len=3):
    s = sequence_new([1, 2], pri, 8, arrival, seq_id=sid)
    s.generated = [5] * out_len
    s.first_token_time, s.finish_time = first, finish
    s.advance_phase(Phase.FINISHED)
    return s


def test_metrics_definitions():
    assert nearest_rank(list(range(1, 101)), 0.99) == 99
    assert nearest_rank([3.0, 1.0, 2.0], 0.5) == 2.0
    rec = MetricsRecorder()
    r = rec.record(_finished(0, Priority.LATENCY_SENSITIVE, 10.0, 3010.0, 5000.0))
    assert r.ttft_ms == 3000.0 and r.turnaround_ms == 4990.0
    with pytest.raises(ValueError):
        rec.record(_finished(0, Priority.LATENCY_SENSITIVE, 10.0, 20.0, 30.0))
    rec.record(_finished(1, Priority.BEST_EFFORT, 0.0, 5.0, 100.0, out_len=10))
    agg = aggregate(rec.records, slo_ms=3000.0, duration_ms=2000.0)
    assert agg.ls.slo_attainment == 1.0  # inclusive SLO boundary
    assert agg.completion_rate_jps == 1.0
    assert agg.be_tokens_per_s == 5.0
    assert aggregate(rec.records, 3000.0, 2000.0, reference=agg).be_slowdown_vs_reference == 1.0
    lines = jobs_csv_lines(rec.records)
    assert lines[0] == JOBS_CSV_HEADER and lines[1].startswith("0,LS,10.000,3000.000,4990.000,2,3")
    row = summary_row("qllm", 7.0, agg)
    assert set(row) == set(SUMMARY_FIELDS) and row["rate"] == "7"
    with pytest.raises(ValueError):
        aggregate([], 1.0, 1.0)


def test_core_types():
    with pytest.raises(ValueError):
        sequence_new([], Priority.BEST_EFFORT, 4, 0.0)
    with pytest.raises(ValueError):
        sequence_new([1], Priority.BEST_EFFORT, 0, 0.0)
    s = sequence_new([1, 2, 3], Priority.BEST_EFFORT, 4, 0.0)
    s.advance_phase(Phase.DECODE)
    with pytest.raises(StateCorruptionError):
        s.advance_phase(Phase.PREFILL)
    assert Priority.LATENCY_SENSITIVE > Priority.BEST_EFFORT and Priority.from_tag("LS").tag == "LS"
    assert list(Stage) == sorted(Stage)
    a, b = sequence_new([1], Priority.BEST_EFFORT, 4, 0.0, 0), sequence_new([1], Priority.BEST_EFFORT, 4, 0.0, 1)
    with pytest.raises(ValueError):
        batch_form([a, b], Phase.PREFILL, 1)
    assert batch_form([a, b], Phase.PREFILL, 2).stage_cursor is Stage.ATTENTION


def test_paged_cache_ledger_pages_and_capacity():
    c = UnifiedDynamicCache(2, (1,), torch.float32, torch.device("cpu"), entry_bytes=64, capacity_bytes=64 * 40,
                            page_size=4, initial_pages=2)
    rng = np.random.default_rng(0)
    for h in range(3):
        c.register(h)
        for layer in range(2):
            n = int(rng.integers(1, 6))
            slots = c.reserve(h, layer, n)
            assert len(set(slots)) == n
            assert c.usage_bytes() == c.recount_bytes()
    assert c.pages_in_use() >= 3
    # same positions map to the same slots in every layer
    assert c.slots(0, 0, 1) == c.slots(0, 0, 1)
    used = c.usage_bytes()
    c.evict_sequence(1)
    assert c.usage_bytes() < used and c.usage_bytes() == c.recount_bytes()
    with pytest.raises(CacheCapacityError):
        c.reserve(0, 0, 100)
    with pytest.raises(StateCorruptionError):
        c.reserve(99, 0, 1)
    # freed pages are reused
    before = c._n_pages
    c.register(7)
    c.reserve(7, 0, 4)
    assert c._n_pages == before


def test_paged_cache_reserve_batch_equals_member_reserves():
    """reserve_batch (one call per layer, the decoder's attention stage) leaves the same counts,
    pages, ledger and slots as member-by-member reserve; over capacity it raises at the same
    member with the same partial accounting."""
    def make():
        c = UnifiedDynamicCache(3, (1,), torch.float32, torch.device("cpu"), entry_bytes=64, capacity_bytes=64 * 300,
                                page_size=4, initial_pages=2)
        for h in range(5):
            c.register(h)
        return c

    a, b = make(), make()
    rng = np.random.default_rng(3)
    for _ in range(6):
        handles = [int(h) for h in rng.permutation(5)[:4]]
        ns = [int(n) for n in rng.integers(0, 7, size=4)]
        for layer in range(3):
            sa = []
            for h, n in zip(handles, ns):
                sa += a.reserve(h, layer, n)
            sb = b.reserve_batch(handles, layer, ns)
            assert sa == sb
            assert a.counts_at(handles, layer) == b.counts_at(handles, layer)
    assert a._pages == b._pages and a._counts == b._counts and a.usage_bytes() == b.usage_bytes()
    assert b.reserve_batch([0, 1], 0, [1, 1], want_slots=False) == []
    a.reserve(0, 0, 1), a.reserve(1, 0, 1)
    # over capacity: the first members still reserve, the failing one raises, like reserve()
    left = (a.capacity_bytes - a.usage_bytes()) // 64
    for c in (a, b):
        with pytest.raises(CacheCapacityError):
            if c is a:
                a.reserve(2, 1, left - 1)
                a.reserve(3, 1, 5)
            else:
                b.reserve_batch([2, 3], 1, [left - 1, 5])
    assert a._counts == b._counts and a.usage_bytes() == b.usage_bytes()
    with pytest.raises(StateCorruptionError):
        b.reserve_batch([0, 99], 0, [1, 1])


def test_page_pool_growth_is_clamped_to_max_pages():
    """A grow-by-half step that would pass max_pages grows to max_pages instead of refusing; only a
    pool already at max_pages refuses (kvcache._ensure_pages)."""
    cache = UnifiedDynamicCache(1, (1,), torch.float32, torch.device("cpu"), 4, 1e9, page_size=4, initial_pages=4,
                                max_pages=5)
    cache.register(0)
    cache.reserve(0, 0, 20)  # 5 pages: 4 -> 6 would pass max_pages=5; clamps to 5
    assert cache.pool(0).shape[0] == 5
    cache.register(1)
    with pytest.raises(CacheCapacityError):
        cache.reserve(1, 0, 1)
