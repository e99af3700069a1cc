"""Wire formats: this repo's jobs.csv / summary.csv / trace files are
byte-identical to the reference's for the same runs, reference-written files load here, and the
reference's own `moesim compare` prints this repo's summary exactly as it prints its own.

Goldens: tests/golden/wire/, written by the unmodified reference (tests/golden/gen_wire.py) for
trace A under the FCFS baseline and QLLM.  The runs here go through this repo's
engine + scheduler + driver on the CPU (routing-replay double, tests/replay.py), whose decision
logs and job records equal the reference's (test_decision_log.py)."""

import contextlib
import io
import sys
from dataclasses import replace
from pathlib import Path

import pytest

from conftest import GOLDEN
from replay import ReplayModel, load_log, policy_for, trace_of
from paper_2503_09304_b200.metrics import aggregate, summary_row, write_jobs_csv, write_summary_csv
from paper_2503_09304_b200.sim import Simulation
from paper_2503_09304_b200.workload import WorkloadSpec, load_trace, save_trace, trace_for_rate

WIRE = GOLDEN / "wire"
SLO_MS = 3000.0  # the reference runner's default (cli.py:58)


def _run(name):
    rec = load_log(name)
    sim = Simulation(trace_of(rec), model=ReplayModel(rec), scheduler=rec["scheduler"],
                     max_batch_size=rec["max_batch_size"], policy=policy_for(rec))
    return sim.run()


def _write_trace_a(tmp: Path) -> Path:
    """What the reference runner writes for trace A: baseline first (the BE slowdown reference),
    then qllm (cli.py:269-305)."""
    rows, base = [], None
    for s in ("baseline", "qllm"):
        res = _run(f"traceA_{s}")
        rep = aggregate(res.records, SLO_MS, res.makespan_ms, base)
        base = base or rep
        write_jobs_csv(res.records, str(tmp / f"traceA_{s}_jobs.csv"))
        rows.append(summary_row(s, 16.0, rep))
    write_summary_csv(rows, str(tmp / "traceA_summary.csv"))
    return tmp / "traceA_summary.csv"


def test_jobs_and_summary_csv_are_byte_identical(tmp_path):
    _write_trace_a(tmp_path)
    for f in ("traceA_baseline_jobs.csv", "traceA_qllm_jobs.csv", "traceA_summary.csv"):
        assert (tmp_path / f).read_bytes() == (WIRE / f).read_bytes(), f


def test_trace_file_is_byte_identical_and_round_trips(tmp_path):
    spec = WorkloadSpec(ls_fraction=0.25, prompt_mean=32, prompt_sigma=0.8, prompt_bounds=(4, 128), output_mean=16,
                        output_sigma=0.9, output_bounds=(1, 48), duration_s=20.0)
    recs = trace_for_rate(spec, 7.0, seed=2, jobs_per_run=16)
    save_trace(recs, str(tmp_path / "t.csv"))
    assert (tmp_path / "t.csv").read_bytes() == (WIRE / "paper_rate7_trace.csv").read_bytes()
    back = load_trace(str(WIRE / "paper_rate7_trace.csv"))
    assert [(r.arrival_ms, r.priority, r.prompt_len, r.max_new_tokens, r.prompt_seed) for r in back] == \
           [(r.arrival_ms, r.priority, r.prompt_len, r.max_new_tokens, r.prompt_seed) for r in recs]


def test_reference_compare_reads_this_repos_summary(tmp_path):
    """`moesim compare` (reference cli.py:399-406) on the summary written here prints the golden
    text.  Needs the reference importable (this container); skipped elsewhere."""
    ref = Path("/root/reference/pkg/src")
    if not ref.exists():
        pytest.skip("reference not present")
    summary = _write_trace_a(tmp_path)
    sys.path.insert(0, str(ref))
    dont = sys.dont_write_bytecode
    sys.dont_write_bytecode = True  # /root/reference is read-only
    try:
        from moesim import cli
    finally:
        sys.path.remove(str(ref))
        sys.dont_write_bytecode = dont
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert cli.main(["compare", "--summary", str(summary)]) == 0
    assert buf.getvalue() == (WIRE / "traceA_compare.txt").read_text()
