"""Wire-format fixtures written by the UNMODIFIED reference (moesim, imported read-only from
/root/reference): the experiment runner's jobs.csv / summary.csv (reference cli.py:269-305,
metrics.py:170-218), a trace file (workload.py:107-145) and the output of `moesim compare` on that
summary (cli.py:399-406).  tests/test_wire_formats.py checks this repo writes the same bytes for
the same runs and reads the reference's files.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_wire.py
"""

from __future__ import annotations

import contextlib
import io
import shutil
import sys
import tempfile
from dataclasses import replace
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

from moesim import cli  # noqa: E402
from moesim.model import ModelConfig  # noqa: E402
from moesim.workload import WorkloadSpec, save_trace  # noqa: E402

OUT = Path(__file__).resolve().parent / "wire"


def trace_a_config(out_dir: str) -> cli.ExperimentConfig:
    """SURVEY.md §8(d) trace A: the tiny model, 16 jobs at 16 req/s, QLLM vs the FCFS baseline."""
    return cli.ExperimentConfig(
        model=ModelConfig(2, 256, 8, 2, 256, seed=0),
        workload=WorkloadSpec(ls_fraction=0.25, prompt_mean=32, prompt_sigma=0.8, prompt_bounds=(4, 128),
                              output_mean=16, output_sigma=0.9, output_bounds=(1, 48)),
        jobs_per_run=16, seed=2, max_batch_size=8, rates=[16.0], schedulers=["baseline", "qllm"], out_dir=out_dir)


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        cfg = trace_a_config(tmp)
        with contextlib.redirect_stdout(io.StringIO()):
            cli.run_experiment(cfg, quiet=True)
        shutil.copy(Path(tmp) / "summary.csv", OUT / "traceA_summary.csv")
        for s in cfg.schedulers:
            shutil.copy(Path(tmp) / f"{s}_rate16" / "jobs.csv", OUT / f"traceA_{s}_jobs.csv")
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            cli.main(["compare", "--summary", str(OUT / "traceA_summary.csv")])
        (OUT / "traceA_compare.txt").write_text(buf.getvalue())
        save_trace(cli.trace_for_rate(replace(cfg, workload=replace(cfg.workload, duration_s=20.0)), 7.0),
                   str(OUT / "paper_rate7_trace.csv"))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
