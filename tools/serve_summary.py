"""Print the key serving numbers of tools/serve.py JSON lines (one row per rate/seed/scheduler)."""
import json
import sys

KEYS = ("ls_ttft_p50_ms", "ls_ttft_p99_ms", "ls_slo_attainment", "ls_scaled_slo_attainment", "be_tokens_per_s",
        "ls_mean_turnaround_ms", "be_mean_turnaround_ms", "decode_iter_ms_median", "preemptions")
for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith('{"rate'):
            continue
        d = json.loads(line)
        print(f"== {path} rate {d['rate']} seed {d.get('seed')} dur {d['duration_s']} jobs {d['jobs']} "
              f"clocks {d.get('clocks')}")
        for k, r in d.items():
            if isinstance(r, dict) and "scheduler" in r:
                vals = " ".join(f"{x.split('_ms')[0]}={r[x]:.4g}" if isinstance(r.get(x), float) else f"{x}={r.get(x)}"
                                for x in KEYS)
                print(f"  {k:16s} {vals}")
                if r.get("preempt_positions"):
                    print(f"  {'':16s} positions {r['preempt_positions']}")
