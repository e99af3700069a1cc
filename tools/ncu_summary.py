"""Summarise `ncu --set full` reports (.ncu-rep) into the per-kernel numbers we cite in profiles/:
duration, DRAM bytes, tensor-pipe / DRAM / L2 utilisation, SM clock, registers.
Usage: ncu_summary.py out.json 'what' label=path.ncu-rep [label=path ...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "sm_clock_hz": ("sm__cycles_elapsed.avg.per_second", None),
    "registers": ("launch__registers_per_thread", None),
}
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Ghz": 1e9, "Mhz": 1e6, "us": 1e3, "ms": 1e6, "ns": 1.0,
        "msecond": 1e6, "usecond": 1e3, "nsecond": 1.0}


def summarize(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[h.index("Kernel Name")][:80]}
        for k, (m, _) in KEYS.items():
            if m not in h:
                continue
            i = h.index(m)
            v = float(r[i].replace(",", ""))
            v *= UNIT.get(units[i], 1.0)
            if k == "duration_us":
                v /= 1e3  # ns -> us
            rec[k] = v
        if "dram_read_bytes" in rec and "duration_us" in rec:
            rec["dram_gbs"] = (rec["dram_read_bytes"] + rec.get("dram_write_bytes", 0)) / rec["duration_us"] / 1e3
        out.append(rec)
    return out


if __name__ == "__main__":
    dst, what = sys.argv[1], sys.argv[2]
    res = {"what": what, "captures": {}}
    for arg in sys.argv[3:]:
        label, path = arg.split("=", 1)
        res["captures"][label] = summarize(path)
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1))
