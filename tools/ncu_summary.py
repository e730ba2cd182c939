#!/usr/bin/env python
"""Summarise ncu --set full captures (.ncu-rep) of single apply passes:
duration, DRAM bytes vs the algorithmic 2 x state bytes, achieved GB/s and
fraction of MEASURED_PEAKS.json, SM clock, tensor / FMA pipe activity.  Writes
the raw CSV next to each report and prints one JSON line per report.

    python tools/ncu_summary.py gpurun_out/r02g/prof_tc6.ncu-rep ... [--state-bytes B]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "sm_ghz": "sm__cycles_elapsed.avg.per_second",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "dram_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
}
SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "Tbyte": 1e12, "Ghz": 1.0, "Mhz": 1e-3, "hz": 1e-9, "%": 1.0, "": 1.0}


def summarise(rep, state_bytes, peak):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    with open(rep.replace(".ncu-rep", "_raw.csv"), "w") as f:
        f.write(out)
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    res = {"report": os.path.relpath(rep, ROOT), "kernel": v[h.index("Kernel Name")][:120]}
    for k, name in KEYS.items():
        if name in h:
            i = h.index(name)
            try:
                res[k] = float(v[i]) * SCALE.get(u[i], 1.0)
            except ValueError:
                res[k] = None
    alg = 2 * state_bytes
    res["algorithmic_bytes"] = alg
    res["dram_bytes_ratio"] = (res["dram_read"] + res["dram_write"]) / alg
    res["achieved_gbs"] = alg / (res["duration_ms"] * 1e-3) / 1e9
    res["frac_of_peak"] = res["achieved_gbs"] / peak
    return res


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    sb = 8 * 2 ** 32
    for a in sys.argv[1:]:
        if a.startswith("--state-bytes="):
            sb = int(a.split("=", 1)[1])
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    for rep in args:
        print(json.dumps(summarise(rep, sb, peak)), flush=True)


if __name__ == "__main__":
    main()
