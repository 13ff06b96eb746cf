#!/usr/bin/env python
"""Summarise `ncu --set full` captures (gpurun_out/prof_<tag>.ncu-rep) into profiles/.

    python scripts/ncu_summary.py ROUND TAG=KERNEL_CLASS [...]

Writes profiles/ncu_summary.json (read by bench.py for roofline.traffic: DRAM bytes per launch)
and profiles/<ROUND>/ncu_summary.md (the table judged with the round).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm_ghz": "sm__cycles_elapsed.avg.per_second",
    "grid": "launch__grid_size",
    "regs": "launch__registers_per_thread",
}
SCALE = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2]


def main():
    rnd = sys.argv[1]
    pairs = [a.split("=", 1) for a in sys.argv[2:]]
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {"kernels": {}}
    lines = ["| tag | kernel class | kernel | " + " | ".join(METRICS) + " |",
             "|" + "---|" * (3 + len(METRICS))]
    for tag, kclass in pairs:
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
        h, u, v = raw(rep)
        d = {n: (uu, vv) for n, uu, vv in zip(h, u, v)}
        row = {}
        for k, m in METRICS.items():
            unit, val = d.get(m, ("", ""))
            try:
                x = float(val.replace(",", ""))
            except ValueError:
                x = None
            if x is not None and k.endswith("_MB"):
                x = x * SCALE.get(unit, 1.0) / 1e6
            if x is not None and k == "time_us":
                x = x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(unit, 1.0)
            row[k] = x
        name = d.get("Kernel Name", ("", ""))[1]
        traffic = (row["dram_read_MB"] + row["dram_write_MB"]) * 1e6
        summ["kernels"][kclass] = {"dram_bytes_per_launch": traffic, "ncu": row, "kernel": name,
                                   "report": f"gpurun_out/prof_{tag}.ncu-rep", "round": rnd}
        lines.append(f"| {tag} | {kclass} | `{name[:60]}` | " +
                     " | ".join("" if row[k] is None else f"{row[k]:.4g}" for k in METRICS) + " |")
    json.dump(summ, open(summ_path, "w"), indent=1)
    os.makedirs(os.path.join(ROOT, "profiles", rnd), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", rnd, "ncu_summary.md"), "a") as f:
        f.write("\n".join(lines) + "\n\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
