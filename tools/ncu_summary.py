"""Summarizes ncu --set full captures (.ncu-rep) into one markdown table.

    python tools/ncu_summary.py label=path.ncu-rep [...]

Reads the raw page via `ncu -i ... --page raw --csv` and prints, per kernel:
duration, DRAM bytes (read+write), DRAM throughput %, achieved SM clock, FMA
pipe activity, tensor pipe activity, issue activity, occupancy, registers.
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("time_us", "gpu__time_duration.sum", 1e-3),
    ("dram_MB", "dram__bytes_read.sum", None),
    ("dram_w_MB", "dram__bytes_write.sum", None),
    ("dram_%", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_GHz", "sm__cycles_elapsed.avg.per_second", None),
    ("fma_pipe_%", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("fma_inst_%", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
    ("ffma_thr_inst", "sm__sass_thread_inst_executed_op_ffma_pred_on.sum", 1),
    ("issue_%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warps_%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("tensor_%", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("l2_hit_%", "lts__t_sector_hit_rate.pct", 1),
]


def unit_scale(unit: str, value: float, key: str) -> float:
    u = unit.strip().lower()
    if key in ("dram_MB", "dram_w_MB"):
        return value * {"byte": 1e-6, "kbyte": 1e-3, "mbyte": 1, "gbyte": 1e3}.get(u, 1)
    if key == "sm_GHz":
        return value * {"hz": 1e-9, "khz": 1e-6, "mhz": 1e-3, "ghz": 1}.get(u, 1)
    if key == "time_us":
        return value * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6}.get(u, 1)
    return value


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    header, units, data = r[0], r[1], r[2:]
    for d in data:
        rec = {"kernel": d[header.index("Kernel Name")]}
        for key, metric, _ in METRICS:
            if metric in header:
                i = header.index(metric)
                try:
                    rec[key] = unit_scale(units[i], float(d[i].replace(",", "")), key)
                except ValueError:
                    rec[key] = d[i]
        yield rec


def main():
    keys = [k for k, _, _ in METRICS]
    print("| capture | kernel | " + " | ".join(keys) + " |")
    print("|" + "---|" * (len(keys) + 2))
    for arg in sys.argv[1:]:
        label, path = arg.split("=", 1)
        for rec in rows(path):
            vals = []
            for k in keys:
                v = rec.get(k)
                vals.append("" if v is None else (f"{v:.4g}" if isinstance(v, float) else str(v)))
            print(f"| {label} | {rec['kernel']} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main()
