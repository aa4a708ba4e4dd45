"""Summarise an ncu --set full report (.ncu-rep) into a per-kernel table:
duration, DRAM bytes (read+write), achieved DRAM bandwidth, occupancy,
registers, grid.  Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
           "lts__t_bytes.sum", "smsp__inst_executed.sum"]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    units = rows[1]
    idx = {n: i for i, n in enumerate(h)}
    recs = []
    for r in rows[2:]:
        rec = {"kernel": r[idx["Kernel Name"]]}
        for m in METRICS:
            if m in idx:
                rec[m] = (r[idx[m]], units[idx[m]])
        recs.append(rec)
    return recs


def num(v):
    val, unit = v
    x = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
             "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
             "second": 1, "s": 1}.get(unit, 1)
    return x * scale


def table(path):
    lines = ["| kernel | us | DRAM MB (r+w) | DRAM GB/s | DRAM % peak | warps active % | regs | grid |",
             "|---|---|---|---|---|---|---|---|"]
    for rec in load(path):
        t = num(rec["gpu__time_duration.sum"])
        by = num(rec["dram__bytes_read.sum"]) + num(rec["dram__bytes_write.sum"])
        lines.append("| {} | {:.2f} | {:.2f} | {:.0f} | {} | {} | {} | {} |".format(
            rec["kernel"][:60], t * 1e6, by / 1e6, by / t / 1e9,
            rec.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", ("?", ""))[0],
            rec.get("sm__warps_active.avg.pct_of_peak_sustained_active", ("?", ""))[0],
            rec.get("launch__registers_per_thread", ("?", ""))[0],
            rec.get("launch__grid_size", ("?", ""))[0]))
    return "\n".join(lines)


if __name__ == "__main__":
    print(table(sys.argv[1]))
