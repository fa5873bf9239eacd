"""Summarise ncu reports (raw page) into one line per kernel: time, DRAM
bytes, achieved DRAM BW, SM/issue utilisation, occupancy, top stall reasons."""
import csv
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "sm__inst_executed.sum.pct_of_peak_sustained_elapsed": "issue%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "launch__registers_per_thread": "regs",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma%",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu%",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu%",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "lts__t_sectors.avg.pct_of_peak_sustained_elapsed": "l2%",
}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return None
    h, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for i, n in enumerate(h):
        if n in KEYS:
            d[KEYS[n]] = (vals[i], units[i])
    stalls = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
            try:
                stalls.append((float(vals[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    tot = sum(s for s, _ in stalls) or 1
    name = vals[h.index("Kernel Name")] if "Kernel Name" in h else path
    return name, d, [(n, round(100 * s / tot)) for s, n in stalls[:4]]


if __name__ == "__main__":
    for p in sys.argv[1:]:
        r = summarise(p)
        if not r:
            print(p, "no data")
            continue
        name, d, st = r
        print(f"== {name[:60]}")
        print("   " + "  ".join(f"{k}={v[0]}{v[1] if v[1] not in ('', '%') else ''}" for k, v in d.items()))
        print("   stalls:", st)
