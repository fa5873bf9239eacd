"""Summarise ncu reports (raw page) into one line per captured kernel launch:
time, DRAM bytes, SM/issue utilisation, pipe utilisation, occupancy, top
stall reasons. Also writes the per-stage DRAM traffic JSON bench.py reads
(--traffic-json PATH)."""
import csv
import json
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
    "smsp__inst_executed.sum": "warp_inst",
}

# kernel-name prefix -> bench stage (profiles/ncu_traffic.json)
STAGE_OF = {"backward_raster": "bwd_raster", "composite": "composite", "backward_geom": "bwd_geom",
            "preprocess": "preprocess", "loss_maps": "loss", "loss_grad": "loss"}


def _bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
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
        res.append((name, d, [(n, round(100 * s / tot)) for s, n in stalls[:4]]))
    return res


if __name__ == "__main__":
    args = sys.argv[1:]
    traffic_path = None
    if "--traffic-json" in args:
        k = args.index("--traffic-json")
        traffic_path = args[k + 1]
        args = args[:k] + args[k + 2:]
    traffic = {}
    for p in args:
        for name, d, st in summarise(p):
            print(f"== {name[:70]}")
            print("   " + "  ".join(f"{k}={v[0]}{v[1] if v[1] not in ('', '%') else ''}" for k, v in d.items()))
            print("   stalls:", st)
            short = name.split("(")[0].replace("void ", "").split("<")[0]
            for pre, stage in STAGE_OF.items():
                if short.startswith(pre) and "dram_rd" in d and "dram_wr" in d:
                    b = _bytes(*d["dram_rd"]) + _bytes(*d["dram_wr"])
                    e = traffic.setdefault(stage, {"dram_bytes_per_launch": 0.0, "kernels": []})
                    if short not in e["kernels"]:
                        e["kernels"].append(short)
                        e["dram_bytes_per_launch"] += b
    if traffic_path:
        for e in traffic.values():
            e["dram_bytes_per_launch"] = int(e["dram_bytes_per_launch"])
        json.dump(traffic, open(traffic_path, "w"), indent=1)
        print("wrote", traffic_path)
