"""Per-CUDA-source-line warp-stall samples from an ncu report (--set full,
-lineinfo): python tools/ncu_lines.py report.ncu-rep [top]."""
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    ns = h.index("Warp Stall Sampling (All Samples)")
    lines = []
    for r in rows[hi + 1:]:
        if len(r) > ns and r[0] not in ("", "Line No"):
            try:
                lines.append((float(r[ns]), r[0], r[1]))
            except ValueError:
                pass
    tot = sum(s for s, _, _ in lines) or 1.0
    for s, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{100 * s / tot:5.1f}%  {ln:>5}  {src.strip()[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
