"""Per-SASS-address executed warp instructions from an ncu report (--set
full, -lineinfo) of a one-kernel report, bucketed into 256-byte address
ranges: python tools/ncu_sass_hist.py report.ncu-rep — prints each range's
share of the executed instructions and its average active threads."""
import csv
import subprocess
import sys


def main(path, bucket=0x100):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = next(i for i, r in enumerate(rows) if r and "Address" in r)
    h = rows[hi]
    ia, isrc, ie, ith = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    tot = 0
    ranges = {}
    items = []
    for r in rows[hi + 1:]:
        try:
            a = int(r[ia], 16)
            n = float(r[ie] or 0)
            t = float(r[ith] or 0)
        except (ValueError, IndexError):
            continue
        tot += n
        ranges.setdefault(a // bucket, [0, 0])
        ranges[a // bucket][0] += n
        ranges[a // bucket][1] += t
        items.append((n, a, r[isrc]))
    print(f"total warp instructions {tot:.0f}")
    for k in sorted(ranges):
        n, t = ranges[k]
        if n > 0.005 * tot:
            print(f"  0x{k * bucket:05x}-0x{(k + 1) * bucket:05x}: {100 * n / tot:5.1f}%  avg threads {t / max(n, 1):5.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
