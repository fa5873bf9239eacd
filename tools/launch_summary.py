"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv
--log-file X.csv) into per-kernel launches / total time / share."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1000.0 if unit in ("nsecond", "ns") else v * 1000.0 if unit in ("msecond", "ms") else v
        tot[r[ki]] += us
        cnt[r[ki]] += 1
    s = sum(tot.values())
    print(f"{'kernel':<44} {'launches':>8} {'total us':>10} {'share':>6}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:44]:<44} {cnt[k]:>8} {v:>10.1f} {100 * v / s:>5.1f}%")
    print(f"{'TOTAL':<44} {sum(cnt.values()):>8} {s:>10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
