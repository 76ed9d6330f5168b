"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel
count, mean and total device time, share of the total. Optional second argument: a
regex; only launches after the first match of it are counted (skips setup)."""
import csv
import re
import sys
from collections import defaultdict


def main(path, after=None):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    d = defaultdict(list)
    started = after is None
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        if not started and re.search(after, r[ki]):
            started = True
        if not started:
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] == "ns" else v * 1e3 if r[ui] == "ms" else v  # -> us
        d[r[ki]].append(v)
    tot = sum(sum(v) for v in d.values()) or 1.0
    print(f"{'launches':>8} {'mean_us':>10} {'total_us':>11} {'share':>6}  kernel")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):8d} {sum(v) / len(v):10.1f} {sum(v):11.1f} {100 * sum(v) / tot:5.1f}%  {k[:110]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
