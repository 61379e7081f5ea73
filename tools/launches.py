"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per launch)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per, names = collections.defaultdict(dict), {}
    for r in data:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[ii])] = r[ki].split("(")[0]
    return [(names[i], per[i]) for i in sorted(per)]


if __name__ == "__main__":
    L = load(sys.argv[1])
    tail = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    for n, m in L[-tail:]:
        print(f"{n:34s} t={m.get('gpu__time_duration.sum', 0):9.0f}ns "
              f"rd={m.get('dram__bytes_read.sum', 0)/1e6:8.2f}MB wr={m.get('dram__bytes_write.sum', 0)/1e6:7.2f}MB")
