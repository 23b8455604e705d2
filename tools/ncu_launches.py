"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[hi + 1:]:
        agg.setdefault(r[ki].split("(")[0][-48:], []).append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k:48s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.1f} us  share={sum(v) / total:6.1%}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        main(p)
