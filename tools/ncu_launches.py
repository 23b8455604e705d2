"""Summarise an ncu --csv launch list per kernel: gpu__time_duration.sum
(mean per launch and share of the total) plus the mean of every other
metric the list carries."""
import csv
import sys

TIME = "gpu__time_duration.sum"


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg, other = {}, {}
    for r in rows[hi + 1:]:
        k = r[ki].split("(")[0][-48:]
        m = r[mi] if mi is not None else TIME
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        if m == TIME:
            agg.setdefault(k, []).append(v)
        else:
            other.setdefault(k, {}).setdefault(m, []).append(v)
    total = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        extra = "".join(f"  {m.split('__')[1][:28]}={sum(x) / len(x):.4g}" for m, x in sorted(other.get(k, {}).items()))
        print(f"  {k:48s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.1f} us  share={sum(v) / total:6.1%}{extra}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        main(p)
