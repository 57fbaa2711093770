"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import sys


def main(path, top=25):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mi = hdr.index("Metric Name")
    rows = [rows[0]] + [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
    scale = {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        agg[r[ki].split("(")[0][:100]][0] += 1
        agg[r[ki].split("(")[0][:100]][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"# {path}: {len(rows) - 1} launches, {tot / 1e6:.2f} ms total (cold-cache, serialised by ncu)")
    print(f"{'ms':>10} {'share':>6} {'n':>6} {'avg_us':>9}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t / 1e6:10.2f} {100 * t / tot:5.1f}% {n:6d} {t / n / 1e3:9.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
