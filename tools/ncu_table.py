"""Per-kernel table from an ncu --csv multi-metric launch list: launches, total / mean duration, share of the
profiled time, DRAM bytes (read + write) per launch and achieved DRAM GB/s, and the duration-weighted means of
the percentage metrics (tensor pipe, SM throughput, warps active).  Usage: python tools/ncu_table.py LIST.csv"""
import collections
import csv
import sys

SCALE = {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "second": 1e9,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path, top=30):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, ii = hdr.index("Kernel Name"), hdr.index("ID")
    mi, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    launch = collections.defaultdict(dict)
    name = {}
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        launch[r[ii]][r[mi]] = v * SCALE.get(r[ui], 1)
        name[r[ii]] = r[ki].split("(")[0][:90]
    pct = sorted({m for L in launch.values() for m in L if m.endswith("pct_of_peak_sustained_elapsed")
                  or m.endswith("pct_of_peak_sustained_active")})
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    for i, L in launch.items():
        a = agg[name[i]]
        t = L.get("gpu__time_duration.sum", 0.0)
        a["n"] += 1
        a["t"] += t
        a["dram"] += L.get("dram__bytes_read.sum", 0.0) + L.get("dram__bytes_write.sum", 0.0)
        for m in pct:
            a[m] += t * L.get(m, 0.0)
    tot = sum(a["t"] for a in agg.values())
    short = {m: m.split("__")[1].split(".")[0][:22] for m in pct}
    print(f"# {path}: {len(launch)} launches, {tot / 1e6:.2f} ms (ncu-serialised, cold cache); pct metrics are "
          f"duration-weighted means")
    print(f"{'ms':>8} {'share':>6} {'n':>5} {'avg_us':>8} {'MB/launch':>10} {'GB/s':>7} " +
          " ".join(f"{short[m]:>22}" for m in pct) + "  kernel")
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["t"])[:top]:
        gbs = a["dram"] / a["t"] if a["t"] else 0.0
        print(f"{a['t'] / 1e6:8.2f} {100 * a['t'] / tot:5.1f}% {int(a['n']):5d} {a['t'] / a['n'] / 1e3:8.1f} "
              f"{a['dram'] / a['n'] / 1e6:10.2f} {gbs:7.0f} " +
              " ".join(f"{a[m] / a['t'] if a['t'] else 0:22.1f}" for m in pct) + f"  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
