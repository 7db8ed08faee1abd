"""Summarise an ncu --csv launch list: time and DRAM bytes per kernel name."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, names = collections.defaultdict(dict), {}
    for r in data:
        if len(r) <= vi:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        n = names[i].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:44]
        a = agg[n]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    print(f"launches {len(per)}  total {tot / 1e3:.1f} us (ncu: serialised, cold cache)")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:46s} n={a[0]:4d} time_us={a[1] / 1e3:9.1f} share={a[1] / tot:6.1%} "
              f"avg_us={a[1] / a[0] / 1e3:7.2f} GB/s={a[2] / max(a[1], 1):8.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
