"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel: python tools/launch_summary.py f.csv [steps]"""
import collections
import csv
import sys


def main(path, steps=1):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    tot = 0.0
    n = 0
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        v = float(r[vi].replace(",", ""))
        name = r[ki].split("(")[0][:70]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
        n += 1
    print(f"{n} launches, {tot / 1e6:.3f} ms total (serialised, cold-cache ncu replay)")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v / 1e6:9.3f} ms {100 * v / tot:5.1f}% {c:5d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
