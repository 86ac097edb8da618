"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel."""
import collections
import csv
import sys

UNITS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:70]
        t = float(d["Metric Value"].replace(",", "")) * UNITS[d["Metric Unit"]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    return agg


if __name__ == "__main__":
    agg = summarise(sys.argv[1])
    tot = sum(a[1] for a in agg.values())
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.3f} ms {c:5d}x {100 * t / tot:6.2f}%  {k}")
    print(f"{tot:10.3f} ms total")
