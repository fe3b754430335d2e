"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel launches and total us."""
import collections
import csv
import sys


def summarise(path, skip=("fill_uniform", "axpy_kernel", "ttm_tile_kernel<float>", "fill_lowrank")):
    agg = collections.OrderedDict()
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    return agg


if __name__ == "__main__":
    agg = summarise(sys.argv[1])
    tot = sum(t for _, t in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:10.1f} us {n:4d}  {100 * t / tot:5.1f}%  {k[:70]}")
    print(f"{tot:10.1f} us total")
