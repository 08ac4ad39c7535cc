"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) of the last N launches.

    python scripts/launch_summary.py gpurun_out/mg_launches.csv [N]
"""
import collections
import csv
import sys


def load(path):
    hdr, per = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            per.setdefault((d["ID"], d["Kernel Name"], d.get("Grid Size", "")), {})[d["Metric Name"]] = \
                float(d["Metric Value"].replace(",", ""))
    return list(per.items())


def main():
    items = load(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else len(items)
    items = items[-n:]
    agg = collections.defaultdict(lambda: [0.0, 0, 0.0])
    tot = 0.0
    for (i, name, g), m in items:
        t = m["gpu__time_duration.sum"]
        tot += t
        short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:48]
        a = agg[short]
        a[0] += t
        a[1] += 1
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    print(f"{len(items)} launches, {tot / 1000:.1f} us")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:50s} n={v[1]:4d} {v[0] / 1000:9.1f} us {100 * v[0] / tot:5.1f}%  {v[2] / 1e9:7.3f} GB")


if __name__ == "__main__":
    main()
