"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                 "ms": 1.0}.get(unit, 1e-6)
        k = d["Kernel Name"].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{ms:9.3f} ms {100 * ms / tot:5.1f}%  x{n:4d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
