#!/usr/bin/env python3
"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel and grid."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    tot, cnt = collections.Counter(), collections.Counter()
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mgdtn::", "")
        key = f"{name} grid={d['Grid Size']}"
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
        tot[key] += v
        cnt[key] += 1
    T = sum(tot.values())
    print(f"{len(data)} launches, sum of device times {T/1e3:.3f} ms")
    for k, v in tot.most_common(top):
        print(f"{v/1e3:9.3f} ms {100*v/T:5.1f}% n={cnt[k]:5d} avg={v/cnt[k]:8.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
