#!/usr/bin/env python3
"""Per-launch table of one PCG iteration from an ncu --csv launch list with
gpu__time_duration.sum (+ optional dram__bytes_read/write.sum): the launches after the
1st and up to the 2nd launch of the marker kernel (default k_pcg_update_sf, once per
iteration of the eager solve).

    python tools/iter_profile.py launches.csv [threshold_us] [marker]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    by = collections.OrderedDict()
    tu = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}
    bu = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for d in data:
        k = d["ID"]
        e = by.setdefault(k, {"name": d["Kernel Name"].split("(")[0].replace("void ", "").replace("mgdtn::", ""),
                              "grid": d["Grid Size"], "t": 0.0, "b": 0.0})
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Name"] == "gpu__time_duration.sum":
            e["t"] = v * tu[d["Metric Unit"]]
        else:
            e["b"] += v * bu[d["Metric Unit"]]
    return list(by.values())


def main(path, thresh=50.0, marker="k_pcg_update_sf"):
    L = load(path)
    idx = [i for i, d in enumerate(L) if marker in d["name"]]
    a, b = idx[0], idx[1]
    tot = tb = 0.0
    for d in L[a + 1:b + 1]:
        tot += d["t"]
        tb += d["b"]
        if d["t"] >= thresh:
            bw = d["b"] / d["t"] / 1e6 if d["t"] > 0 else 0
            print(f"{d['t']:9.1f} us {d['b'] / 1e9:7.3f} GB {bw:5.2f} TB/s  {d['name'][:44]:44s} {d['grid']}")
    print(f"iteration: {tot / 1e3:.3f} ms, {tb / 1e9:.2f} GB DRAM, {tb / tot / 1e6:.2f} TB/s")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 50.0,
         sys.argv[3] if len(sys.argv) > 3 else "k_pcg_update_sf")
