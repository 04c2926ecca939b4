"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for d in data:
    k = d["Kernel Name"].split("(")[0].replace("sfg::<unnamed>::", "")[:48]
    v = float(d["Metric Value"].replace(",", ""))
    m = d["Metric Name"]
    if m == "gpu__time_duration.sum":
        agg[k][0] += 1
        agg[k][1] += v
    elif m == "dram__bytes_read.sum":
        agg[k][2] += v
    elif m == "dram__bytes_write.sum":
        agg[k][3] += v
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':48s} {'n':>4s} {'us/launch':>10s} {'share':>6s} {'rd MB/l':>9s} {'wr MB/l':>9s} {'GB/s':>7s}")
for k, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
    us = t / n / 1e3
    print(f"{k:48s} {n:4d} {us:10.1f} {t / tot:6.1%} {rd / n / 1e6:9.1f} {wr / n / 1e6:9.1f} {(rd + wr) / t:7.0f}")
