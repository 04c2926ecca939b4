"""Per-kernel-family DRAM traffic (read + write bytes per launch) from an ncu
launch list, for bench.py's roofline.traffic field.

  python scripts/traffic.py <launches.csv> <config> > profiles/traffic_config<N>.json
"""
import collections
import csv
import json
import sys

FAMILIES = {
    1: {"convert": ["k_coo_to_csr"], "spmv": ["k_spmv_csr"]},
    2: {"convert": ["k_row_ptr", "k_row_scan", "k_split", "k_iota", "k_ell_fill"],
        "spmv": ["k_spmv_ell", "k_spmv_coo"]},
    3: {"convert_dcsr": ["k_coo_to_dcsr"], "convert_csc": ["k_col_hist", "k_count_scan", "k_csc_scatter", "k_csc_fix"],
        "spmm": ["k_spmm_rows"]},
    4: {"spmm_bcsr_tc": ["k_bcsr_tc"]},
    5: {"convert": ["k_coo_to_csr"], "spmm": ["k_spmm_rows"]},
}

path, cfg = sys.argv[1], int(sys.argv[2])
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
per = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for d in data:
    name = d["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0].replace("void ", "").strip()
    m = d["Metric Name"]
    v = float(d["Metric Value"].replace(",", ""))
    if m == "gpu__time_duration.sum":
        cnt[name] += 1
    per[name][m] += v
out = {"source": path, "config": cfg, "families": {}}
for fam, kernels in FAMILIES[cfg].items():
    traffic = 0.0
    time_ns = 0.0
    for k in kernels:
        if cnt[k]:
            traffic += (per[k]["dram__bytes_read.sum"] + per[k]["dram__bytes_write.sum"]) / cnt[k]
            time_ns += per[k]["gpu__time_duration.sum"] / cnt[k]
    out["families"][fam] = {"dram_bytes_per_launch": int(traffic), "ncu_time_us": round(time_ns / 1e3, 1),
                            "kernels": kernels}
print(json.dumps(out, indent=1))
