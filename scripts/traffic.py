"""Per-kernel-family DRAM traffic (read + write bytes per launch) from an ncu
launch list, for bench.py's roofline.traffic field.

  python scripts/traffic.py <launches.csv> <config> > profiles/traffic_config<N>.json
"""
import collections
import csv
import json
import sys

# kernel names as the launch list prints them, template arguments dropped
FAMILIES = {
    1: {"convert": ["k_coo_to_csr"], "spmv": ["k_spmv_csr"]},
    2: {"convert": ["k_row_ptr", "k_row_scan", "k_split", "k_iota", "k_ell_fill"],
        "spmv": ["k_spmv_ell", "k_spmv_coo", "k_carry_fix"]},
    3: {"convert_dcsr": ["k_dcsr_count", "k_dcsr_heads"],
        "convert_csc": ["k_bkt_count", "k_count_scan", "k_bkt_part", "k_bkt_sort"],
        "spmm": ["k_spmm_rows"]},
    # the per-matrix schedule (k_bcsr_plan / k_bcsr_sched) is built once and
    # cached: the step is the panel kernel alone
    4: {"spmm_bcsr_tc": ["k_bcsr_tc"]},
    5: {"convert": ["k_coo_to_csr"], "spmm": ["k_merge_cuts", "k_spmm_merge", "k_spmm_carry_fix"]},
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
    # a family entry names a kernel or a prefix of its instantiations
    # (k_spmm_rows -> k_spmm_rows_batch, ...)
    for name in cnt:
        if any(name == k or name.startswith(k + "_") for k in kernels):
            traffic += (per[name]["dram__bytes_read.sum"] + per[name]["dram__bytes_write.sum"]) / cnt[name]
            time_ns += per[name]["gpu__time_duration.sum"] / cnt[name]
    out["families"][fam] = {"dram_bytes_per_launch": int(traffic), "ncu_time_us": round(time_ns / 1e3, 1),
                            "kernels": kernels}
print(json.dumps(out, indent=1))
