"""Condense an `ncu --set full` report into a per-kernel text summary for
profiles/: duration, DRAM bytes and throughput, cache hit rates, occupancy,
issue rate and the top warp-stall reasons (PC sampling).

  python scripts/ncu_summary.py <report.ncu-rep> [kernel-regex] > profiles/<name>.txt
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}

WANT = [
    ("gpu__time_duration.sum", "duration", 1, ""),
    ("dram__bytes_read.sum", "dram read", 1, ""),
    ("dram__bytes_write.sum", "dram write", 1, ""),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput", 1, "% of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate", 1, "%"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate", 1, "%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy", 1, "%"),
    ("launch__registers_per_thread", "registers/thread", 1, ""),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy", 1, "%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput", 1, "% of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput", 1, "% of peak"),
    # tensor pipe (tcgen05 kernels): MMA cycles, the shared-memory operand
    # reads feeding it, and the tensor-memory path
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active", 1, "% of peak"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc pipe instructions", 1, "% of peak"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem reads by the MMA",
     1, "% of peak"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor memory active", 1, "% of peak"),
]


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


for r in data:
    name = r[col["Kernel Name"]].split("(")[0]
    print(f"== {name}  (grid {r[col.get('launch__grid_size', 0)]}, block {r[col.get('launch__block_size', 0)]})")
    for key, label, scale, unit in WANT:
        if key in col and num(r[col[key]]) is not None:
            v = num(r[col[key]])
            u = units[col[key]] or unit
            print(f"   {label:22s} {v:12.2f} {u}")
    stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: num(r[i]) for h, i in col.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
    stalls = {k: v for k, v in stalls.items() if v}
    tot = sum(stalls.values()) or 1
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
    print("   top stalls: " + ", ".join(f"{k} {v / tot:.0%}" for k, v in top))
