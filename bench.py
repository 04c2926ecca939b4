#!/usr/bin/env python3
"""Benchmark of the B200 sparse hot path (BASELINE.json north star).

A step = one pass of the hot path over one synthetic matrix resident in HBM:
canonical (row-sorted) COO -> format conversion -> SpMV, i.e. the reference's
convert_structure + materialize + run_kernel (planner.hpp:261, storage.hpp:97,
kernel.hpp:236). Default workload: BASELINE config 2 (hybrid ELL+COO
conversion + SpMV on R-MAT scale 22, edge factor 16, threshold T=8).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1|2|3]
                  [--impl ours|reference]

Prints ONE JSON line (rank 0). value = nnz converted+multiplied per second
over all ranks (Mnnz/s). `e2e` runs the same step through the C-ABI with
host buffers (from_coo from pinned host arrays, SpMV with host x / host y).
`roofline` = dominant kernel's algorithmic bytes / CUDA-event time vs the
measured HBM copy peak. `cpu_baseline` = the unmodified reference (oracle/_ref)
on a bounded row-block sample, on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV/SpMM GFLOP/s + achieved HBM GB/s; format conversion Mnnz/s"
UNIT = "Mnnz/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops", 1654.1)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ----------------------------------------------------------------- workloads
class Workload:
    """Defines setup (device-resident canonical COO + dense operand), the
    step, and the algorithmic bytes of each kernel family in the step."""

    name = ""
    fmt = ""

    def __init__(self, args, rank, world):
        self.args, self.rank, self.world = args, rank, world

    # algorithmic bytes: each array read once, written once
    def convert_bytes(self):
        raise NotImplementedError

    def spmv_bytes(self):
        raise NotImplementedError


class Cfg1(Workload):
    """COO->CSR conversion + CSR SpMV fp32, uniform 2^20 x 2^20, 16/row."""
    fmt = "CSR"

    def setup(self, ctx):
        self.scale = 20
        m = n = 1 << self.scale
        glob = ctx.gen_uniform(1, m * self.world, n, 16) if self.world > 1 else ctx.gen_uniform(1, m, n, 16)
        return glob

    def convert_bytes(self, nnz, m, n, info):
        return 20 * nnz + 4 * (m + 1)  # read row,col,val; write idx,val,ptr

    def spmv_bytes(self, nnz, m, n, info):
        return 8 * nnz + 4 * (m + 1) + 4 * n + 4 * m


class Cfg2(Workload):
    """Hybrid ELL+COO conversion (decompose T=8) + SpMV, R-MAT s22 ef16."""
    fmt = "HYB(8)"

    def setup(self, ctx):
        self.scale = 22 + (self.world.bit_length() - 1 if self.world > 1 else 0)
        return ctx.gen_rmat(7, self.scale, 16 << self.scale)

    def convert_bytes(self, nnz, m, n, info):
        # decompose: count pass (row + val) 8*nnz + 4M; split: read 12*nnz,
        # write COO 12*nnz_sel; ELL: write 8*K*M (+ read 8*nnz_rem for the
        # remainder entries, counted in the 12*nnz read)
        return 8 * nnz + 4 * m + 12 * nnz + 12 * info["nnz_coo"] + 8 * info["ell_cells"]

    def spmv_bytes(self, nnz, m, n, info):
        return 8 * info["ell_cells"] + 12 * info["nnz_coo"] + 4 * n + 4 * m


class Cfg3(Workload):
    """DCSR conversion + SpMV on hypersparse 4M x 4M, 2/row (SpMM later)."""
    fmt = "DCSR"

    def setup(self, ctx):
        m = 1 << 22
        return ctx.gen_hypersparse(5, m, m, 2 * m)

    def convert_bytes(self, nnz, m, n, info):
        return 20 * nnz + 8 * info.get("nnr", 0) + 4

    def spmv_bytes(self, nnz, m, n, info):
        return 8 * nnz + 8 * info.get("nnr", 0) + 4 * n + 4 * m


WORKLOADS = {1: Cfg1, 2: Cfg2, 3: Cfg3}


# ------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"sfg_clocks_{os.getpid()}.csv")

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 6:
                    try:
                        rows.append((float(parts[0]), float(parts[1]), parts[2:]))
                    except ValueError:
                        pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, rs in rows for i, r in enumerate(rs) if r.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2403_05802_b200 as sfg

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    ctx = sfg.Context(local, stream.cuda_stream)
    wl = WORKLOADS[args.config](args, rank, world)

    # ---- setup: canonical COO resident in HBM, this rank's row block
    glob = wl.setup(ctx)
    if world > 1:
        bounds = ctx.row_partition(glob, world)
        coo = ctx.slice_rows(glob, bounds[rank], bounds[rank + 1])
        row0 = bounds[rank]
        del glob
    else:
        coo, bounds, row0 = glob, [0, glob.shape[0]], 0
    m, n = coo.shape
    nnz = int(coo.view().nvals)
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    ctx.gen_dense(3, n, x.data_ptr())
    if world > 1:
        # equal padded chunks for the all-gather
        t = torch.tensor([m], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        chunk = int(t.item())
    else:
        chunk = m
    y = torch.zeros(max(chunk, 1), dtype=torch.float32, device="cuda")
    y_full = torch.empty(max(chunk, 1) * world, dtype=torch.float32, device="cuda") if world > 1 else y
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    # info for the algorithmic byte counts
    a = ctx.convert(coo, wl.fmt)
    info = {}
    if wl.fmt.startswith("HYB"):
        ell, cpart = a.parts()
        ev, cv = ell.view(), cpart.view()
        info = {"ell_cells": int(ev.nvals), "ell_k": int(ev.level[0].node_count),
                "nnz_coo": int(cv.nvals), "nnz_ell": nnz - int(cv.nvals)}
    elif wl.fmt == "DCSR":
        info = {"nnr": int(a.view().level[0].node_count)}
    del a

    def gather_y():
        if world > 1:
            # reassemble y over NVLink: rank r's rows land at y_full[r*chunk:]
            dist.all_gather_into_tensor(y_full, y)

    def step():
        a = ctx.convert(coo, wl.fmt)
        ctx.spmv_device(a, x.data_ptr(), y.data_ptr())
        del a
        gather_y()

    def timed(fn, k, flush_between=True):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        for i in range(k):
            if flush_between:
                flush.zero_()
            ev[i][0].record(stream)
            fn()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        return [s.elapsed_time(e) for s, e in ev]

    # ---- warmup
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, barrier + sync on both sides
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        # keep the GPU under this load long enough for nvidia-smi to sample
        # the clocks; the timed steps follow inside the same sampling window
        t_end = time.time() + (0 if args.profile else 1.5)
        while time.time() < t_end:
            step()
            torch.cuda.synchronize()
        l0 = sfg.launch_count()
        step_ms = timed(step, args.steps)
    launches = (sfg.launch_count() - l0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        tn = torch.tensor([nnz], device="cuda", dtype=torch.float64)
        dist.all_reduce(tn)
        total_nnz = float(tn.item())
    else:
        total_nnz = float(nnz)
    ms_per_step = total_ms / args.steps
    value = total_nnz / (ms_per_step * 1e-3) / 1e6

    # ---- kernel-level roofline: convert alone, spmv alone (CUDA events)
    hbm, _, peak_src = load_peaks()
    conv_ms = statistics.mean(timed(lambda: ctx.convert(coo, wl.fmt), args.steps))
    a = ctx.convert(coo, wl.fmt)
    spmv_ms = statistics.mean(timed(lambda: ctx.spmv_device(a, x.data_ptr(), y.data_ptr()),
                                    args.steps))
    cb = wl.convert_bytes(nnz, m, n, info)
    sb = wl.spmv_bytes(nnz, m, n, info)
    kernels = {
        "convert": {"ms": conv_ms, "alg_bytes": cb, "GB/s": cb / conv_ms / 1e6,
                    "Mnnz/s": nnz / conv_ms / 1e3},
        "spmv": {"ms": spmv_ms, "alg_bytes": sb, "GB/s": sb / spmv_ms / 1e6,
                 "GFLOP/s": 2 * nnz / spmv_ms / 1e6},
    }
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    ach = kernels[dom]["GB/s"]
    roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(ach / hbm, 4), "traffic": None, "kernel": dom,
            "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs"}

    # ---- e2e through the C-ABI with host buffers (pinned)
    r_h, c_h, v_h = coo.coo_arrays()
    pin = lambda arr: torch.from_numpy(arr).pin_memory()
    r_p, c_p, v_p = pin(r_h), pin(c_h), pin(v_h)
    x_p = pin(x.cpu().numpy())
    y_p = torch.empty(m, dtype=torch.float32).pin_memory()
    import ctypes as C
    lib = sfg.load()

    def e2e_step():
        h = C.c_void_p()
        sfg._check(lib.sfg_from_coo(ctx.h, m, n, nnz, C.c_void_p(r_p.data_ptr()), C.c_void_p(c_p.data_ptr()),
                                    C.c_void_p(v_p.data_ptr()), sfg.FLAG_HOST | sfg.FLAG_SORTED, C.byref(h)))
        t = sfg.Tensor(ctx, h)
        a2 = ctx.convert(t, wl.fmt)
        sfg._check(lib.sfg_spmv(ctx.h, a2.h, C.c_void_p(x_p.data_ptr()), C.c_void_p(y_p.data_ptr()),
                                sfg.COMPUTE_HOST))

    if args.profile:
        print(json.dumps({"profile_run": True, "value": round(value, 2), "kernels": kernels}))
        return
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = statistics.mean(timed(e2e_step, max(3, min(args.steps, 10)), flush_between=False))
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": round(total_nnz / (e2e_ms * 1e-3) / 1e6, 2), "unit": UNIT,
           "h2d_bytes_per_step": int(12 * nnz + 4 * n), "d2h_bytes_per_step": int(4 * m),
           "ms_per_step": round(e2e_ms, 4)}

    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generators, csrc/synth.h)",
            "config": {"workload": f"config {args.config}: {wl.__doc__.strip()}",
                       "format": wl.fmt, "rows": int(bounds[-1]) if world > 1 else m, "cols": n,
                       "nnz_per_rank": nnz, "nnz_total": int(total_nnz), "scale": getattr(wl, "scale", None),
                       "step": f"canonical COO -> {wl.fmt} conversion -> SpMV" +
                               (" -> NCCL all-gather of y" if world > 1 else ""),
                       "l2": "flushed (256 MB write) before every timed step",
                       "parallelism": f"row-partitioned x{world}" if world > 1 else "single GPU",
                       **{k: v for k, v in info.items()}},
            "roofline": roof,
            "kernels": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in d.items()}
                        for k, d in kernels.items()},
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
    if world > 1:
        dist.barrier()
    if rank == 0 and args.config in (1, 2) and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args.config, steps=1)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------- reference (CPU) arm
def reference_sample(config):
    """Bounded row-block sample of the workload, from the oracle's
    generator (identical matrix to the GPU arm's)."""
    import oracle
    port = oracle.Port()
    if config == 1:
        full = port.gen_uniform(1, 1 << 20, 1 << 20, 16)
        rows = (0, 1 << 16)  # 1/16 of the rows: 1,048,576 nnz
    else:
        full = port.gen_rmat(7, 22, 16 << 22)
        rows = (1 << 20, (1 << 20) + (1 << 17))  # a mid-graph row block
    r, c, v = full.arrays()
    sel = (r >= rows[0]) & (r < rows[1])
    r, c, v = r[sel] - rows[0], c[sel], v[sel]
    m, n = rows[1] - rows[0], full.shape[1]
    x = port.gen_dense(3, n)
    desc = f"rows [{rows[0]}, {rows[1]}) of the config-{config} matrix: {m} x {n}, {len(v)} nnz"
    return m, n, r, c, v, x, desc


def cpu_baseline(config, steps=1, kind="reference"):
    import oracle
    lib = oracle.Ref() if (kind == "reference" and oracle.ref_available()) else oracle.Port()
    kind = "reference" if isinstance(lib, oracle.Ref) else "port"
    m, n, r, c, v, x, desc = reference_sample(config)
    threads = os.cpu_count() or 1
    coo = lib.from_coo(m, n, r, c, v)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        if config == 1:
            a = lib.convert(coo, "CSR")
            lib.spmv(a, x, threads=threads)
        else:
            sel, rem, _ = lib.decompose_rows(coo, 8)
            e, co = lib.convert(rem, "ELL"), lib.convert(sel, "COO")
            lib.spmv(e, x, threads=threads) + lib.spmv(co, x, threads=threads)
        times.append(time.perf_counter() - t0)
    sec = statistics.mean(times)
    return {"value": round(len(v) / sec / 1e6, 4), "unit": UNIT, "cores": threads, "kind": kind,
            "sample": desc + f"; convert single-threaded (reference), run_kernel threads={threads}",
            "sec_per_step": round(sec, 3)}


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    if args.config not in (1, 2):
        print(json.dumps({"impl": "reference", "unavailable": f"config {args.config} has no CPU sample"}))
        return
    for _ in range(args.warmup):
        pass  # the reference has no warm-up effects worth timing twice
    cb = cpu_baseline(args.config, steps=args.steps)
    wl = WORKLOADS[args.config]
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["sec_per_step"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, csrc/synth.h)",
        "config": {"workload": f"config {args.config}: {wl.__doc__.strip()}", "format": wl.fmt},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no clock soak, no e2e, no CPU baseline")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
