#!/usr/bin/env python3
"""Benchmark of the B200 sparse hot path (BASELINE.json north star).

A step = one pass of the hot path over one synthetic matrix resident in HBM:
canonical (row-sorted) COO -> format conversion -> SpMV/SpMM, i.e. the
reference's convert_structure + materialize + run_kernel (planner.hpp:261,
storage.hpp:97, kernel.hpp:236). Default workload: BASELINE config 5
(COO->CSR conversion + CSR SpMM N=32 fp32 on R-MAT scale 26, edge factor 16:
the largest configuration that fits one GPU, and the one the north star
row-partitions over 1/2/4/8 GPUs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1..5]
                  [--impl ours|reference]

Prints ONE JSON line (rank 0). value = nnz converted+multiplied per second
over all ranks (Mnnz/s; config 4, which has no conversion in the step, is
reported in GFLOP/s). `e2e` runs the same step through the C-ABI with host
buffers (from_coo from pinned host arrays, SpMV with host x / host y).
`roofline` = dominant kernel family's algorithmic bytes / CUDA-event time vs
the measured HBM copy peak (and vs the nominal 8 TB/s). `cpu_baseline` /
--impl reference = the unmodified reference (oracle/_ref) on a bounded
row-strided sample (every k-th row, so rows keep the matrix's average
length), with the host's CPU model, core count and RAM.
N > 1 (torchrun): nnz-balanced row blocks, the output reassembled with an
NCCL all-gather; config 5 partitions the one scale-26 matrix (strong
scaling), configs 1 and 2 grow the matrix with N (weak scaling).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV/SpMM GFLOP/s + achieved HBM GB/s; format conversion Mnnz/s"
NOMINAL_HBM_GBS = 8000.0  # the north star's "roughly 8 TB/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("bf16_tflops", 1654.1)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ----------------------------------------------------------------- workloads
class Workload:
    """setup() builds the device-resident input; step() is one pass of the
    path; kernels() lists the kernel families timed for the roofline as
    (name, fn, algorithmic bytes, flops)."""
    unit = "Mnnz/s"
    fmt = ""
    scaling = "weak"  # per-GPU work fixed as N grows (the matrix grows with N)
    has_cpu_sample = True  # bounded reference sample (cpu_baseline)

    def __init__(self, sfg, ctx, rank, world):
        self.sfg, self.ctx, self.rank, self.world = sfg, ctx, rank, world
        self.info = {}

    def rows_block(self, glob):
        """This rank's nnz-balanced row block."""
        if self.world == 1:
            self.bounds = [0, glob.shape[0]]
            return glob
        self.bounds = self.ctx.row_partition(glob, self.world)
        return self.ctx.slice_rows(glob, self.bounds[self.rank], self.bounds[self.rank + 1])

    def work_units(self):
        return self.nnz

    def bind_output(self, t):
        """Compute into `t` (this rank's chunk of the gathered output)."""
        if hasattr(self, "c"):
            self.c = t
        self.y = t

    def describe(self):
        return self.__doc__.strip()


class SpmvWorkload(Workload):
    """conversion to self.fmt + SpMV"""

    def setup_dense(self, torch):
        m, n = self.coo.shape
        self.m, self.n = m, n
        self.nnz = int(self.coo.view().nvals)
        self.x = torch.empty(n, dtype=torch.float32, device="cuda")
        self.ctx.gen_dense(3, n, self.x.data_ptr())
        self.y = torch.zeros(max(m, 1), dtype=torch.float32, device="cuda")

    def step(self):
        a = self.ctx.convert(self.coo, self.fmt)
        self.ctx.spmv_device(a, self.x.data_ptr(), self.y.data_ptr())

    def kernels(self):
        a = self.ctx.convert(self.coo, self.fmt)
        self.probe(a)
        self.kept = a
        return [("convert", lambda: self.ctx.convert(self.coo, self.fmt), self.convert_bytes(), 0),
                ("spmv", lambda: self.ctx.spmv_device(a, self.x.data_ptr(), self.y.data_ptr()),
                 self.spmv_bytes(), 2 * self.nnz)]

    def probe(self, a):
        pass

    def out_rows(self):
        return self.y


class Cfg1(SpmvWorkload):
    """COO->CSR conversion + CSR SpMV fp32, uniform 2^20 x 2^20, 16/row"""
    fmt = "CSR"
    has_cpu_sample = True

    def setup(self, torch):
        self.coo = self.rows_block(self.ctx.gen_uniform(1, (1 << 20) * self.world, 1 << 20, 16))
        self.setup_dense(torch)

    def convert_bytes(self):
        return 20 * self.nnz + 4 * (self.m + 1)

    def spmv_bytes(self):
        return 8 * self.nnz + 4 * (self.m + 1) + 4 * self.n + 4 * self.m


class Cfg2(SpmvWorkload):
    """hybrid ELL+COO conversion (decompose, T=8) + SpMV, R-MAT scale 22 (+log2 N), edge factor 16"""
    fmt = "HYB(8)"
    threshold = 8  # --threshold: SURVEY.md §8d sweeps T in {4, 8, 16, 32}; 8 is the default line
    has_cpu_sample = True

    def describe(self):
        return self.__doc__.strip().replace("T=8", f"T={self.threshold}")

    def setup(self, torch):
        self.fmt = f"HYB({self.threshold})"
        self.scale = 22 + (self.world.bit_length() - 1 if self.world > 1 else 0)
        self.coo = self.rows_block(self.ctx.gen_rmat(7, self.scale, 16 << self.scale))
        self.setup_dense(torch)

    def probe(self, a):
        ell, cpart = a.parts()
        ev, cv = ell.view(), cpart.view()
        self.info = {"ell_cells": int(ev.nvals), "ell_k": int(ev.level[0].node_count),
                     "nnz_coo": int(cv.nvals), "nnz_ell": self.nnz - int(cv.nvals), "threshold": self.threshold}

    def convert_bytes(self):
        i = self.info
        # count pass over the rows (4 nnz; the source is known
        # zero-free, so values are not read) + row pointers, split (row, col,
        # val read once), COO part written, ELL cells written
        return 4 * self.nnz + 4 * self.m + 12 * self.nnz + 12 * i["nnz_coo"] + 8 * i["ell_cells"]

    def spmv_bytes(self):
        i = self.info
        return 8 * i["ell_cells"] + 12 * i["nnz_coo"] + 4 * self.n + 4 * self.m


class Cfg3(Workload):
    """DCSR and CSC conversion + DCSR SpMM N=64 fp32, hypersparse 4M x 4M, 2/row (i.i.d., dedup)"""
    nd = 64

    def setup(self, torch):
        m = 1 << 22
        self.coo = self.rows_block(self.ctx.gen_hypersparse(5, m * self.world, m, 2 * m * self.world))
        self.m, self.n = self.coo.shape
        self.nnz = int(self.coo.view().nvals)
        self.b = torch.empty(self.n * self.nd, dtype=torch.float32, device="cuda")
        self.ctx.gen_dense(3, self.n * self.nd, self.b.data_ptr())
        self.c = torch.zeros(max(self.m, 1) * self.nd, dtype=torch.float32, device="cuda")
        self.y = self.c
        self.fmt = "DCSR"

    def step(self):
        a = self.ctx.convert(self.coo, "DCSR")
        self.ctx.convert(self.coo, "CSC")
        self.ctx.spmm_device(a, self.b.data_ptr(), self.sfg.F32, self.nd, self.c.data_ptr())

    def kernels(self):
        a = self.ctx.convert(self.coo, "DCSR")
        nnr = int(a.view().level[0].node_count)
        self.info = {"nnr": nnr, "nd": self.nd}
        self.kept = a
        nz, m, n, nd = self.nnz, self.m, self.n, self.nd
        return [("convert_dcsr", lambda: self.ctx.convert(self.coo, "DCSR"), 20 * nz + 8 * nnr + 4, 0),
                ("convert_csc", lambda: self.ctx.convert(self.coo, "CSC"), 20 * nz + 4 * (n + 1), 0),
                ("spmm", lambda: self.ctx.spmm_device(a, self.b.data_ptr(), self.sfg.F32, nd, self.c.data_ptr()),
                 8 * nz + 8 * nnr + 4 * n * nd + 4 * m * nd, 2 * nz * nd)]

    def out_rows(self):
        return self.c


class Cfg4(Workload):
    """BCSR(r,r) SpMM N=128 (16x16: tcgen05, bf16 one MMA per block, f32 3xTF32), block-sparse 512K x 512K,
    10% block density, generated as BCSR"""
    unit = "GFLOP/s"
    nd = 128
    block = 16       # --block: 16 or 4
    vdtype = "bf16"  # --bcsr-dtype: bf16 (values and B) or f32

    def describe(self):
        return (f"BCSR({self.block},{self.block}) {self.vdtype} SpMM N=128"
                f"{' (tcgen05)' if self.vdtype == 'bf16' else (' (tcgen05 3xTF32)' if self.block == 16 else ' (CUDA cores)')}, "
                "block-sparse 512K x 512K, 10% block density, generated as BCSR")

    def setup(self, torch):
        m = 1 << 19
        r = self.block
        bf = self.vdtype == "bf16"
        self.m = self.n = m
        self.a = self.ctx.gen_block_sparse(11, m, m, r, r, 0.1, value_dtype=self.sfg.BF16 if bf else self.sfg.F32)
        v = self.a.view()
        self.nblocks = int(v.level[1].node_count)
        self.nnz = self.nblocks * r * r
        self.b = torch.empty(m * self.nd, dtype=torch.bfloat16 if bf else torch.float32, device="cuda")
        self.b.uniform_(-1, 1)
        self.c = torch.zeros(m * self.nd, dtype=torch.float32, device="cuda")
        self.y = self.c
        self.fmt = f"BCSR({r},{r}) {self.vdtype}"
        self.bounds = [0, m]
        self.info = {"nblocks": self.nblocks, "nd": self.nd, "value_dtype": self.vdtype, "b_dtype": self.vdtype}
        if r == 16 or bf:
            # the tensor-core path builds its per-matrix block schedule on the
            # first product and caches it on the tensor: timed here once
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record()
            self.step()
            ev[1].record()
            torch.cuda.synchronize()
            self.info["first_call_ms_with_schedule_build"] = round(ev[0].elapsed_time(ev[1]), 3)

    def step(self):
        bdt = self.sfg.BF16 if self.vdtype == "bf16" else self.sfg.F32
        self.ctx.spmm_device(self.a, self.b.data_ptr(), bdt, self.nd, self.c.data_ptr())

    def work_units(self):
        return 2 * self.nnz * self.nd / 1e3  # unit conversion below: (MFLOP) -> GFLOP/s

    def operand_roofline(self, ms):
        """The tcgen05 kernels are bound by the MMAs' shared-memory operand
        reads (ncu 'smem reads by the MMA'): bytes the MMAs read
        per product against 148 SMs x 128 B/cycle at the maximum SM clock."""
        if self.block == 16:
            per_mma = 128 * 16 * 2 + 16 * 16 * 2 if self.vdtype == "bf16" else 128 * 8 * 4 + 16 * 8 * 4
            mmas = self.nblocks * (1 if self.vdtype == "bf16" else 6)
        elif self.vdtype == "bf16":
            per_mma = 128 * 16 * 2 + 128 * 16 * 2  # a 16-row B tile and a 128-row x 16-column window
            mmas = self.info.get("windows")
            if not mmas:
                return None
        else:
            return None
        peak = 148 * 128 * 1.965e9 / 1e9  # GB/s
        ach = per_mma * mmas / ms / 1e6
        return {"achieved": round(ach, 1), "peak": round(peak, 1), "unit": "GB/s", "frac": round(ach / peak, 4),
                "bytes_per_mma": per_mma, "mmas": int(mmas)}

    def kernels(self):
        nb, m, n, nd, r = self.nblocks, self.m, self.n, self.nd, self.block
        s = 2 if self.vdtype == "bf16" else 4
        byts = nb * r * r * s + 4 * nb + 4 * (m // r + 1) + s * n * nd + 4 * m * nd
        tc = r == 16 or self.vdtype == "bf16"
        return [("spmm_bcsr_tc" if tc else "spmm_bcsr", self.step, byts, 2 * self.nnz * nd)]


class Cfg5(SpmvWorkload):
    """CSR conversion + CSR SpMM N=32 fp32, R-MAT scale 26 (row-partitioned over N GPUs)"""
    fmt = "CSR"
    nd = 32
    scaling = "strong"  # one scale-26 matrix split over the N GPUs

    def setup(self, torch):
        self.scale = 26
        self.coo = self.rows_block(self.ctx.gen_rmat(7, self.scale, 16 << self.scale))
        m, n = self.coo.shape
        self.m, self.n = m, n
        self.nnz = int(self.coo.view().nvals)
        self.b = torch.empty(n * self.nd, dtype=torch.float32, device="cuda")
        self.ctx.gen_dense(3, n * self.nd, self.b.data_ptr())
        self.c = torch.zeros(max(m, 1) * self.nd, dtype=torch.float32, device="cuda")
        self.y = self.c

    def step(self):
        a = self.ctx.convert(self.coo, "CSR")
        self.ctx.spmm_device(a, self.b.data_ptr(), self.sfg.F32, self.nd, self.c.data_ptr())

    def kernels(self):
        a = self.ctx.convert(self.coo, "CSR")
        self.kept = a
        nz, m, n, nd = self.nnz, self.m, self.n, self.nd
        return [("convert", lambda: self.ctx.convert(self.coo, "CSR"), 20 * nz + 4 * (m + 1), 0),
                ("spmm", lambda: self.ctx.spmm_device(a, self.b.data_ptr(), self.sfg.F32, nd, self.c.data_ptr()),
                 8 * nz + 4 * (m + 1) + 4 * n * nd + 4 * m * nd, 2 * nz * nd)]

    def out_rows(self):
        return self.c

    def gather_roofline(self, ms):
        """The SpMM is bound by its random 128-byte B-row gathers (DESIGN
        §4): one per entry; measured on this part (scripts/row_gather_bench.cu,
        profiles/r02_row_gather_bench.log) 35.7 G rows/s when every gather
        misses L2 and 154 G rows/s from L2, and ncu puts this SpMM's L2 hit
        rate at ~36 % — the floor of the gathers alone is their time at those
        rates."""
        rows, hit, hbm_rate, l2_rate = self.nnz, 0.36, 35.7e9, 154e9
        floor = ((1 - hit) * rows / hbm_rate + hit * rows / l2_rate) * 1e3
        return {"gathers": int(rows), "achieved_G_rows_per_s": round(rows / ms / 1e6, 2),
                "floor_ms": round(floor, 3), "frac": round(floor / ms, 4), "l2_hit_rate_ncu": hit,
                "rates_G_rows_per_s": {"hbm": 35.7, "l2": 154.0}}


WORKLOADS = {1: Cfg1, 2: Cfg2, 3: Cfg3, 4: Cfg4, 5: Cfg5}


# ------------------------------------------------------------------- clocks
_SAMPLER = r"""
import json, sys, time
import pynvml as N
dev, period = int(sys.argv[1]), float(sys.argv[2])
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(dev)
out = {"max": N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM), "s": [], "call_ms": 0.0}
print("ready", flush=True)
import select
while True:
    t0 = time.perf_counter()
    out["s"].append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), N.nvmlDeviceGetCurrentClocksEventReasons(h)))
    out["call_ms"] = max(out["call_ms"], (time.perf_counter() - t0) * 1e3)
    r, _, _ = select.select([sys.stdin], [], [], period)
    if r:
        break
print(json.dumps(out), flush=True)
"""


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons in a separate
    process: NVML calls can take milliseconds inside the driver, and made
    in this process they could delay this process's kernel launches."""

    def __init__(self, device, period=0.05):
        self.device, self.period = device, period
        self.samples, self.ok, self.err = [], False, ""

    def __enter__(self):
        import subprocess
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.device), str(self.period)],
                                         stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                         text=True)
            line = self.proc.stdout.readline().strip()
            if line != "ready":
                raise RuntimeError(line or self.proc.stderr.read()[-300:])
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = str(e)
        return self

    def __exit__(self, *exc):
        if not self.ok:
            return
        try:
            out, err = self.proc.communicate(input="stop\n", timeout=30)
            d = json.loads(out.strip().splitlines()[-1])
            self.max_mhz, self.samples, self.call_ms = d["max"], [tuple(x) for x in d["s"]], d["call_ms"]
        except Exception as e:  # noqa: BLE001
            self.ok, self.err = False, str(e)

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.err}"]}
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                 0x4: "sw_power_cap"}
        reasons = sorted({n for _, r in self.samples for bit, n in names.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples),
                "source": "NVML in a sampler process, 50 ms period", "nvml_call_ms_max": round(self.call_ms, 2)}


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2403_05802_b200 as sfg
    from paper_2403_05802_b200.rowpart import padded_chunk

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    # --rowpart runs the row-partitioned path (communicator, chunked output,
    # all-gather) even at N = 1, under torchrun: a check of that code path
    rowpart = world > 1 or args.rowpart
    if rowpart:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    ctx = sfg.Context(local, stream.cuda_stream)
    wl = WORKLOADS[args.config](sfg, ctx, rank, world)
    wl.setup(torch)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    if rowpart:
        # the library's own NCCL communicator (sfg_comm_create); the id
        # travels over torch.distributed
        uid = [sfg.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ctx.comm_create(world, rank, uid[0])
        width = wl.out_rows().numel() // max(wl.m, 1)
        chunk = padded_chunk(wl.m)
        # P equal chunks; this rank's product is computed straight into
        # chunk `rank`, then one in-place all-gather completes the output
        ybuf = torch.zeros(world * chunk * width, dtype=torch.float32, device="cuda")
        wl.bind_output(ybuf[rank * chunk * width: rank * chunk * width + max(wl.m, 1) * width])

    def step():
        wl.step()
        if rowpart:
            ctx.allgather_chunks(comm, ybuf.data_ptr(), chunk * width)

    def timed(fn, k, flush_between=True):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        host_ms.clear()
        for i in range(k):
            if flush_between:
                flush.zero_()
            ev[i][0].record(stream)
            h0 = time.perf_counter()
            fn()
            host_ms.append((time.perf_counter() - h0) * 1e3)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        return [s.elapsed_time(e) for s, e in ev]

    host_ms = []

    warm = max(args.warmup, 3)
    # a full (gen-2) Python GC pass over torch's object graph can stall the
    # host for hundreds of ms in the middle of a step: collect now, then keep
    # the collector off for the measurement
    gc.collect()
    gc.disable()
    for _ in range(warm):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, barrier + sync on both sides; clocks sampled
    with ClockSampler(local) as clk:
        # keep the GPU under this load long enough for the sampler to see the
        # clocks; the timed steps follow inside the same sampling window
        t_end = time.time() + (0 if args.profile else 1.0)
        while time.time() < t_end:
            step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = sfg.launch_count()
        step_ms = timed(step, args.steps)
        step_host_ms = list(host_ms)
        launches = sfg.launch_count() - l0
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    total_ms = sum(step_ms)
    units = float(wl.work_units())
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        tn = torch.tensor([units], device="cuda", dtype=torch.float64)
        dist.all_reduce(tn)
        units = float(tn.item())
    ms_per_step = total_ms / args.steps
    value = units / (ms_per_step * 1e-3) / 1e6
    split = None
    if rowpart:
        # the same steps without the output all-gather
        # (compute only), max over ranks, next to the gathered step above
        dist.barrier()
        comp = sum(timed(wl.step, args.steps))
        t = torch.tensor([comp], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        comp_ms = float(t.item()) / args.steps
        split = {"compute_only_ms": round(comp_ms, 4), "with_allgather_ms": round(ms_per_step, 4),
                 "allgather_bytes_per_rank": int(4 * chunk * width * (world - 1))}

    # ---- kernel families alone (CUDA events on the launching stream)
    hbm, _, peak_src = load_peaks()
    kernels = {}
    for name, fn, byts, flops in wl.kernels():
        for _ in range(2):
            fn()
        ms = statistics.median(timed(fn, max(args.steps, 5)))
        d = {"ms": round(ms, 4), "alg_bytes": int(byts), "GB/s": round(byts / ms / 1e6, 1),
             "hbm_frac": round(byts / ms / 1e6 / hbm, 4)}
        if flops:
            d["GFLOP/s"] = round(flops / ms / 1e6, 1)
        kernels[name] = d
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    ach = kernels[dom]["GB/s"]
    roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
            "traffic": None, "kernel": dom, "peak_source": f"{peak_src} MEASURED_PEAKS.json hbm_gbs",
            "peak_nominal": NOMINAL_HBM_GBS, "frac_nominal": round(ach / NOMINAL_HBM_GBS, 4)}
    for k in kernels.values():
        k["hbm_frac_nominal"] = round(k["GB/s"] / NOMINAL_HBM_GBS, 4)
    if hasattr(wl, "operand_roofline"):  # the bound of the tensor-core kernels
        roof["operand_smem"] = wl.operand_roofline(kernels[dom]["ms"])
    if hasattr(wl, "gather_roofline") and dom == "spmm":  # the gather floor of the config-5 SpMM
        roof["gather"] = wl.gather_roofline(kernels[dom]["ms"])
    # DRAM bytes per launch of the dominant family, from the committed ncu
    # launch list of this config (profiles/traffic_config<N>.json)
    variant = "" if args.config != 4 or (args.block, args.bcsr_dtype) == (16, "bf16") else \
        f"_{args.block}x{args.block}_{args.bcsr_dtype}"  # the config-4 file is the 16x16 bf16 launch list
    tpath = os.path.join(ROOT, "profiles", f"traffic_config{args.config}{variant}.json")
    if os.path.exists(tpath):
        try:
            fam = json.load(open(tpath))["families"].get(dom)
            if fam:
                roof["traffic"] = fam["dram_bytes_per_launch"]
                roof["traffic_alg_ratio"] = round(fam["dram_bytes_per_launch"] / kernels[dom]["alg_bytes"], 3)
                roof["traffic_source"] = f"ncu dram__bytes_read+write, {os.path.relpath(tpath, ROOT)}"
        except Exception:
            pass

    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "value": round(value, 2), "kernels": kernels}))
        return

    e2e = (e2e_measure(args, sfg, ctx, wl, timed, torch, dist, world) if not args.no_e2e
           else {"value": None, "unit": wl.unit, "skipped": "--no-e2e"})

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": wl.unit, "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None,
            "dtype": Cfg4.vdtype if args.config == 4 else "f32",
            "data": "synthetic (seeded generators, csrc/synth.h)",
            "config": {"workload": f"config {args.config}: {wl.describe()}", "format": wl.fmt,
                       "rows": int(wl.bounds[-1]), "cols": int(wl.n), "nnz_per_rank": int(wl.nnz),
                       "nnz_total": int(units) if wl.unit == "Mnnz/s" else None,
                       "scale": getattr(wl, "scale", None),
                       "l2": "flushed (256 MB write) before every timed step",
                       "parallelism": f"row-partitioned x{world}, in-place NCCL all-gather of the output "
                                      "(C-ABI sfg_allgather_chunks)"
                       if rowpart else "single GPU", **wl.info},
            "step_ms": {"min": round(min(step_ms), 4), "median": round(statistics.median(step_ms), 4),
                        "max": round(max(step_ms), 4), "all": [round(t, 4) for t in step_ms],
                        "host_enqueue_ms": [round(t, 3) for t in step_host_ms]},
            "roofline": roof, "kernels": kernels, "e2e": e2e, "gpu_launches": int(launches),
            **({"rowpart": split} if split else {}),
            "clocks": clk.summary(),
        }
        if world == 1 and wl.has_cpu_sample and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(args.config, steps=1)
        print(json.dumps(out), flush=True)
    if rowpart:
        dist.barrier()
        comm.close()
        dist.destroy_process_group()


def e2e_measure(args, sfg, ctx, wl, timed, torch, dist, world):
    """Same step through the C-ABI with HOST buffers: from_coo from pinned
    row/col/val, conversion, SpMV/SpMM with host x/B in and y/C out."""
    import ctypes as C

    lib = sfg.load()
    if args.config == 4:
        # no conversion in the config-4 step: host B in, host C out
        b_p = torch.empty(wl.b.numel(), dtype=wl.b.dtype).pin_memory()
        b_p.copy_(wl.b.cpu())
        c_p = torch.empty(wl.c.numel(), dtype=torch.float32).pin_memory()
        bdt = sfg.BF16 if wl.b.dtype == torch.bfloat16 else sfg.F32

        def e2e_step():
            sfg._check(lib.sfg_spmm(ctx.h, wl.a.h, C.c_void_p(b_p.data_ptr()), bdt, wl.nd, wl.nd,
                                    C.c_void_p(c_p.data_ptr()), wl.nd, sfg.COMPUTE_HOST))
        h2d, d2h = b_p.numel() * b_p.element_size(), c_p.numel() * 4
    else:
        r_h, c_h, v_h = wl.coo.coo_arrays()
        pin = lambda arr: torch.from_numpy(arr).pin_memory()
        r_p, c_p, v_p = pin(r_h), pin(c_h), pin(v_h)
        nd = getattr(wl, "nd", 1)
        dense = wl.b if hasattr(wl, "b") else wl.x
        x_p = pin(dense.cpu().numpy())
        y_p = torch.empty(max(wl.m, 1) * nd, dtype=torch.float32).pin_memory()
        fmt = wl.fmt

        def e2e_step():
            h = C.c_void_p()
            sfg._check(lib.sfg_from_coo(ctx.h, wl.m, wl.n, wl.nnz, C.c_void_p(r_p.data_ptr()),
                                        C.c_void_p(c_p.data_ptr()), C.c_void_p(v_p.data_ptr()),
                                        sfg.FLAG_HOST | sfg.FLAG_SORTED, C.byref(h)))
            t = sfg.Tensor(ctx, h)
            a2 = ctx.convert(t, fmt)
            if args.config == 3:
                ctx.convert(t, "CSC")
            if nd == 1:
                sfg._check(lib.sfg_spmv(ctx.h, a2.h, C.c_void_p(x_p.data_ptr()), C.c_void_p(y_p.data_ptr()),
                                        sfg.COMPUTE_HOST))
            else:
                sfg._check(lib.sfg_spmm(ctx.h, a2.h, C.c_void_p(x_p.data_ptr()), sfg.F32, nd, nd,
                                        C.c_void_p(y_p.data_ptr()), nd, sfg.COMPUTE_HOST))
        h2d, d2h = 12 * wl.nnz + x_p.numel() * 4, y_p.numel() * 4
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    ms = statistics.mean(timed(e2e_step, max(3, min(args.steps, 10)), flush_between=False))
    units = float(wl.work_units())
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tn = torch.tensor([units], device="cuda", dtype=torch.float64)
        dist.all_reduce(tn)
        units = float(tn.item())
    return {"value": round(units / (ms * 1e-3) / 1e6, 2), "unit": wl.unit, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 4)}


# ------------------------------------------------------- reference (CPU) arm
def host_info():
    """CPU model, logical cores and RAM of this host (the CPU baseline's machine)."""
    model, ram = "?", None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "ram_gib": ram}


def sampled_rows(r, c, v, m, stride):
    """About one row in `stride`, picked by a hash of the row id, renumbered
    densely: the sample keeps the matrix's own row-length distribution (a
    contiguous block, or every stride-th row, of an R-MAT matrix would not:
    low row ids and ids with low zero bits are the heavy rows)."""
    keep = ((np.arange(m, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) >> np.uint64(40)) % np.uint64(stride) == 0
    newid = np.cumsum(keep) - 1
    sel = keep[r]
    return int(keep.sum()), newid[r[sel]].astype(r.dtype), c[sel], v[sel]


def reference_sample(config):
    """Bounded row-strided sample of the workload, from the oracle's
    generator (the same matrix the GPU arm uses)."""
    import oracle
    port = oracle.Port()
    if config == 1:
        full, stride = port.gen_uniform(1, 1 << 20, 1 << 20, 16), 16  # 65,536 rows, 1,048,576 nnz
    else:
        full, stride = port.gen_rmat(7, 22, 16 << 22), 32  # 131,072 rows, ~2.0 M nnz
    m, r, c, v = sampled_rows(*full.arrays(), full.shape[0], stride)
    n = full.shape[1]
    x = port.gen_dense(3, n)
    desc = (f"1/{stride} of the rows of the config-{config} matrix (hash-picked): {m} x {n}, {len(v)} nnz "
            f"({len(v) / m:.2f} per row; the full matrix: {full.nnz / full.shape[0]:.2f})")
    return m, n, r, c, v, x, desc


def cpu_baseline(config, steps=1):
    """The unmodified reference (oracle/_ref; the C port if it is absent) on
    a bounded sample of the config's workload, on this host's cores."""
    import oracle
    lib = oracle.Ref() if oracle.ref_available() else oracle.Port()
    kind = "reference" if isinstance(lib, oracle.Ref) else "port"
    port = oracle.Port()
    threads = os.cpu_count() or 1
    unit, per_step_units = "Mnnz/s", None
    if config in (1, 2):
        m, n, r, c, v, x, desc = reference_sample(config)
        coo = lib.from_coo(m, n, r, c, v)

        def step():
            if config == 1:
                a = lib.convert(coo, "CSR")
                lib.spmv(a, x, threads=threads)
            else:
                sel, rem, _ = lib.decompose_rows(coo, Cfg2.threshold)
                e, co = lib.convert(rem, "ELL"), lib.convert(sel, "COO")
                lib.spmv(e, x, threads=threads) + lib.spmv(co, x, threads=threads)
        work = len(v)
    elif config == 3:
        # the config-3 generator at 1/16 of the extent (B = n x 64 in f64
        # stays in host memory); per-entry work is the same
        m = n = 1 << 18
        r, c, v = port.gen_hypersparse(5, m, n, 2 * m).arrays()
        b = port.gen_dense(3, n * 64).reshape(n, 64)
        coo = lib.from_coo(m, n, r, c, v)
        desc = f"config-3 generator at {m} x {n}, {len(v)} nnz, Nd = 64"

        def step():
            a = lib.convert(coo, "DCSR")
            lib.convert(coo, "CSC")
            lib.spmm(a, b, threads=threads)
        work = len(v)
    elif config == 4:
        m = n = 4096  # <= 4096^2 for the CPU reference
        r, c, v = port.gen_block_sparse(11, m, n, 16, 16, 0.1).arrays()
        b = port.gen_dense(3, n * 128).reshape(n, 128)
        a = lib.convert(lib.from_coo(m, n, r, c, v), "BCSR", 16, 16)
        desc = f"config-4 generator at {m} x {n} (BCSR 16x16, {len(v)} stored values), Nd = 128, SpMM only"
        unit = "GFLOP/s"

        def step():
            lib.spmm(a, b, threads=threads)
        work = 2 * len(v) * 128 / 1e3  # MFLOP -> GFLOP/s below
    else:
        # config-5 generator at scale 22 (scale <= 22; at
        # scale 26 the reference's f64 B alone is 17 GB), 1/16 of the rows
        full = port.gen_rmat(7, 22, 16 << 22)
        stride = 16
        m, r, c, v = sampled_rows(*full.arrays(), full.shape[0], stride)
        n = full.shape[1]
        b = port.gen_dense(3, n * 32).reshape(n, 32)
        coo = lib.from_coo(m, n, r, c, v)
        desc = (f"1/{stride} of the rows of R-MAT scale 22 (config-5 generator, hash-picked): {m} x {n}, "
                f"{len(v)} nnz ({len(v) / m:.2f} per row; the full matrix: {full.nnz / full.shape[0]:.2f}), Nd = 32")

        def step():
            a = lib.convert(coo, "CSR")
            lib.spmm(a, b, threads=threads)
        work = len(v)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = statistics.mean(times)
    return {"value": round(work / sec / 1e6, 4), "unit": unit, "cores": threads, "kind": kind,
            "sample": desc + f"; conversions single-threaded (as in the reference), run_kernel threads={threads}",
            "host": host_info(), "sec_per_step": round(sec, 3)}


def run_reference(args):
    if int(os.environ.get("RANK", 0)) != 0:
        return
    cb = cpu_baseline(args.config, steps=args.steps)
    wcls = WORKLOADS[args.config]
    doc = wcls.describe(wcls)
    fmt = f"HYB({Cfg2.threshold})" if wcls is Cfg2 else wcls.fmt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": cb["unit"], "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(cb["sec_per_step"] * 1e3, 3),
        "higher_is_better": True, "scaling": wcls.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators, csrc/synth.h)",
        "config": {"workload": f"config {args.config}: {doc}", "format": fmt},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "host")},
        "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--threshold", type=int, default=8, help="config 2: hybrid split threshold T")
    ap.add_argument("--block", type=int, default=16, choices=[4, 16], help="config 4: BCSR block size")
    ap.add_argument("--bcsr-dtype", default="bf16", choices=["bf16", "f32"], help="config 4: values and B")
    ap.add_argument("--rowpart", action="store_true",
                    help="row-partitioned path at N=1 too (under torchrun; exercises the NCCL all-gather)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: no clock soak, no e2e, no CPU baseline")
    args = ap.parse_args()
    Cfg2.threshold = args.threshold
    Cfg4.block, Cfg4.vdtype = args.block, args.bcsr_dtype
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
