"""Hybrid BELL/COO vs CSR SpMM on a block-structured matrix (the paper's GPU
case study, PAPER.md "Hybrid BELL/COO"): 16 x 16 blocks at 10 % block
density, 90 % filled, plus one scattered entry per row on average; nd = 128
fp32. Times the conversion from canonical COO and the SpMM (CUDA events,
L2 flushed before each launch; median of 10) and checks the two products
agree.

  python scripts/bench_hbell.py [m] > profiles/r02_bench_hbell.log
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2403_05802_b200 as sfg  # noqa: E402


def blocky(seed, m, b=16, dens_blocks=0.10, fill=0.9, per_row_scatter=1.0):
    rng = np.random.default_rng(seed)
    nb = m // b
    br, bc = np.nonzero(rng.random((nb, nb)) < dens_blocks)
    ii, jj = np.meshgrid(np.arange(b), np.arange(b), indexing="ij")
    r = (br[:, None] * b + ii.reshape(1, -1)).ravel()
    c = (bc[:, None] * b + jj.reshape(1, -1)).ravel()
    keep = rng.random(len(r)) < fill
    r, c = r[keep], c[keep]
    ns = int(per_row_scatter * m)
    r = np.concatenate([r, rng.integers(0, m, ns)])
    c = np.concatenate([c, rng.integers(0, m, ns)])
    key = np.unique(r.astype(np.int64) * m + c)
    r, c = key // m, key % m
    v = (0.5 + rng.random(len(r))) * np.where(rng.random(len(r)) < 0.5, -1, 1)
    return r.astype(np.int32), c.astype(np.int32), v.astype(np.float32)


def timed(fn, k=10):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = []
    for _ in range(k + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out[2:])


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    nd = 128
    r, c, v = blocky(1, m)
    ctx = sfg.Context(0, torch.cuda.current_stream().cuda_stream)
    coo = ctx.from_coo(m, m, r, c, v, sorted=True)
    b = torch.empty(m * nd, device="cuda").uniform_(-1, 1)
    cc = torch.empty(m * nd, device="cuda")
    res = {"matrix": f"{m} x {m}, 16x16 blocks at 10% (90% filled) + 1 scattered entry per row", "nnz": len(v),
           "nd": nd}
    outs = {}
    for fmt in ("CSR", "HBELL(16,128)"):
        conv = timed(lambda: ctx.convert(coo, fmt))
        a = ctx.convert(coo, fmt)
        spmm = timed(lambda: ctx.spmm_device(a, b.data_ptr(), sfg.F32, nd, cc.data_ptr()))
        ctx.spmm_device(a, b.data_ptr(), sfg.F32, nd, cc.data_ptr())
        torch.cuda.synchronize()
        outs[fmt] = cc.clone()
        info = {"convert_ms": round(conv, 4), "spmm_ms": round(spmm, 4),
                "spmm_GFLOP/s": round(2 * len(v) * nd / spmm / 1e6, 1)}
        if fmt.startswith("HBELL"):
            bell, rest = a.parts()
            bv = bell.view()
            info.update({"bell_slots": int(bv.level[0].idx_len), "bell_cells": int(bv.nvals),
                         "coo_entries": int(rest.view().nvals)})
        res[fmt] = info
    d = (outs["CSR"] - outs["HBELL(16,128)"]).abs().max().item()
    res["max_abs_diff"] = d
    print(json.dumps(res))


if __name__ == "__main__":
    main()
