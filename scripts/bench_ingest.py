"""Unsorted-COO ingest (measured separately per §8d):
from_coo on device arrays in random order -> canonical (row, col)-sorted,
deduplicated COO (radix sort + unique), vs the unmodified reference's
from_coo (tensor.hpp:118-162) on a host sample of the same entries.

  python scripts/bench_ingest.py   # configs 1 and 2 shapes, one JSON line each
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_05802_b200 as sfg  # noqa: E402

ctx = sfg.Context(0, torch.cuda.current_stream().cuda_stream)


def dev_arrays(t):
    v = t.view()
    n = int(v.nvals)
    r = torch.empty(n, dtype=torch.int32, device="cuda")
    c = torch.empty(n, dtype=torch.int32, device="cuda")
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    for dst, src in ((r, v.level[0].idx), (c, v.level[1].idx), (x, v.values)):
        ctx.copy_device(dst.data_ptr(), src, n * 4)
    return r, c, x


def run(name, t, m, n):
    r, c, x = dev_arrays(t)
    nnz = r.numel()
    perm = torch.randperm(nnz, device="cuda")
    rs, cs, xs = r[perm].contiguous(), c[perm].contiguous(), x[perm].contiguous()
    torch.cuda.synchronize()
    for _ in range(2):
        ctx.from_coo_device(m, n, nnz, rs.data_ptr(), cs.data_ptr(), xs.data_ptr())
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 1e9
    for _ in range(5):
        ev[0].record()
        out = ctx.from_coo_device(m, n, nnz, rs.data_ptr(), cs.data_ptr(), xs.data_ptr())
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    r2, c2, x2 = dev_arrays(out)
    exact = bool(torch.equal(r2, r) and torch.equal(c2, c) and torch.equal(x2, x))
    res = {"workload": name, "nnz": nnz, "unsorted_from_coo_ms": round(best, 3),
           "device_Mnnz_per_s": round(nnz / best / 1e3, 1), "bit_exact_vs_canonical": exact,
           "bytes_moved_per_entry_note": "radix sort of (row,col) keys + value payload, then unique + emit"}
    try:
        import oracle
        if oracle.ref_available():
            ref = oracle.Ref()
            k = min(nnz, 1 << 20)
            idx = np.random.default_rng(0).choice(nnz, k, replace=False)
            hr, hc, hx = (a.cpu().numpy()[np.sort(idx)] for a in (r, c, x))
            p = np.random.default_rng(1).permutation(k)
            t0 = time.perf_counter()
            ref.from_coo(m, n, hr[p], hc[p], hx[p].astype(np.float64))
            sec = time.perf_counter() - t0
            res["reference"] = {"sample_entries": k, "seconds": round(sec, 3),
                                "Mnnz_per_s": round(k / sec / 1e6, 3), "threads": 1}
    except Exception as e:  # pragma: no cover
        res["reference_error"] = str(e)
    print(json.dumps(res), flush=True)


run("config 1 shape: uniform 2^20 x 2^20, 16/row", ctx.gen_uniform(1, 1 << 20, 1 << 20, 16), 1 << 20, 1 << 20)
run("config 2 shape: R-MAT scale 22, edge factor 16 (unique)", ctx.gen_rmat(7, 22, 16 << 22), 1 << 22, 1 << 22)
