"""COO -> BCSR(r, c) conversion throughput ("GPU
conversion throughput at 32768^2"; CPU-oracle parity at <= 4096^2).

Input: the config-4 generator (blocks Bernoulli(0.1), fully dense, values
never 0) at 32768 x 32768, as canonical COO (the generated BCSR converted
back). Timed: the conversion from resident COO, CUDA events, L2 flushed
before every step. Parity: the same pipeline at 4096 x 4096 against the
unmodified reference (oracle/_ref), bit-exact. One JSON line per block shape.

  python scripts/bench_bcsr_convert.py
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
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def coo_of(m, r, c):
    return ctx.convert(ctx.gen_block_sparse(11, m, m, r, c, 0.1), "COO")


for (r, c) in ((16, 16), (4, 4)):
    m = 32768
    coo = coo_of(m, r, c)
    nnz = int(coo.view().nvals)
    fmt = f"BCSR({r},{c})"
    for _ in range(3):
        ctx.convert(coo, fmt)
    torch.cuda.synchronize()
    times = []
    for _ in range(10):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = ctx.convert(coo, fmt)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    v = out.view()
    nblocks = int(v.level[1].node_count)
    ms = float(np.median(times))
    # algorithmic bytes: COO read once (12 B / entry), block values written
    # (r*c*4 B per block, zero fill included), block columns + row pointers
    alg = 12 * nnz + nblocks * r * c * 4 + 4 * nblocks + 4 * (m // r + 1)
    res = {"workload": f"COO -> {fmt}, config-4 generator at {m} x {m}, density 0.1", "nnz": nnz,
           "blocks": nblocks, "ms": round(ms, 3), "Mnnz_per_s": round(nnz / ms / 1e3, 1),
           "GB_per_s": round(alg / ms / 1e6, 1), "l2": "flushed before every step"}
    # parity + CPU reference at 4096^2
    try:
        import oracle
        if oracle.ref_available():
            ref, port = oracle.Ref(), oracle.Port()
            ms_ = 4096
            rr, cc, vv = port.gen_block_sparse(11, ms_, ms_, r, c, 0.1).arrays()
            t0 = time.perf_counter()
            rm = ref.convert(ref.from_coo(ms_, ms_, rr, cc, vv), "BCSR", r, c)
            ref_s = time.perf_counter() - t0
            d = ctx.convert(ctx.from_coo(ms_, ms_, rr, cc, vv), fmt).download()
            o = rm.download()
            exact = all(np.array_equal(a.idx, b.idx) and np.array_equal(a.ptr, b.ptr)
                        for a, b in zip(d.levels, o.levels)) and np.array_equal(d.values, o.values)
            res["reference"] = {"sample": f"{ms_} x {ms_}", "entries": len(vv), "seconds": round(ref_s, 2),
                                "Mnnz_per_s": round(len(vv) / ref_s / 1e6, 3), "threads": 1,
                                "bit_exact_vs_device": bool(exact)}
    except Exception as ex:  # noqa: BLE001
        res["reference"] = {"unavailable": str(ex)[:200]}
    print(json.dumps(res), flush=True)
