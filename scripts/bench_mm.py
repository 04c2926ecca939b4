"""Matrix Market ingest throughput: the device reader (ctx.read_matrix_market:
parse + from_coo sort) vs the unmodified reference (read_matrix_market +
from_coo through oracle/_ref), on a generated file of the config-1 shape
(uniform rows, 16 entries each; mixed number formats).

  python scripts/bench_mm.py [rows] [per_row]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
per = int(sys.argv[2]) if len(sys.argv) > 2 else 16
path = "/tmp/sfg_bench.mtx"
rng = np.random.default_rng(0)
r = np.repeat(np.arange(1, rows + 1), per)
c = np.concatenate([rng.choice(rows, per, replace=False) + 1 for _ in range(min(rows, 4096))])
c = np.resize(c, r.size)
v = rng.random(r.size) * 2 - 1
t0 = time.time()
with open(path, "w") as f:
    f.write(f"%%MatrixMarket matrix coordinate real general\n{rows} {rows} {r.size}\n")
    chunk = 1 << 20
    for s in range(0, r.size, chunk):
        e = min(r.size, s + chunk)
        f.write("".join(f"{a} {b} {x:.9g}\n" for a, b, x in zip(r[s:e].tolist(), c[s:e].tolist(), v[s:e].tolist())))
size = os.path.getsize(path)
print(f"wrote {r.size} entries, {size / 1e6:.1f} MB in {time.time() - t0:.1f} s", flush=True)

import torch  # noqa: E402

import paper_2403_05802_b200 as sfg  # noqa: E402

ctx = sfg.Context(0, torch.cuda.current_stream().cuda_stream)
ctx.read_matrix_market(path)  # warm: allocations cached, file in page cache
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    t0 = time.perf_counter()
    t = ctx.read_matrix_market(path)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
out = {"entries": int(r.size), "bytes": size, "device_s": best, "device_MB_per_s": size / best / 1e6,
       "device_Mnnz_per_s": r.size / best / 1e6}
try:
    import oracle
    if oracle.ref_available():
        ref = oracle.Ref()
        t0 = time.perf_counter()
        coo = ref.read_mm(path)
        out["reference_s"] = time.perf_counter() - t0
        out["reference_Mnnz_per_s"] = r.size / out["reference_s"] / 1e6
        rr, cc, vv = coo.arrays()
        dr, dc, dv = t.coo_arrays()
        out["bit_exact"] = bool(np.array_equal(rr, dr) and np.array_equal(cc, dc)
                                and np.array_equal(vv.astype(np.float32).view(np.uint32), dv.view(np.uint32)))
except Exception as e:  # pragma: no cover
    out["reference_error"] = str(e)
print(json.dumps(out))
