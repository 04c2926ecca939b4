"""Config-5 CSR SpMM (R-MAT scale S, nd = 32) timing under the SFG_SPMM_*
knobs of the current process: median of K launches (CUDA events, L2
flushed before each), and a bit-identity check of C across launches.

  SFG_SPMM_L2=4 python scripts/spmm_cfg5_exp.py [scale] [launches]
"""
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2403_05802_b200 as sfg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
k = int(sys.argv[2]) if len(sys.argv) > 2 else 5
nd = 32
stream = torch.cuda.current_stream()
ctx = sfg.Context(0, stream.cuda_stream)
coo = ctx.gen_rmat(7, scale, 16 << scale)
m, n = coo.shape
a = ctx.convert(coo, "CSR")
del coo
b = torch.empty(n * nd, dtype=torch.float32, device="cuda")
ctx.gen_dense(3, n * nd, b.data_ptr())
c = torch.empty(m * nd, dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ms, sums = [], []
ref = None
for i in range(k + 1):
    flush.zero_()
    c.fill_(float("nan"))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.spmm_device(a, b.data_ptr(), sfg.F32, nd, c.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    if i:
        ms.append(e0.elapsed_time(e1))
    if ref is None:
        ref = c.clone()
    elif not torch.equal(ref.view(torch.int32), c.view(torch.int32)):
        print("NOT bit-identical across launches")
print(f"L2={os.environ.get('SFG_SPMM_L2', '0')} MINB={os.environ.get('SFG_SPMM_MINB', '-')} "
      f"HOT={os.environ.get('SFG_SPMM_HOT', '-')} scale={scale} nnz={a.view().nvals} "
      f"spmm ms median {statistics.median(ms):.3f} min {min(ms):.3f} nan={bool(torch.isnan(c).any())}")
