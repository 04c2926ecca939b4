"""Drive scripts/coo_exp.cu on the config-2 COO part (R-MAT s22, HYB(8))."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2403_05802_b200 as sfg  # noqa: E402

lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_bin", "libcooexp.so"))
lib.coo_exp_run.restype = C.c_float
lib.coo_exp_run.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_int64, C.c_int]
ctx = sfg.Context(0, torch.cuda.current_stream().cuda_stream)
coo = ctx.gen_rmat(7, 22, 16 << 22)
h = ctx.convert(coo, "HYB(8)")
ell, part = h.parts()
v = part.view()
nnz = int(v.nvals)
row, col, val = v.level[0].idx, v.level[1].idx, v.values
n = coo.shape[1]
x = torch.rand(n, device="cuda")
out = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
names = {0: "strided R16 +row", 1: "strided R16 no-row", 2: "strided R8 +row", 3: "int4 x2 +row",
         4: "int4 x2 no-row", 5: "gather-only R16", 6: "int4 x4 +row"}
for var in ([] if os.environ.get("SKIP_VARIANTS") else range(7)):
    for bps in (4, 8):
        ms = lib.coo_exp_run(var, bps, row, col, val, x.data_ptr(), out.data_ptr(), nnz, 5)
        print(f"{names[var]:22s} blocks/SM {bps}: {ms * 1e3:7.1f} us  {nnz / ms / 1e6:7.1f} Gnnz/s", flush=True)
# the production kernel, same data
y = torch.zeros(coo.shape[0], device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
best = 1e9
for _ in range(6):
    ev[0].record()
    ctx.spmv_device(part, x.data_ptr(), y.data_ptr())
    ev[1].record()
    torch.cuda.synchronize()
    best = min(best, ev[0].elapsed_time(ev[1]))
print(f"production k_spmv_coo (+zero y): {best * 1e3:7.1f} us")
