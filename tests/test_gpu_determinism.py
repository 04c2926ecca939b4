"""Run-to-run bit-identity of SpMV / SpMM. The reference reduces its thread
partials in worker order "so the result is deterministic"
(kernel.hpp:370-384); the device kernels reduce without float atomics
(carry slots added in chunk order, per-lane partials summed in lane
order), so ten launches on the same input give the same bits. CSC is the
exception (a scatter over rows; documented in DESIGN.md)."""
import numpy as np
import pytest
import torch

from matrices import power_law_coo

pytestmark = pytest.mark.gpu

FORMATS = ["COO", "CSR", "DCSR", "ELL", "HYB(8)", "BCSR(4,4)", "BCSR(16,16)"]


def _matrix(ctx, fmt, m=20000, n=20000):
    # heavy rows (hundreds of entries, spanning several merge-path / COO
    # chunks) next to empty and short rows
    r, c, v = power_law_coo(3, m, n, avg=12, alpha=1.1)
    return ctx.convert(ctx.from_coo(m, n, r, c, v), fmt), m, n


@pytest.mark.parametrize("fmt", FORMATS)
def test_spmv_bit_identical(ctx, fmt):
    a, m, n = _matrix(ctx, fmt)
    x = torch.rand(n, device="cuda") * 2 - 1
    y = torch.empty(m, device="cuda")
    outs = []
    for _ in range(10):
        y.fill_(float("nan"))
        ctx.spmv_device(a, x.data_ptr(), y.data_ptr())
        outs.append(y.clone())
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int32), outs[0].view(torch.int32)), fmt


@pytest.mark.parametrize("nd", [1, 16, 32, 64, 128, 40])
@pytest.mark.parametrize("fmt", FORMATS)
def test_spmm_bit_identical(ctx, fmt, nd):
    a, m, n = _matrix(ctx, fmt, 6000, 6000)
    b = torch.rand(n * nd, device="cuda") * 2 - 1
    c = torch.empty(m * nd, device="cuda")
    outs = []
    for _ in range(10):
        c.fill_(float("nan"))
        ctx.spmm_device(a, b.data_ptr(), 0, nd, c.data_ptr())
        outs.append(c.clone())
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int32), outs[0].view(torch.int32)), (fmt, nd)


def test_spmm_accumulate_bit_identical(ctx):
    a, m, n = _matrix(ctx, "CSR", 6000, 6000)
    nd = 32
    b = torch.rand(n * nd, device="cuda")
    c0 = torch.rand(m * nd, device="cuda")
    outs = []
    for _ in range(5):
        c = c0.clone()
        ctx.spmm_device(a, b.data_ptr(), 0, nd, c.data_ptr(), accumulate=True)
        outs.append(c)
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("block,density", [(16, 0.1), (16, 0.6), (4, 0.1)])
def test_bcsr_tensor_core_bit_identical(ctx, block, density):
    """The tcgen05 BCSR paths with bf16 values and B (16x16 panel kernel:
    MMA warps own block rows; 4x4 window kernel: one MMA warp per
    accumulator) give the same bits on every run."""
    import paper_2403_05802_b200 as sfg
    rng = np.random.default_rng(block)
    m = n = 2048
    nb = m // block
    br, bc = np.nonzero(rng.random((nb, nb)) < density)
    ii, jj = np.meshgrid(np.arange(block), np.arange(block), indexing="ij")
    r = (br[:, None] * block + ii.ravel()[None, :]).ravel()
    c = (bc[:, None] * block + jj.ravel()[None, :]).ravel()
    v = (rng.random(len(r)) * 2 - 1).astype(np.float32).astype(np.float64)
    a = ctx.convert(ctx.from_coo(m, n, r, c, v), f"BCSR({block},{block})", value_dtype=sfg.BF16)
    b = (torch.rand(n * 128, device="cuda") * 2 - 1).to(torch.bfloat16)
    cc = torch.empty(m * 128, device="cuda")
    outs = []
    for _ in range(10):
        cc.fill_(float("nan"))
        ctx.spmm_device(a, b.data_ptr(), sfg.BF16, 128, cc.data_ptr())
        outs.append(cc.clone())
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int32), outs[0].view(torch.int32)), (block, density)
