"""GPU parity: SpMM C = A B over every format (fp32 and bf16 B) vs the f64
oracle, |C_hat - C| <= 1e-5 * sum_j |a_ij| |B_jk| per output."""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL
from matrices import power_law_coo, random_coo

pytestmark = pytest.mark.gpu

FORMATS = ["COO", "CSR", "CSC", "DCSR", "ELL", "BCSR(2,2)", "BCSR(4,4)", "BCSR(16,16)", "HYB(3)"]


def oracle_spmm(port, p, fmt, b):
    if fmt.startswith("BCSR"):
        rr, cc = (int(t) for t in fmt[5:-1].split(","))
        return port.spmm(port.convert(p, "BCSR", rr, cc), b)
    if fmt.startswith("HYB"):
        t = int(fmt[4:-1])
        s, r, _ = port.decompose_rows(p, t)
        return port.spmm(port.convert(r, "ELL"), b) + port.spmm(port.convert(s, "COO"), b)
    return port.spmm(port.convert(p, fmt), b)


def abs_bound(r, c, v, m, b):
    out = np.zeros((m, b.shape[1]))
    np.add.at(out, r, np.abs(v)[:, None] * np.abs(b[c]))
    return out


def check(cd, cr, bound, ctx):
    err = np.abs(cd.astype(np.float64) - cr)
    bad = err > TOL * bound + 1e-30
    assert not bad.any(), (ctx, np.argwhere(bad)[:3], err[bad][:3])


@pytest.mark.parametrize("nd", [1, 7, 32, 64, 128])
@pytest.mark.parametrize("fmt", FORMATS)
def test_spmm_formats(ctx, port, fmt, nd):
    m, n = 130, 97
    r, c, v = random_coo(nd, m, n, 0.2, zeros=0.1)
    rng = np.random.default_rng(nd)
    b = (rng.random((n, nd)) * 2 - 1).astype(np.float32)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    cd = ctx.spmm(ctx.convert(d, fmt), b)
    cr = oracle_spmm(port, p, fmt, b.astype(np.float64))
    check(cd, cr, abs_bound(r, c, v, m, b.astype(np.float64)), (fmt, nd))


@pytest.mark.parametrize("fmt", ["CSR", "COO", "DCSR", "HYB(8)"])
def test_spmm_power_law_nd64(ctx, port, fmt):
    m, n = 3000, 2000
    r, c, v = power_law_coo(1, m, n, avg=15, alpha=1.2)
    b = (np.random.default_rng(0).random((n, 64)) * 2 - 1).astype(np.float32)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    cd = ctx.spmm(ctx.convert(d, fmt), b)
    cr = oracle_spmm(port, p, fmt, b.astype(np.float64))
    check(cd, cr, abs_bound(r, c, v, m, b.astype(np.float64)), fmt)


def to_bf16_bits(a):
    f = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    return (((f + 0x7FFF + ((f >> 16) & 1)) >> 16)).astype(np.uint16)


def bits_to_f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("fmt", ["CSR", "BCSR(16,16)", "BCSR(4,4)", "ELL"])
def test_spmm_bf16_b(ctx, port, fmt):
    """bf16 B: the oracle runs on the bf16-rounded operand."""
    m, n, nd = 256, 192, 128
    r, c, v = random_coo(9, m, n, 0.15)
    b = (np.random.default_rng(2).random((n, nd)) * 2 - 1).astype(np.float32)
    bb = to_bf16_bits(b)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    cd = ctx.spmm(ctx.convert(d, fmt), bb, b_dtype=sfg.BF16)
    b64 = bits_to_f64(bb)
    cr = oracle_spmm(port, p, fmt, b64)
    check(cd, cr, abs_bound(r, c, v, m, b64), fmt)


def test_spmm_accumulate_and_ld(ctx):
    t = ctx.convert(ctx.from_coo(2, 2, [0, 1], [1, 0], [2.0, 3.0]), "CSR")
    b = np.array([[1, 2, 0], [3, 4, 0]], np.float32)  # ldb = 3, nd = 2
    cbuf = ctx.buffer(2 * 4 * 4).upload(np.full((2, 4), 10, np.float32))
    bbuf = ctx.buffer(b.nbytes).upload(b)
    ctx.spmm_device(t, bbuf.ptr, sfg.F32, 2, cbuf.ptr, ldb=3, ldc=4, accumulate=True)
    out = cbuf.download(np.float32, 8).reshape(2, 4)
    assert out.tolist() == [[16, 18, 10, 10], [13, 16, 10, 10]]


def bf16_round(a):
    return bits_to_f64(to_bf16_bits(a))


@pytest.mark.parametrize("shape", [(256, 256), (250, 200), (16, 16), (1000, 3000), (4096, 512)])
@pytest.mark.parametrize("density", [0.02, 0.3, 0.9])  # 0.9: block columns shared by > 16 block rows
def test_bcsr16_bf16_tensor_core(ctx, port, shape, density):
    """BCSR(16,16) with bf16 values and bf16 B, nd = 128: the tcgen05 path
    (bcsr_tc.cu). The oracle runs on the bf16-rounded values and B."""
    m, n = shape
    rng = np.random.default_rng(m + n)
    nbr, nbc = (m + 15) // 16, (n + 15) // 16
    mask = rng.random((nbr, nbc)) < density
    mask[nbr // 2] = False  # an empty block row
    br, bc = np.nonzero(mask)
    ii, jj = np.meshgrid(np.arange(16), np.arange(16), indexing="ij")
    rows = (br[:, None] * 16 + ii.ravel()[None, :]).ravel()
    cols = (bc[:, None] * 16 + jj.ravel()[None, :]).ravel()
    keep = (rows < m) & (cols < n)
    rows, cols = rows[keep], cols[keep]
    vals = (0.5 + rng.integers(0, 1 << 23, rows.size) / 2.0 ** 23) * np.where(rng.random(rows.size) < .5, -1, 1)
    vals = bf16_round(vals)
    b = (rng.random((n, 128)) * 2 - 1).astype(np.float32)
    bb = to_bf16_bits(b)
    d = ctx.convert(ctx.from_coo(m, n, rows, cols, vals), "BCSR(16,16)", value_dtype=sfg.BF16)
    cd = ctx.spmm(d, bb, b_dtype=sfg.BF16)
    p = port.from_coo(m, n, rows, cols, vals)
    b64 = bits_to_f64(bb)
    cr = port.spmm(port.convert(p, "BCSR", 16, 16), b64)
    check(cd, cr, abs_bound(rows, cols, vals, m, b64), ("bcsr-tc", shape, density))


@pytest.mark.parametrize("shape", [(256, 256), (250, 202), (9, 40), (1000, 3000), (4100, 520)])
@pytest.mark.parametrize("density", [0.01, 0.1, 0.9])
@pytest.mark.parametrize("accumulate", [False, True])
def test_bcsr4_bf16_tensor_core(ctx, port, shape, density, accumulate):
    """BCSR(4,4) with bf16 values and bf16 B, nd = 128: the tcgen05 path over
    128-row x 16-column windows (bcsr_tc.cu k_bcsr4_tc). The oracle runs on
    the bf16-rounded values and B."""
    m, n = shape
    rng = np.random.default_rng(m * 3 + n)
    nbr, nbc = (m + 3) // 4, (n + 3) // 4
    mask = rng.random((nbr, nbc)) < density
    mask[nbr // 2] = False  # an empty block row
    if nbr > 64:
        mask[32:64] = False  # an empty 32-block-row group
    br, bc = np.nonzero(mask)
    ii, jj = np.meshgrid(np.arange(4), np.arange(4), indexing="ij")
    rows = (br[:, None] * 4 + ii.ravel()[None, :]).ravel()
    cols = (bc[:, None] * 4 + jj.ravel()[None, :]).ravel()
    keep = (rows < m) & (cols < n) & (rng.random(rows.size) < 0.9)
    rows, cols = rows[keep], cols[keep]
    vals = bf16_round((rng.random(rows.size) * 2 - 1) * np.exp2(rng.integers(-3, 3, rows.size)))
    b = (rng.random((n, 128)) * 2 - 1).astype(np.float32)
    bb = to_bf16_bits(b)
    d = ctx.convert(ctx.from_coo(m, n, rows, cols, vals), "BCSR(4,4)", value_dtype=sfg.BF16)
    c0 = (rng.random((m, 128)) * 2 - 1).astype(np.float32)
    cbuf = ctx.buffer(c0.nbytes).upload(c0)
    bbuf = ctx.buffer(bb.nbytes).upload(bb)
    ctx.spmm_device(d, bbuf.ptr, sfg.BF16, 128, cbuf.ptr, accumulate=accumulate)
    cd = cbuf.download(np.float32, m * 128).reshape(m, 128)
    b64 = bits_to_f64(bb)
    cr = port.spmm(port.convert(port.from_coo(m, n, rows, cols, vals), "BCSR", 4, 4), b64)
    if accumulate:
        cr = cr + c0.astype(np.float64)
    check(cd, cr, abs_bound(rows, cols, vals, m, b64) + np.abs(c0) * accumulate, ("bcsr4-tc", shape, density))


@pytest.mark.parametrize("shape", [(256, 256), (250, 200), (1000, 3000), (4096, 512)])
@pytest.mark.parametrize("density", [0.02, 0.3, 0.9])
@pytest.mark.parametrize("accumulate", [False, True])
def test_bcsr16_fp32_tensor_core(ctx, port, shape, density, accumulate):
    """BCSR(16,16) with fp32 values and fp32 B, nd = 128: the 3xTF32 tcgen05
    path (bcsr_tc.cu, kind::tf32 hi.hi + lo.hi + hi.lo) held to the fp32
    tolerance against the f64 oracle on full-mantissa operands."""
    m, n = shape
    rng = np.random.default_rng(m * 7 + n)
    nbr, nbc = (m + 15) // 16, (n + 15) // 16
    mask = rng.random((nbr, nbc)) < density
    mask[nbr // 2] = False  # an empty block row
    br, bc = np.nonzero(mask)
    ii, jj = np.meshgrid(np.arange(16), np.arange(16), indexing="ij")
    rows = (br[:, None] * 16 + ii.ravel()[None, :]).ravel()
    cols = (bc[:, None] * 16 + jj.ravel()[None, :]).ravel()
    keep = (rows < m) & (cols < n) & (rng.random(rows.size) < 0.95)  # some zeros inside blocks
    rows, cols = rows[keep], cols[keep]
    vals = ((rng.random(rows.size) * 2 - 1) * np.exp2(rng.integers(-6, 6, rows.size))).astype(np.float32)
    b = ((rng.random((n, 128)) * 2 - 1) * np.exp2(rng.integers(-4, 4, (n, 128)))).astype(np.float32)
    d = ctx.convert(ctx.from_coo(m, n, rows, cols, vals.astype(np.float64)), "BCSR(16,16)")
    c0 = (rng.random((m, 128)) * 2 - 1).astype(np.float32)
    cbuf = ctx.buffer(c0.nbytes).upload(c0)
    bbuf = ctx.buffer(b.nbytes).upload(b)
    ctx.spmm_device(d, bbuf.ptr, sfg.F32, 128, cbuf.ptr, accumulate=accumulate)
    cd = cbuf.download(np.float32, m * 128).reshape(m, 128)
    p = port.from_coo(m, n, rows, cols, vals.astype(np.float64))
    cr = port.spmm(port.convert(p, "BCSR", 16, 16), b.astype(np.float64))
    if accumulate:
        cr = cr + c0.astype(np.float64)
    bound = abs_bound(rows, cols, vals.astype(np.float64), m, b.astype(np.float64)) + np.abs(c0) * accumulate
    check(cd, cr, bound, ("bcsr-tf32", shape, density, accumulate))


@pytest.mark.parametrize("accumulate", [False, True])
def test_spmm_csr_heavy_and_empty_rows(ctx, port, accumulate):
    """CSR SpMM is load balanced over (rows + entries): one row far longer
    than a merge chunk (1024 items), runs of empty rows, a full last row."""
    rng = np.random.default_rng(4)
    m, n, nd = 5000, 6000, 32
    rows = [np.full(5000, 3), np.full(2500, 4), rng.integers(100, 4000, 20000), np.full(3000, m - 1)]
    r = np.concatenate(rows)
    c = rng.integers(0, n, len(r))
    key = np.unique(r.astype(np.int64) * n + c)
    r, c = key // n, key % n
    v = (rng.random(len(r)) * 2 - 1).astype(np.float32)
    b = (rng.random((n, nd)) * 2 - 1).astype(np.float32)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    a = ctx.convert(d, "CSR")
    c0 = (rng.random((m, nd)) * 2 - 1).astype(np.float32)
    cbuf = ctx.buffer(c0.nbytes).upload(c0)
    bbuf = ctx.buffer(b.nbytes).upload(b)
    ctx.spmm_device(a, bbuf.ptr, sfg.F32, nd, cbuf.ptr, accumulate=accumulate)
    cd = cbuf.download(np.float32, m * nd).reshape(m, nd)
    cr = port.spmm(port.convert(p, "CSR"), b.astype(np.float64))
    if accumulate:
        cr = cr + c0.astype(np.float64)
    check(cd, cr, abs_bound(r, c, v, m, b.astype(np.float64)) + np.abs(c0) * accumulate, ("heavy", accumulate))


@pytest.mark.parametrize("fmt", ["CSR", "DCSR", "COO", "ELL"])
@pytest.mark.parametrize("nd", [32, 64, 128])
def test_spmm_unaligned_dense_pointers(ctx, port, fmt, nd):
    """B and C may start at any element offset (vector paths are chosen only
    for aligned pointers)."""
    rng = np.random.default_rng(nd)
    m, n = 300, 200
    key = np.unique(rng.integers(0, m * n, 3000))
    r, c = key // n, key % n
    v = (rng.random(len(r)) * 2 - 1).astype(np.float32)
    b = (rng.random((n, nd)) * 2 - 1).astype(np.float32)
    a = ctx.convert(ctx.from_coo(m, n, r, c, v), fmt)
    bbuf = ctx.buffer(b.nbytes + 4).upload(np.concatenate([np.zeros(1, np.float32), b.ravel()]))
    cbuf = ctx.buffer(m * nd * 4 + 4)
    ctx.spmm_device(a, bbuf.ptr + 4, sfg.F32, nd, cbuf.ptr + 4)
    cd = cbuf.download(np.float32, m * nd + 1)[1:].reshape(m, nd)
    cr = port.spmm(port.convert(port.from_coo(m, n, r, c, v), fmt), b.astype(np.float64))
    check(cd, cr, abs_bound(r, c, v, m, b.astype(np.float64)), (fmt, nd, "unaligned"))
