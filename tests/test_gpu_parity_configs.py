"""GPU parity at the BASELINE.json configurations' own sizes, plus the
kernels only those sizes reach.

* k_spmm_rows_batch (the short-row DCSR SpMM: <= 8 entries per stored row,
  config 3's dominant kernel) against the f64 oracle: nd 32/64/128, vector
  and strided (non-vector) operands, long runs of empty rows, accumulate.
* config 3 in full (4M x 4M, 2/row): DCSR and CSC bit-exact, DCSR SpMM N=64.
* config 5 (R-MAT scale 26): CSR bit-exact over the whole matrix and against
  the oracle on row blocks, SpMM N=32 on the heaviest rows (0-1023) and a
  mid block.
* config 4 (BCSR 16x16 bf16, 512K x 512K, 10 % blocks): the tcgen05 SpMM on
  three block-row groups of the full matrix, the oracle on the bf16-rounded
  operands; and the low-density k_bcsr_tc_group path.
* a direct GPU vs unmodified-reference (oracle/_ref) check at R-MAT scale 14
  for every target format plus SpMV and SpMM.

Tolerance (north_star): |c_hat - c| <= 1e-5 * sum_j |a_ij| |b_jk| per output
(+ |c_in| when accumulating); conversions bit-exact.
"""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL, assert_same_materialized

pytestmark = pytest.mark.gpu


def check_close(cd, cr, bound, ctx):
    err = np.abs(np.asarray(cd, np.float64) - cr)
    bad = err > TOL * bound + 1e-30
    if bad.any():
        i = tuple(np.argwhere(bad)[0])
        raise AssertionError(f"{ctx}: {int(bad.sum())} outputs out of tolerance, first {i}: "
                             f"dev={cd[i]!r} ref={cr[i]!r} err={err[i]:.3e} bound={TOL * bound[i]:.3e}")


def oracle_spmm_bound(port, m, n, r, c, v, b, fmt="CSR"):
    """(C, sum_j |a_ij||b_jk|) by the C port in f64."""
    ca = port.spmm(port.convert(port.from_coo(m, n, r, c, v), fmt), b)
    cb = port.spmm(port.convert(port.from_coo(m, n, r, c, np.abs(v)), fmt), np.abs(b))
    return ca, cb


def short_rows_coo(seed, m, n, stored, max_len=8, gap_runs=True):
    """Row-sorted unique COO with `stored` nonempty rows of 1..max_len
    entries (mean <= 8 so the short-row kernel is chosen); with gap_runs
    the stored rows come in clusters separated by long empty runs."""
    rng = np.random.default_rng(seed)
    if gap_runs:
        # clusters of ~64 stored rows with runs of up to 20,000 empty rows between
        starts = np.sort(rng.choice(m - 128, stored // 64 + 1, replace=False))
        rows = np.unique(np.concatenate([s + np.sort(rng.choice(128, 64, replace=False)) for s in starts]))
        rows = rows[rows < m][:stored]
    else:
        rows = np.sort(rng.choice(m, stored, replace=False))
    lens = rng.integers(1, max_len + 1, len(rows))
    lens[rng.random(len(rows)) < 0.02] = 3 * max_len  # a few longer rows
    r = np.repeat(rows, lens)
    c = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lens])
    v = (0.5 + rng.integers(0, 1 << 23, len(r)) / float(1 << 23)) * np.where(rng.random(len(r)) < 0.5, -1, 1)
    return r.astype(np.int64), c.astype(np.int64), v.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("nd", [32, 64, 128])
@pytest.mark.parametrize("layout", ["vector", "strided"])
@pytest.mark.parametrize("accumulate", [False, True])
def test_spmm_rows_batch_short_dcsr(ctx, port, nd, layout, accumulate):
    m, n = 1 << 16, 1 << 14
    r, c, v = short_rows_coo(nd + accumulate, m, n, stored=6000)
    assert len(r) <= 8 * len(np.unique(r))  # the <= 8 entries/row kernel is the one chosen
    a = ctx.convert(ctx.from_coo(m, n, r, c, v), "DCSR")
    rng = np.random.default_rng(5)
    # strided: leading dimensions not multiples of the vector width
    ldb, ldc = (nd, nd) if layout == "vector" else (nd + 1, nd + 3)
    b = (rng.random((n, ldb)) * 2 - 1).astype(np.float32)
    c0 = (rng.random((m, ldc)) * 2 - 1).astype(np.float32) if accumulate else np.full((m, ldc), 7.0, np.float32)
    bb = sfg.DeviceBuffer(ctx, b.nbytes).upload(b)
    cbuf = sfg.DeviceBuffer(ctx, c0.nbytes).upload(c0)
    ctx.spmm_device(a, bb.ptr, sfg.F32, nd, cbuf.ptr, ldb=ldb, ldc=ldc, accumulate=accumulate)
    out = cbuf.download(np.float32, m * ldc).reshape(m, ldc)
    cr, bound = oracle_spmm_bound(port, m, n, r, c, v, b[:, :nd].astype(np.float64), "DCSR")
    if accumulate:
        cr = cr + c0[:, :nd]
        bound = bound + np.abs(c0[:, :nd])
    check_close(out[:, :nd], cr, bound, (nd, layout, accumulate))
    # the columns past nd of a strided C are not touched
    np.testing.assert_array_equal(out[:, nd:], c0[:, nd:])


def test_spmm_rows_batch_no_gaps_and_tail(ctx, port):
    """Every row stored except a long empty tail (the zeroing after the last
    stored row up to M), nd = 64."""
    m, n, nd = 50_000, 4096, 64
    rng = np.random.default_rng(3)
    rows = np.arange(30_000)
    lens = rng.integers(1, 5, len(rows))
    r = np.repeat(rows, lens)
    c = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lens])
    v = (rng.random(len(r)) + 0.5).astype(np.float32).astype(np.float64)
    a = ctx.convert(ctx.from_coo(m, n, r, c, v), "DCSR")
    b = (rng.random((n, nd)) * 2 - 1).astype(np.float32)
    out = ctx.spmm(a, b)
    cr, bound = oracle_spmm_bound(port, m, n, r, c, v, b.astype(np.float64), "DCSR")
    check_close(out, cr, bound, "tail")
    assert not out[30_000:].any()


# --------------------------------------------------------------- config 3
@pytest.mark.slow
def test_config3_full(ctx, port):
    """BASELINE config 3 at full size: hypersparse 4M x 4M, 2/row. DCSR and
    CSC bit-exact; DCSR SpMM N=64 (the short-row kernel) within tolerance."""
    m = n = 1 << 22
    d, p = ctx.gen_hypersparse(5, m, n, 2 * m), port.gen_hypersparse(5, m, n, 2 * m)
    r, c, v = p.arrays()
    for x, y in zip(d.coo_arrays(), (r, c, v)):
        np.testing.assert_array_equal(x.astype(np.float64), y)
    dcsr = ctx.convert(d, "DCSR")
    assert_same_materialized(dcsr.download(), port.convert(p, "DCSR").download(), "cfg3 DCSR")
    assert_same_materialized(ctx.convert(d, "CSC").download(), port.convert(p, "CSC").download(), "cfg3 CSC")
    nd = 64
    bdev = sfg.DeviceBuffer(ctx, n * nd * 4)
    ctx.gen_dense(3, n * nd, bdev.ptr)
    cdev = sfg.DeviceBuffer(ctx, m * nd * 4).upload(np.full(m * nd, np.nan, np.float32))
    ctx.spmm_device(dcsr, bdev.ptr, sfg.F32, nd, cdev.ptr)
    out = cdev.download(np.float32, m * nd).reshape(m, nd)
    b = bdev.download(np.float32, n * nd).reshape(n, nd).astype(np.float64)
    cr, bound = oracle_spmm_bound(port, m, n, r, c, v, b, "DCSR")
    check_close(out, cr, bound, "cfg3 SpMM")


# --------------------------------------------------------------- config 5
@pytest.fixture(scope="module")
def cfg5(ctx):
    """R-MAT scale 26 (config 5) on the device, its CSR, and B (N = 32)."""
    torch = pytest.importorskip("torch")
    coo = ctx.gen_rmat(7, 26, 16 << 26)
    csr = ctx.convert(coo, "CSR")
    n = 1 << 26
    b = torch.empty(n * 32, dtype=torch.float32, device="cuda")
    ctx.gen_dense(3, n * 32, b.data_ptr())
    torch.cuda.synchronize()
    yield coo, csr, b
    del csr, coo, b
    ctx.release_cached()


def csr_arrays(ctx, t, r0=None, r1=None):
    """(ptr, idx, val) of a device CSR, rows [r0, r1) only when given."""
    v = t.view()
    m = v.rows
    r0, r1 = (0, m) if r0 is None else (r0, r1)
    ptr = ctx.download_ptr(v.level[1].ptr, np.int32, r1 - r0 + 1, r0).astype(np.int64)
    idx = ctx.download_ptr(v.level[1].idx, np.int32, ptr[-1] - ptr[0], ptr[0])
    val = ctx.download_ptr(v.values, np.float32, ptr[-1] - ptr[0], ptr[0])
    return ptr, idx, val


@pytest.mark.slow
def test_config5_csr_bit_exact(ctx, port, cfg5):
    """Whole matrix: CSR ptr = prefix sum of the row counts of the sorted
    unique COO, idx/val = its columns/values (Fill(0)+Merge(0) of a sorted
    COO, operators.hpp:346-391); row blocks against the oracle's materialize."""
    coo, csr, _ = cfg5
    row, col, val = coo.coo_arrays()
    m = 1 << 26
    key = row.astype(np.int64) << 32 | col.astype(np.int64)
    assert np.all(np.diff(key) > 0)  # canonical: sorted and unique
    del key
    ptr, idx, v = csr_arrays(ctx, csr)
    want = np.zeros(m + 1, np.int64)
    np.cumsum(np.bincount(row, minlength=m), out=want[1:])
    np.testing.assert_array_equal(ptr, want)
    np.testing.assert_array_equal(idx, col)
    np.testing.assert_array_equal(v.view(np.uint32), val.view(np.uint32))
    for r0, r1 in ((0, 1024), (1 << 25, (1 << 25) + 4096), (m - 4096, m)):
        e0, e1 = want[r0], want[r1]
        p = port.from_coo(r1 - r0, m, row[e0:e1] - r0, col[e0:e1], val[e0:e1])
        o = port.convert(p, "CSR").download()
        dptr, didx, dval = csr_arrays(ctx, csr, r0, r1)
        np.testing.assert_array_equal(dptr - dptr[0], o.levels[1].ptr)
        np.testing.assert_array_equal(didx, o.levels[1].idx)
        np.testing.assert_array_equal(dval.astype(np.float64), o.values)


@pytest.mark.slow
def test_config5_spmm_blocks(ctx, port, cfg5):
    """SpMM N=32 over the full scale-26 CSR; rows 0-1023 (the heaviest, up
    to ~10^5 entries each) and a mid block against the oracle."""
    import torch
    coo, csr, b = cfg5
    m, nd = 1 << 26, 32
    c = torch.full((m * nd,), float("nan"), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ctx.spmm_device(csr, b.data_ptr(), sfg.F32, nd, c.data_ptr())
    ctx.synchronize()
    assert not torch.isnan(c).any().item()
    bm = b.view(-1, nd)
    for r0, r1 in ((0, 1024), (1 << 25, (1 << 25) + 8192)):
        ptr, idx, val = csr_arrays(ctx, csr, r0, r1)
        rows = np.repeat(np.arange(r1 - r0), np.diff(ptr))
        ucols, cmap = np.unique(idx, return_inverse=True)
        bsub = bm[torch.from_numpy(ucols.astype(np.int64)).cuda()].cpu().numpy().astype(np.float64)
        cr, bound = oracle_spmm_bound(port, r1 - r0, len(ucols), rows, cmap, val.astype(np.float64), bsub)
        out = c.view(-1, nd)[r0:r1].cpu().numpy()
        check_close(out, cr, bound, ("cfg5", r0))


# --------------------------------------------------------------- config 4
def bf16_bits_to_f64(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def bcsr_group_check(ctx, port, a, bbits, c_out, nd, brows, ctx_name):
    """Block rows [b0, b1) of a device BCSR(16,16) bf16 SpMM result against
    the oracle on the same (bf16) values and B."""
    v = a.view()
    m, n = v.rows, v.cols
    nbr = v.level[1].ptr_len - 1
    b64 = bf16_bits_to_f64(bbits).reshape(n, nd)
    for b0, b1 in brows:
        b1 = min(b1, nbr)
        ptr = ctx.download_ptr(v.level[1].ptr, np.int32, b1 - b0 + 1, b0).astype(np.int64)
        bcol = ctx.download_ptr(v.level[1].idx, np.int32, ptr[-1] - ptr[0], ptr[0]).astype(np.int64)
        vals = ctx.download_ptr(v.values, np.uint16, (ptr[-1] - ptr[0]) * 256, ptr[0] * 256)
        blk_row = np.repeat(np.arange(b1 - b0), np.diff(ptr))
        ii, jj = np.meshgrid(np.arange(16), np.arange(16), indexing="ij")
        r = (blk_row[:, None] * 16 + ii.reshape(-1)[None, :]).reshape(-1)
        cidx = (bcol[:, None] * 16 + jj.reshape(-1)[None, :]).reshape(-1)
        vv = bf16_bits_to_f64(vals)
        keep = (vv != 0) & (r + b0 * 16 < m) & (cidx < n)
        rows_here = min(b1 * 16, m) - b0 * 16
        cr, bound = oracle_spmm_bound(port, rows_here, n, r[keep], cidx[keep], vv[keep], b64)
        check_close(c_out[b0 * 16: b0 * 16 + rows_here], cr, bound, (ctx_name, b0))


@pytest.mark.slow
def test_config4_tcgen05_full_matrix_groups(ctx, port):
    """tcgen05 BCSR(16,16) bf16 SpMM N=128 on the full 512K x 512K, 10 %
    block-density matrix: three 32-block-row groups (first, middle, last)."""
    torch = pytest.importorskip("torch")
    m = 1 << 19
    nd = 128
    a = ctx.gen_block_sparse(11, m, m, 16, 16, 0.1, value_dtype=sfg.BF16)
    g = torch.Generator(device="cpu").manual_seed(4)
    b = (torch.rand((m, nd), generator=g) * 2 - 1).to(torch.bfloat16)
    bdev = b.cuda()
    c = torch.full((m, nd), float("nan"), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ctx.spmm_device(a, bdev.data_ptr(), sfg.BF16, nd, c.data_ptr())
    ctx.synchronize()
    nbr = m // 16
    groups = [(0, 32), (nbr // 2, nbr // 2 + 32), (nbr - 32, nbr)]
    rows = np.concatenate([np.arange(b0 * 16, b1 * 16) for b0, b1 in groups])
    c_host = np.full((m, nd), np.nan, np.float32)
    c_host[rows] = c[torch.from_numpy(rows).cuda()].cpu().numpy()
    bcsr_group_check(ctx, port, a, b.view(torch.int16).numpy().view(np.uint16), c_host, nd, groups, "cfg4")


@pytest.mark.parametrize("density", [0.004, 0.002])
def test_bcsr_tc_group_low_density(ctx, port, density):
    """Block density <= 0.5 %: the plan is skipped and k_bcsr_tc_group
    merges the block rows' columns in the kernel."""
    torch = pytest.importorskip("torch")
    m, nd = 32768, 128
    a = ctx.gen_block_sparse(13, m, m, 16, 16, density, value_dtype=sfg.BF16)
    g = torch.Generator(device="cpu").manual_seed(6)
    b = (torch.rand((m, nd), generator=g) * 2 - 1).to(torch.bfloat16)
    bdev = b.cuda()
    c = torch.full((m, nd), float("nan"), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ctx.spmm_device(a, bdev.data_ptr(), sfg.BF16, nd, c.data_ptr())
    ctx.synchronize()
    bcsr_group_check(ctx, port, a, b.view(torch.int16).numpy().view(np.uint16), c.cpu().numpy(), nd,
                     [(0, m // 16)], ("tc_group", density))


# ------------------------------------------ GPU vs the unmodified reference
S14 = 14


@pytest.fixture(scope="module")
def rmat14(ctx, port, ref):
    p = port.gen_rmat(7, S14, 16 << S14)
    r, c, v = p.arrays()
    m = 1 << S14
    return ctx.gen_rmat(7, S14, 16 << S14), ref.from_coo(m, m, r, c, v), (r, c, v)


@pytest.mark.parametrize("fmt", ["COO", "CSR", "CSC", "DCSR", "BCSR(4,4)"])
def test_rmat14_vs_reference_convert(ctx, ref, rmat14, fmt):
    d, rt, _ = rmat14
    if fmt.startswith("BCSR"):
        want = ref.convert(rt, "BCSR", 4, 4)
    else:
        want = ref.convert(rt, fmt)
    assert_same_materialized(ctx.convert(d, fmt).download(), want.download(), ("s14", fmt))


def test_rmat14_vs_reference_hybrid(ctx, ref, rmat14):
    d, rt, _ = rmat14
    ell, coo = ctx.convert(d, "HYB(8)").parts()
    sel, rem, _ = ref.decompose_rows(rt, 8)
    assert_same_materialized(ell.download(), ref.convert(rem, "ELL").download(), "s14 HYB ELL")
    assert_same_materialized(coo.download(), ref.convert(sel, "COO").download(), "s14 HYB COO")


def test_uniform_s14_vs_reference_ell(ctx, port, ref):
    """ELL over every row (K = max row length) on a 16K x 16K, 16/row matrix
    (on R-MAT, K would be the heaviest row's ~5,000 slots)."""
    p = port.gen_uniform(1, 1 << S14, 1 << S14, 16)
    r, c, v = p.arrays()
    d = ctx.gen_uniform(1, 1 << S14, 1 << S14, 16)
    want = ref.convert(ref.from_coo(1 << S14, 1 << S14, r, c, v), "ELL")
    assert_same_materialized(ctx.convert(d, "ELL").download(), want.download(), "s14 ELL")


@pytest.mark.parametrize("fmt", ["CSR", "DCSR", "COO", "CSC", "HYB(8)", "BCSR(4,4)"])
def test_rmat14_vs_reference_spmv_spmm(ctx, port, ref, rmat14, fmt):
    d, rt, (r, c, v) = rmat14
    m = 1 << S14
    x = port.gen_dense(3, m)
    nd = 32
    b = port.gen_dense(4, m * nd).reshape(m, nd)
    a = ctx.convert(d, fmt)
    if fmt.startswith("HYB"):
        sel, rem, _ = ref.decompose_rows(rt, 8)
        e, co = ref.convert(rem, "ELL"), ref.convert(sel, "COO")
        y_ref = ref.spmv(e, x) + ref.spmv(co, x)
        c_ref = ref.spmm(e, b) + ref.spmm(co, b)
    else:
        mat = ref.convert(rt, "BCSR", 4, 4) if fmt.startswith("BCSR") else ref.convert(rt, fmt)
        y_ref, c_ref = ref.spmv(mat, x), ref.spmm(mat, b)
    absa = np.abs(v)
    ybound = np.bincount(r, weights=absa * np.abs(x[c]), minlength=m)
    check_close(ctx.spmv(a, x.astype(np.float32)), y_ref, ybound, ("s14 spmv", fmt))
    cbound = port.spmm(port.convert(port.from_coo(m, m, r, c, absa), "CSR"), np.abs(b))
    check_close(ctx.spmm(a, b.astype(np.float32)), c_ref, cbound, ("s14 spmm", fmt))
