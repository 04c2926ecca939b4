"""GPU parity: COO -> CSC and COO -> BCSR(r, c) (fp32 and bf16 values),
bit-exact against the oracle; SpMV over both within the 1e-5 bound."""
import numpy as np
import pytest

from gpu_common import assert_same_materialized, check_spmv, dense_abs_bound
from matrices import EDGE_SHAPES, matrix_a, power_law_coo, random_coo

pytestmark = pytest.mark.gpu

BLOCKS = [(2, 2), (3, 2), (4, 4), (16, 16), (1, 8), (8, 1)]
CASES = [(s, m, n, d, z) for s, (m, n) in enumerate(EDGE_SHAPES) for d, z in ((0.3, 0.0), (0.5, 0.2))]


def bf16_round(a):
    """Round-to-nearest-even to bf16, returned as f64."""
    f = np.asarray(a, np.float32).view(np.uint32).astype(np.uint64)
    rounded = ((f + 0x7FFF + ((f >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("seed,m,n,density,zeros", CASES)
def test_csc_bit_exact(ctx, port, seed, m, n, density, zeros):
    r, c, v = random_coo(seed, m, n, density, zeros)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    assert_same_materialized(ctx.convert(d, "CSC").download(), port.convert(p, "CSC").download(),
                             ("CSC", m, n))


@pytest.mark.parametrize("seed", range(3))
def test_csc_long_columns_general_path(ctx, port, seed):
    # transposed power law: long columns force the radix-sort path
    m, n = 3000, 2000
    r, c, v = power_law_coo(seed, n, m, avg=20, alpha=1.1)
    r, c = c, r
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    assert_same_materialized(ctx.convert(d, "CSC").download(), port.convert(p, "CSC").download(), "CSC")


@pytest.mark.parametrize("m,n,nnz", [(1 << 22, 1 << 22, 300_000), (5000, 70_000, 150_000), (100, 1500, 60_000)])
def test_csc_column_blocks(ctx, port, m, n, nnz):
    # the column-bucket partition path: buckets of w <= 8,192 columns (w not a
    # power of two: 7,086 for the first case, whose 592 buckets are rounded
    # up to whole waves of the SM count), each sorted in shared memory; the
    # last bucket is partial; (100, 1500, 60000) puts ~40 rows in a column
    # (dense short matrix)
    rng = np.random.default_rng(nnz)
    key = np.unique(rng.integers(0, m * n, nnz, dtype=np.int64))
    r, c = key // n, key % n
    v = (rng.random(len(key)) + 0.5).astype(np.float32)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    assert_same_materialized(ctx.convert(d, "CSC").download(), port.convert(p, "CSC").download(), ("CSC", m, n))


def test_csc_block_overflow_takes_histogram_path(ctx, port):
    # 15 entries in each of the first 2,000 columns plus scattered ones: the
    # first column bucket holds > 22,528 entries (more than one pass-2 CTA
    # sorts), so the conversion takes the per-column histogram path (short
    # columns, atomic cursors)
    m, n = 50_000, 100_000
    rng = np.random.default_rng(3)
    dense_r = np.concatenate([rng.choice(m, 15, replace=False) for _ in range(2000)])
    dense_c = np.repeat(np.arange(2000), 15)
    key = np.unique(np.concatenate([dense_r * n + dense_c, rng.integers(0, m * n, 1000, dtype=np.int64)]))
    r, c = key // n, key % n
    assert np.bincount(c).max() <= 32 and np.count_nonzero(c < 7693) > 22_528
    v = (rng.random(len(key)) + 0.5).astype(np.float32)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    assert_same_materialized(ctx.convert(d, "CSC").download(), port.convert(p, "CSC").download(), "CSC")


def test_csc_matrix_a(ctx):
    g = matrix_a()
    t = ctx.from_coo(g["rows"], g["cols"], g["coo_d0"], g["coo_d1"], g["coo_val"])
    a = ctx.convert(t, "CSC").download()
    assert a.levels[1].ptr.tolist() == [0, 1, 3, 4, 6]
    assert a.levels[1].idx.tolist() == [0, 1, 2, 2, 2, 4]


@pytest.mark.parametrize("rc", BLOCKS)
@pytest.mark.parametrize("seed,m,n,density,zeros", CASES)
def test_bcsr_bit_exact(ctx, port, rc, seed, m, n, density, zeros):
    r, c, v = random_coo(seed, m, n, density, zeros)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    fmt = f"BCSR({rc[0]},{rc[1]})"
    assert_same_materialized(ctx.convert(d, fmt).download(),
                             port.convert(p, "BCSR", *rc).download(), (fmt, m, n))


def test_bcsr_goldens(ctx):
    g = matrix_a()
    t = ctx.from_coo(g["rows"], g["cols"], g["coo_d0"], g["coo_d1"], g["coo_val"])
    b = ctx.convert(t, "BCSR(2,2)").download()
    assert b.levels[1].ptr.tolist() == g["bcsr_ptr"]
    assert b.levels[1].idx.tolist() == g["bcsr_idx"]
    assert b.values.tolist() == g["bcsr_val"]
    assert b.explain() == g["storage_explain"]["BCSR"]
    e = ctx.from_coo(3, 3, [0, 2, 2], [0, 0, 2], [1.0, 2.0, 3.0])
    b = ctx.convert(e, "BCSR(2,2)").download()  # SURVEY §9 edge blocks
    assert b.levels[1].ptr.tolist() == [0, 1, 3]
    assert b.values.tolist() == [1, 0, 0, 0, 2, 0, 0, 0, 3, 0, 0, 0]


@pytest.mark.parametrize("rc", [(4, 4), (16, 16)])
def test_bcsr_bf16_values(ctx, port, rc):
    import paper_2403_05802_b200 as sfg
    m, n = 200, 300
    r, c, v = random_coo(3, m, n, 0.2)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    dev = ctx.convert(d, f"BCSR({rc[0]},{rc[1]})", value_dtype=sfg.BF16).download()
    ora = port.convert(p, "BCSR", *rc).download()
    ora.values = bf16_round(ora.values)
    assert_same_materialized(dev, ora, "bf16")


@pytest.mark.parametrize("fmt", ["CSC", "BCSR(2,2)", "BCSR(4,4)", "BCSR(16,16)", "BCSR(3,5)"])
@pytest.mark.parametrize("seed,shape", list(enumerate([(1, 1), (17, 33), (64, 64), (300, 257)])))
def test_spmv_csc_bcsr(ctx, port, fmt, seed, shape):
    m, n = shape
    r, c, v = random_coo(seed, m, n, 0.3, zeros=0.1)
    x = (np.random.default_rng(seed).random(n) * 2 - 1).astype(np.float32)
    d, p = ctx.from_coo(m, n, r, c, v), port.from_coo(m, n, r, c, v)
    if fmt == "CSC":
        pm = port.convert(p, "CSC")
    else:
        rr, cc = (int(t) for t in fmt[5:-1].split(","))
        pm = port.convert(p, "BCSR", rr, cc)
    y = ctx.spmv(ctx.convert(d, fmt), x)
    yr = port.spmv(pm, x.astype(np.float64))
    check_spmv(y, yr, dense_abs_bound(r, c, v, m, x.astype(np.float64)), fmt)


@pytest.mark.slow
def test_bcsr_conversion_throughput_scale(ctx, port):
    """Config-4 style block-sparse input at 4096^2, 10% blocks (CPU-checkable)."""
    rng = np.random.default_rng(4)
    for r_, c_ in [(4, 4), (16, 16)]:
        nb = 4096 // r_
        mask = rng.random((nb, nb)) < 0.1
        br, bc = np.nonzero(mask)
        ii, jj = np.meshgrid(np.arange(r_), np.arange(c_), indexing="ij")
        rows = (br[:, None] * r_ + ii.ravel()[None, :]).ravel()
        cols = (bc[:, None] * c_ + jj.ravel()[None, :]).ravel()
        vals = (0.5 + rng.integers(0, 1 << 23, rows.size) / 2.0 ** 23).astype(np.float32)
        d, p = ctx.from_coo(4096, 4096, rows, cols, vals), port.from_coo(4096, 4096, rows, cols, vals)
        assert_same_materialized(ctx.convert(d, f"BCSR({r_},{c_})").download(),
                                 port.convert(p, "BCSR", r_, c_).download(), (r_, c_))


@pytest.mark.parametrize("rc", [(4, 4), (16, 16), (3, 5)])
@pytest.mark.parametrize("shape", [(512, 512), (100, 77)])
def test_block_sparse_generator_equals_conversion(ctx, port, rc, shape):
    """Config-4 input generated directly as BCSR == convert(COO expansion)."""
    import paper_2403_05802_b200 as sfg
    m, n = shape
    d = ctx.gen_block_sparse(9, m, n, rc[0], rc[1], 0.1).download()
    p = port.gen_block_sparse(9, m, n, rc[0], rc[1], 0.1)
    assert_same_materialized(d, port.convert(p, "BCSR", *rc).download(), (rc, shape))
    db = ctx.gen_block_sparse(9, m, n, rc[0], rc[1], 0.1, value_dtype=sfg.BF16).download()
    ora = port.convert(p, "BCSR", *rc).download()
    ora.values = bf16_round(ora.values)
    assert_same_materialized(db, ora, "bf16")
