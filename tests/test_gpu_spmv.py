"""GPU parity: SpMV over every materialized format vs the f64 oracle walk
(run_kernel, kernel.hpp:236-384), within |y_hat - y| <= 1e-5 sum|a||x|."""
import numpy as np
import pytest

from gpu_common import check_spmv, dense_abs_bound
from matrices import EDGE_SHAPES, matrix_a, power_law_coo, random_coo

pytestmark = pytest.mark.gpu

ROW_FORMATS = ["COO", "CSR", "DCSR", "ELL"]


def run(ctx, port, fmt, m, n, r, c, v, x, ctxmsg):
    d = ctx.from_coo(m, n, r, c, v)
    p = port.from_coo(m, n, r, c, v)
    dm, pm = ctx.convert(d, fmt), port.convert(p, fmt)
    y = ctx.spmv(dm, x)
    yr = port.spmv(pm, x.astype(np.float64))
    check_spmv(y, yr, dense_abs_bound(r, c, v, m, x.astype(np.float64)), ctxmsg)
    return y


@pytest.mark.parametrize("fmt", ROW_FORMATS)
def test_matrix_a_ones(ctx, port, fmt):
    g = matrix_a()
    t = ctx.from_coo(g["rows"], g["cols"], g["coo_d0"], g["coo_d1"], g["coo_val"])
    y = ctx.spmv(ctx.convert(t, fmt), np.ones(4, np.float32))
    assert y.tolist() == g["spmv_y"]


@pytest.mark.parametrize("seed,shape", list(enumerate(EDGE_SHAPES)))
@pytest.mark.parametrize("fmt", ROW_FORMATS)
def test_random(ctx, port, fmt, seed, shape):
    m, n = shape
    r, c, v = random_coo(seed, m, n, 0.4, zeros=0.1)
    x = np.random.default_rng(seed).random(n).astype(np.float32)
    run(ctx, port, fmt, m, n, r, c, v, x, (fmt, m, n))


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("fmt", ROW_FORMATS)
def test_power_law(ctx, port, fmt, seed):
    m, n = 5000, 4000
    r, c, v = power_law_coo(seed, m, n, avg=20, alpha=1.2)
    x = (np.random.default_rng(seed).random(n) * 2 - 1).astype(np.float32)  # cancellation
    run(ctx, port, fmt, m, n, r, c, v, x, (fmt, seed))


@pytest.mark.parametrize("fmt", ROW_FORMATS)
def test_long_rows_and_chunk_boundaries(ctx, port, fmt):
    # rows spanning many warps' COO chunks and CSR lane groups
    m, n = 7, 200000
    rng = np.random.default_rng(1)
    rows, cols = [], []
    for i, L in enumerate([0, 1, 31, 33, 257, 70000, 3]):
        cols.append(np.sort(rng.choice(n, L, replace=False)))
        rows.append(np.full(L, i))
    r, c = np.concatenate(rows), np.concatenate(cols)
    v = (0.5 + rng.integers(0, 1 << 23, len(r)) / 2.0 ** 23).astype(np.float32)
    x = rng.random(n).astype(np.float32)
    run(ctx, port, fmt, m, n, r, c, v, x, fmt)


def test_accumulate_flag(ctx):
    import paper_2403_05802_b200 as sfg
    t = ctx.convert(ctx.from_coo(3, 3, [0, 1, 2], [0, 1, 2], [1.0, 2.0, 3.0]), "CSR")
    xb = ctx.buffer(12).upload(np.ones(3, np.float32))
    yb = ctx.buffer(12).upload(np.array([10, 20, 30], np.float32))
    ctx.spmv_device(t, xb.ptr, yb.ptr, accumulate=True)
    assert yb.download(np.float32, 3).tolist() == [11, 22, 33]


@pytest.mark.slow
def test_config1_full_size_spmv(ctx, port):
    m = n = 1 << 20
    d, p = ctx.gen_uniform(1, m, n, 16), port.gen_uniform(1, m, n, 16)
    x = port.gen_dense(2, n)
    y = ctx.spmv(ctx.convert(d, "CSR"), x.astype(np.float32))
    yr = port.spmv(port.convert(p, "CSR"), x)
    r, c, v = p.arrays()
    check_spmv(y, yr, dense_abs_bound(r, c, v, m, x), "cfg1")


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("t_min", [1, 4, 8, 10 ** 6])
def test_hybrid_spmv(ctx, port, seed, t_min):
    m, n = 6000, 5000
    r, c, v = power_law_coo(seed, m, n, avg=12, alpha=1.3)
    x = (np.random.default_rng(seed).random(n) * 2 - 1).astype(np.float32)
    d = ctx.from_coo(m, n, r, c, v)
    y = ctx.spmv(ctx.convert(d, f"HYB({t_min})"), x)
    p = port.from_coo(m, n, r, c, v)
    ps, pr, _ = port.decompose_rows(p, t_min)
    xd = x.astype(np.float64)
    yr = port.spmv(port.convert(pr, "ELL"), xd) + port.spmv(port.convert(ps, "COO"), xd)
    check_spmv(y, yr, dense_abs_bound(r, c, v, m, xd), ("HYB", t_min))


@pytest.mark.slow
def test_config2_full_size_hybrid_spmv(ctx, port):
    d, p = ctx.gen_rmat(7, 22, 16 << 22), port.gen_rmat(7, 22, 16 << 22)
    n = 1 << 22
    x = port.gen_dense(3, n)
    y = ctx.spmv(ctx.convert(d, "HYB(8)"), x.astype(np.float32))
    ps, pr, _ = port.decompose_rows(p, 8)
    yr = port.spmv(port.convert(pr, "ELL"), x) + port.spmv(port.convert(ps, "COO"), x)
    r, c, v = p.arrays()
    check_spmv(y, yr, dense_abs_bound(r, c, v, n, x), "cfg2 hybrid")
