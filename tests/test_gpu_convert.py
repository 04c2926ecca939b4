"""GPU parity: from_coo and the COO -> {COO, CSR, DCSR, CSC, ELL, BCSR}
conversions through the C-ABI, bit-exact against the CPU oracle (which is
itself pinned to the reference, tests/test_oracle.py)."""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import assert_same_materialized
from matrices import EDGE_SHAPES, matrix_a, power_law_coo, random_coo

pytestmark = pytest.mark.gpu

ROW_FORMATS = ["COO", "CSR", "DCSR", "ELL"]


def dev_and_port(ctx, port, m, n, r, c, v, sorted_input=False, sum_dups=False):
    d = ctx.from_coo(m, n, r, c, v, sorted=sorted_input, sum_duplicates=sum_dups)
    p = port.from_coo(m, n, r, c, v, sum_duplicates=sum_dups)
    return d, p


def test_matrix_a_from_shuffled_coo(ctx, port):
    g = matrix_a()
    p = np.array([5, 0, 4, 3, 1, 2])  # FromCooSortsInput, test_tensor.cpp:47-54
    r, c, v = (np.array(g[k])[p] for k in ("coo_d0", "coo_d1", "coo_val"))
    t = ctx.from_coo(g["rows"], g["cols"], r, c, v)
    rr, cc, vv = t.coo_arrays()
    assert rr.tolist() == g["coo_d0"] and cc.tolist() == g["coo_d1"] and vv.tolist() == g["coo_val"]
    csr = ctx.convert(t, "CSR").download()
    assert csr.levels[1].ptr.tolist() == g["csr_ptr"]
    assert csr.levels[1].idx.tolist() == g["csr_idx"]
    assert csr.values.tolist() == g["csr_val"]
    assert csr.explain() == g["storage_explain"]["CSR"]


def test_from_coo_errors(ctx):
    with pytest.raises(sfg.SfgError) as ei:
        ctx.from_coo(3, 3, [1, 1], [2, 2], [5.0, 7.0])
    assert ei.value.kind == "DuplicateCoordinate"
    with pytest.raises(sfg.SfgError) as ei:
        ctx.from_coo(3, 3, [3], [0], [1.0])
    assert ei.value.kind == "InvalidOperation"
    with pytest.raises(sfg.SfgError) as ei:
        ctx.from_coo(3, 3, [0, 1, 1], [0, 2, 2], [1.0, 2.0, 3.0], sorted=True)
    assert ei.value.kind == "DuplicateCoordinate"
    t = ctx.from_coo(3, 3, [1, 0, 1], [2, 0, 2], [5.0, 1.0, 7.0], sum_duplicates=True)
    assert t.coo_arrays()[2].tolist() == [1.0, 12.0]
    # the offending entry sits in a lane other than 0 of its warp
    rows = np.arange(40) % 5
    rows[37] = 9
    for sorted_input in (False, True):
        with pytest.raises(sfg.SfgError) as ei:
            ctx.from_coo(5, 40, rows if not sorted_input else np.sort(rows), np.arange(40), np.ones(40),
                         sorted=sorted_input)
        assert ei.value.kind == "InvalidOperation"


def test_from_coo_names_smallest_duplicate(ctx):
    # the reference walks the sorted entries and throws at the first repeat
    # (tensor.hpp:147-153): the smallest duplicated coordinate, wherever the
    # copies sit in the unsorted input and however many tiles the sort spans
    rng = np.random.default_rng(5)
    m = n = 4096
    keys = rng.choice(m * n, size=200_000, replace=False)
    r, c = (keys // n).astype(np.int32), (keys % n).astype(np.int32)
    order = np.argsort(keys)
    big, small = order[-1], order[1000]
    r2, c2 = np.append(r, [r[big], r[small]]), np.append(c, [c[big], c[small]])
    perm = rng.permutation(r2.size)
    with pytest.raises(sfg.SfgError) as ei:
        ctx.from_coo(m, n, r2[perm], c2[perm], np.ones(r2.size, np.float32))
    assert ei.value.kind == "DuplicateCoordinate"
    assert f"({r[small]},{c[small]})" in str(ei.value)


@pytest.mark.parametrize("seed", range(6))
def test_from_coo_sort_and_sum_duplicates(ctx, port, seed):
    m, n = [(1, 1), (17, 33), (300, 7), (64, 64), (1000, 999), (5, 4)][seed]
    r, c, v = random_coo(seed, m, n, 0.3, dups=(seed * 7) % 23)
    d, p = dev_and_port(ctx, port, m, n, r, c, v, sum_dups=True)
    # duplicates are summed in f64 like the reference (tensor.hpp:154) and
    # rounded once to fp32: equal to the oracle's f64 sums narrowed to fp32
    for a, b in zip(d.coo_arrays(), p.arrays()):
        np.testing.assert_array_equal(a, b.astype(a.dtype))


def test_from_coo_large_unsorted(ctx, port):
    rng = np.random.default_rng(5)
    m, n = 70000, 3 << 20
    k = 400000
    r = rng.integers(0, m, k)
    c = rng.integers(0, n, k)
    key = np.unique(r.astype(np.int64) * n + c)
    key = rng.permutation(key)
    r, c = key // n, key % n
    v = (0.5 + rng.integers(0, 1 << 23, len(key)) / 2.0 ** 23).astype(np.float32)
    d, p = dev_and_port(ctx, port, m, n, r, c, v)
    for a, b in zip(d.coo_arrays(), p.arrays()):
        np.testing.assert_array_equal(a.astype(np.float64), b)


CASES = [(s, m, n, d, z) for s, (m, n) in enumerate(EDGE_SHAPES) for d, z in ((0.3, 0.0), (0.5, 0.2))]


@pytest.mark.parametrize("seed,m,n,density,zeros", CASES)
@pytest.mark.parametrize("fmt", ROW_FORMATS)
def test_row_formats_bit_exact(ctx, port, fmt, seed, m, n, density, zeros):
    r, c, v = random_coo(seed, m, n, density, zeros)
    d, p = dev_and_port(ctx, port, m, n, r, c, v)
    assert_same_materialized(ctx.convert(d, fmt).download(), port.convert(p, fmt).download(),
                             (fmt, m, n))


@pytest.mark.parametrize("fmt", ROW_FORMATS)
def test_empty_and_sparse_rows(ctx, port, fmt):
    # empty matrix, one entry at the last row (long empty-row gap), one row
    for m, n, r, c in [(4, 4, [], []), (100000, 5, [99999], [4]), (1, 9, [0, 0], [2, 8]),
                       (70000, 70000, [0, 69999], [0, 69999])]:
        v = np.ones(len(r))
        d, p = dev_and_port(ctx, port, m, n, r, c, v)
        assert_same_materialized(ctx.convert(d, fmt).download(), port.convert(p, fmt).download(),
                                 (fmt, m, n))


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("fmt", ROW_FORMATS)
def test_power_law_rows(ctx, port, fmt, seed):
    m, n = 3000, 2500
    r, c, v = power_law_coo(seed, m, n, avg=12)
    d, p = dev_and_port(ctx, port, m, n, r, c, v, sorted_input=True)
    assert_same_materialized(ctx.convert(d, fmt).download(), port.convert(p, fmt).download(), fmt)


def test_generators_match_oracle(ctx, port):
    d = ctx.gen_uniform(3, 4096, 1 << 16, 16)
    p = port.gen_uniform(3, 4096, 1 << 16, 16)
    for a, b in zip(d.coo_arrays(), p.arrays()):
        np.testing.assert_array_equal(a.astype(np.float64), b)
    d = ctx.gen_rmat(7, 12, 1 << 16)
    p = port.gen_rmat(7, 12, 1 << 16)
    for a, b in zip(d.coo_arrays(), p.arrays()):
        np.testing.assert_array_equal(a.astype(np.float64), b)
    d = ctx.gen_hypersparse(9, 1 << 15, 1 << 15, 1 << 14)
    p = port.gen_hypersparse(9, 1 << 15, 1 << 15, 1 << 14)
    for a, b in zip(d.coo_arrays(), p.arrays()):
        np.testing.assert_array_equal(a.astype(np.float64), b)
    buf = ctx.buffer(4 * 1000)
    ctx.gen_dense(11, 1000, buf.ptr)
    np.testing.assert_array_equal(buf.download(np.float32, 1000).astype(np.float64),
                                  port.gen_dense(11, 1000))


@pytest.mark.slow
def test_config1_full_size_csr(ctx, port):
    """BASELINE config 1 at full size: 2^20 x 2^20, 16/row, bit-exact CSR."""
    m = n = 1 << 20
    d = ctx.gen_uniform(1, m, n, 16)
    p = port.gen_uniform(1, m, n, 16)
    assert_same_materialized(ctx.convert(d, "CSR").download(), port.convert(p, "CSR").download(),
                             "cfg1 CSR")


@pytest.mark.parametrize("seed,m,n,density,zeros", CASES)
@pytest.mark.parametrize("t_min", [0, 1, 2, 4, 1000])
def test_decompose_rows(ctx, port, seed, m, n, density, zeros, t_min):
    r, c, v = random_coo(seed, m, n, density, zeros)
    d, p = dev_and_port(ctx, port, m, n, r, c, v)
    ds, dr = ctx.decompose_rows(d, t_min)
    ps, pr, _ = port.decompose_rows(p, t_min)
    for a, b in zip(ds.coo_arrays() + dr.coo_arrays(), ps.arrays() + pr.arrays()):
        np.testing.assert_array_equal(a.astype(np.float64), b)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("t_min", [1, 3, 8, 50])
def test_hybrid_parts_bit_exact(ctx, port, seed, t_min):
    m, n = 4000, 3000
    r, c, v = power_law_coo(seed, m, n, avg=10)
    if seed % 2:  # explicit zeros (SURVEY §8c trap 1)
        v = v.copy()
        v[::7] = 0.0
    d, p = dev_and_port(ctx, port, m, n, r, c, v, sorted_input=True)
    h = ctx.convert(d, f"HYB({t_min})")
    ell, coo = h.parts()
    ps, pr, _ = port.decompose_rows(p, t_min)
    assert_same_materialized(ell.download(), port.convert(pr, "ELL").download(), ("ELL", t_min))
    assert_same_materialized(coo.download(), port.convert(ps, "COO").download(), ("COO", t_min))


def test_ell_explicit_zero_slots(ctx, port):
    # explicit zero at (0,1) moves to the trailing ELL slot
    d = ctx.from_coo(2, 3, [0, 0, 0, 1], [0, 1, 2, 1], [1.0, 0.0, 3.0, 5.0])
    e = ctx.convert(d, "ELL").download()
    assert e.levels[2].idx.tolist() == [0, 1, 2, 0, 1, 0]
    assert e.values.tolist() == [1, 5, 3, 0, 0, 0]
    g = matrix_a()
    t = ctx.from_coo(g["rows"], g["cols"], g["coo_d0"], g["coo_d1"], g["coo_val"])
    e = ctx.convert(t, "ELL").download()
    assert e.levels[2].idx.tolist() == g["ell_idx"] and e.values.tolist() == g["ell_val"]
    assert e.explain() == g["storage_explain"]["ELL"]


@pytest.mark.slow
def test_config2_full_size_hybrid(ctx, port):
    """BASELINE config 2 at full size: R-MAT s22 ef16, hybrid T=8, bit-exact."""
    d, p = ctx.gen_rmat(7, 22, 16 << 22), port.gen_rmat(7, 22, 16 << 22)
    for a, b in zip(d.coo_arrays(), p.arrays()):
        np.testing.assert_array_equal(a.astype(np.float64), b)
    h = ctx.convert(d, "HYB(8)")
    ell, coo = h.parts()
    ps, pr, _ = port.decompose_rows(p, 8)
    assert_same_materialized(ell.download(), port.convert(pr, "ELL").download(), "cfg2 ELL")
    assert_same_materialized(coo.download(), port.convert(ps, "COO").download(), "cfg2 COO")


def test_block_cache_reuse_and_release(ctx, port):
    """Freed tensor arrays are cached by the context and reused by the next
    conversion; release_cached hands them back to the driver pool."""
    ctx.release_cached()
    d = ctx.gen_rmat(3, 12, 16 << 12)
    ref = ctx.convert(d, "HYB(4)")
    want = [p.download() for p in ref.parts()]
    del ref
    cached = ctx.release_cached()
    assert cached > 0 and ctx.release_cached() == 0
    for _ in range(3):  # the reused blocks give the same result
        h = ctx.convert(d, "HYB(4)")
        for a, b in zip((p.download() for p in h.parts()), want):
            assert_same_materialized(a, b, "reuse")
        del h


def test_int32_index_range_is_enforced(ctx):
    # SURVEY §8c trap (7): extents or nnz past the int32 index range raise
    # InvalidOperation before anything is allocated or read
    for m, n in ((1 << 31, 8), (8, 1 << 31)):
        with pytest.raises(sfg.SfgError) as ei:
            ctx.from_coo(m, n, [0], [0], [1.0])
        assert ei.value.kind == "InvalidOperation"
    with pytest.raises(sfg.SfgError) as ei:
        ctx.from_coo_device(8, 8, 1 << 31, 0, 0, 0)  # never dereferenced
    assert ei.value.kind == "InvalidOperation"
