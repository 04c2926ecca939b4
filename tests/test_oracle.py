"""Pins the CPU oracle (tests/ only, no GPU).

1. Both the reference shim (oracle/_ref, the unmodified headers) and the C
   restatement (oracle/sfo.c) reproduce the reference's frozen golden
   vectors for matrix A (proj/tests/oracle_data.hpp via tests/golden).
2. The restatement equals the reference bit-for-bit on seeded random
   matrices: every level array, bound, node count and value, and the f64
   SpMV/SpMM outputs (same accumulation order).
"""
import numpy as np
import pytest

import oracle
from matrices import EDGE_SHAPES, matrix_a, power_law_coo, random_coo

FMTS = [("COO", 0, 0), ("CSR", 0, 0), ("CSC", 0, 0), ("DCSR", 0, 0), ("ELL", 0, 0),
        ("BCSR", 2, 2), ("BCSR", 3, 2), ("BCSR", 4, 4), ("BCSR", 16, 16)]


def impls(port, ref):
    return [("port", port), ("ref", ref)]


def a_coo(lib, shuffled=False):
    g = matrix_a()
    r, c, v = (np.array(g[k]) for k in ("coo_d0", "coo_d1", "coo_val"))
    if shuffled:  # FromCooSortsInput, test_tensor.cpp:47-54
        p = np.array([5, 0, 4, 3, 1, 2])
        r, c, v = r[p], c[p], v[p]
    return lib.from_coo(g["rows"], g["cols"], r, c, v)


@pytest.mark.parametrize("which", ["port", "ref"])
def test_matrix_a_goldens(port, ref, which):
    lib = port if which == "port" else ref
    g = matrix_a()
    t = a_coo(lib, shuffled=True)
    r, c, v = t.arrays()
    assert r.tolist() == g["coo_d0"] and c.tolist() == g["coo_d1"] and v.tolist() == g["coo_val"]

    csr = lib.convert(t, "CSR").download()
    assert csr.levels[1].ptr.tolist() == g["csr_ptr"]
    assert csr.levels[1].idx.tolist() == g["csr_idx"]
    assert csr.values.tolist() == g["csr_val"]
    assert csr.explain() == g["storage_explain"]["CSR"]

    ell = lib.convert(t, "ELL").download()
    assert ell.levels[0].idx.tolist() == [0, 1, 2]
    assert ell.levels[2].idx.tolist() == g["ell_idx"]
    assert ell.values.tolist() == g["ell_val"]
    assert ell.explain() == g["storage_explain"]["ELL"]

    bcsr = lib.convert(t, "BCSR", 2, 2).download()
    assert bcsr.levels[1].ptr.tolist() == g["bcsr_ptr"]
    assert bcsr.levels[1].idx.tolist() == g["bcsr_idx"]
    assert bcsr.values.tolist() == g["bcsr_val"]
    assert bcsr.explain() == g["storage_explain"]["BCSR"]

    for fmt, rr, cc in FMTS:
        m = lib.convert(t, fmt, rr, cc)
        assert lib.spmv(m, np.ones(4)).tolist() == g["spmv_y"], fmt

    _, _, totals = lib.decompose_rows(t, 1)
    assert totals.tolist() == g["row_nnz"]


@pytest.mark.parametrize("which", ["port", "ref"])
def test_survey_live_outputs(port, ref, which):
    """SURVEY.md §9 live materialize outputs (CSC, DCSR, explicit zero, 3x3 edge)."""
    lib = port if which == "port" else ref
    t = a_coo(lib)
    csc = lib.convert(t, "CSC").download()
    assert csc.levels[1].ptr.tolist() == [0, 1, 3, 4, 6]
    assert csc.levels[1].idx.tolist() == [0, 1, 2, 2, 2, 4]
    assert csc.values.tolist() == [1, 2, 3, 4, 5, 6]
    dcsr = lib.convert(t, "DCSR").download()
    assert dcsr.levels[0].idx.tolist() == [0, 1, 2, 4]
    assert dcsr.levels[1].ptr.tolist() == [0, 1, 2, 5, 6]
    # explicit zero stays in CSR, moves to the trailing ELL slot
    z = lib.from_coo(2, 3, [0, 0, 0, 1], [0, 1, 2, 1], [1.0, 0.0, 3.0, 5.0])
    assert lib.convert(z, "CSR").download().values.tolist() == [1, 0, 3, 5]
    ell = lib.convert(z, "ELL").download()
    assert ell.levels[2].idx.tolist() == [0, 1, 2, 0, 1, 0]
    assert ell.values.tolist() == [1, 5, 3, 0, 0, 0]
    e = lib.from_coo(3, 3, [0, 2, 2], [0, 0, 2], [1.0, 2.0, 3.0])
    b = lib.convert(e, "BCSR", 2, 2).download()
    assert b.levels[1].ptr.tolist() == [0, 1, 3]
    assert b.levels[1].idx.tolist() == [0, 0, 1]
    assert b.values.tolist() == [1, 0, 0, 0, 2, 0, 0, 0, 3, 0, 0, 0]
    # empty input
    emp = lib.from_coo(4, 4, [], [], [])
    assert lib.convert(emp, "ELL").download().values.size == 0
    assert lib.convert(emp, "DCSR").download().levels[1].ptr.tolist() == [0]


@pytest.mark.parametrize("which", ["port", "ref"])
def test_from_coo_errors_and_duplicates(port, ref, which):
    lib = port if which == "port" else ref
    with pytest.raises(oracle.OracleError) as ei:
        lib.from_coo(3, 3, [1, 1], [2, 2], [5.0, 7.0])
    assert ei.value.kind == "DuplicateCoordinate"
    t = lib.from_coo(3, 3, [1, 0, 1], [2, 0, 2], [5.0, 1.0, 7.0], sum_duplicates=True)
    assert t.arrays()[2].tolist() == [1.0, 12.0]
    with pytest.raises(oracle.OracleError) as ei:
        lib.from_coo(3, 3, [3], [0], [1.0])
    assert ei.value.kind == "InvalidOperation"


def levels_equal(a, b, ctx):
    assert len(a.levels) == len(b.levels), ctx
    for i, (la, lb) in enumerate(zip(a.levels, b.levels)):
        assert (la.flags, la.lo, la.hi, la.node_count) == (lb.flags, lb.lo, lb.hi, lb.node_count), (ctx, i)
        np.testing.assert_array_equal(la.idx, lb.idx, err_msg=f"{ctx} L{i} idx")
        np.testing.assert_array_equal(la.ptr, lb.ptr, err_msg=f"{ctx} L{i} ptr")
    np.testing.assert_array_equal(a.values, b.values, err_msg=f"{ctx} values")


CASES = [(s, m, n, d, z) for s, (m, n) in enumerate(EDGE_SHAPES) for d, z in ((0.3, 0.0), (0.5, 0.2))]


@pytest.mark.parametrize("seed,m,n,density,zeros", CASES)
def test_port_matches_reference(port, ref, seed, m, n, density, zeros):
    r, c, v = random_coo(seed, m, n, density, zeros)
    tp, tr = port.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v)
    for x, y in zip(tp.arrays(), tr.arrays()):
        np.testing.assert_array_equal(x, y)
    rng = np.random.default_rng(seed)
    x = rng.random(n)
    b = rng.random((n, 3))
    for fmt, rr, cc in FMTS:
        mp, mr = port.convert(tp, fmt, rr, cc), ref.convert(tr, fmt, rr, cc)
        levels_equal(mp.download(), mr.download(), (fmt, rr, cc, m, n))
        np.testing.assert_array_equal(port.spmv(mp, x), ref.spmv(mr, x))
        np.testing.assert_array_equal(port.spmm(mp, b), ref.spmm(mr, b))


@pytest.mark.parametrize("seed", range(4))
def test_port_matches_reference_power_law(port, ref, seed):
    m, n = 60, 50
    r, c, v = power_law_coo(seed, m, n)
    tp, tr = port.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v)
    for fmt, rr, cc in FMTS:
        levels_equal(port.convert(tp, fmt, rr, cc).download(),
                     ref.convert(tr, fmt, rr, cc).download(), fmt)
    for t_min in (0, 1, 2, 4, 8, 1000):
        sp, rp, tot_p = port.decompose_rows(tp, t_min)
        sr, rr_, tot_r = ref.decompose_rows(tr, t_min)
        np.testing.assert_array_equal(tot_p, tot_r)
        for a, b in zip(sp.arrays() + rp.arrays(), sr.arrays() + rr_.arrays()):
            np.testing.assert_array_equal(a, b)
        # hybrid: ELL of the remainder + COO of the selection
        x = np.random.default_rng(seed).random(n)
        yp = port.spmv(port.convert(rp, "ELL"), x) + port.spmv(port.convert(sp, "COO"), x)
        yr = ref.spmv(ref.convert(rr_, "ELL"), x) + ref.spmv(ref.convert(sr, "COO"), x)
        np.testing.assert_array_equal(yp, yr)


def test_sum_duplicates_matches_reference(port, ref):
    r, c, v = random_coo(7, 20, 20, 0.3, dups=25)
    a, b = port.from_coo(20, 20, r, c, v, True), ref.from_coo(20, 20, r, c, v, True)
    for x, y in zip(a.arrays(), b.arrays()):
        np.testing.assert_array_equal(x, y)


def test_reference_plans(ref):
    """The host dispatch table straight from plan_conversion."""
    g = matrix_a()
    assert ref.plan("COO", "CSR") == g["plan_coo_to_csr"]
    assert ref.plan("COO", "COO") == []
    assert ref.plan("COO", "DCSR") == ["Merge(0)"]
    assert ref.plan("COO", "CSC") == ["Swap(0,1)", "Sort", "Fill(0)", "Merge(0)"]
    assert ref.plan("COO", "BCSR(4,4)") == [
        "TileSplit(0,4)", "TileSplit(2,4)", "Swap(1,2)", "Sort", "Fill(3)", "Fill(2)", "Fill(0)",
        "Vectorize(2)", "Merge(0)"]
    assert ref.plan("COO", "ELL") == ["Sum(0)", "Enumerate(0)", "Sort", "Fill(1)", "Merge(0)"]
    for k, want in g["storage_explain"].items():
        assert ref.explain(k) == want


def test_generators_are_canonical(port):
    t = port.gen_uniform(1, 64, 1 << 12, 16)
    r, c, v = t.arrays()
    assert len(r) == 64 * 16
    assert np.all(np.diff(r * (1 << 12) + c) > 0)
    assert np.all(v != 0) and np.all(np.abs(v) >= 0.5) and np.all(np.abs(v) < 1.5)
    g = port.gen_rmat(7, 10, 1 << 14)
    r, c, v = g.arrays()
    assert np.all(np.diff(r * (1 << 10) + c) > 0)
    assert np.bincount(r, minlength=1 << 10)[0] > np.bincount(r, minlength=1 << 10)[-1]
    x = port.gen_dense(3, 1000)
    assert np.all(x > 0) and np.all(x <= 1) and np.all(x.astype(np.float32) == x)
