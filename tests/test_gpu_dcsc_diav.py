"""DCSC (formats.hpp:43: (d1, d0); merge(0), trim(0,1)) and DIA-variant
(formats.hpp:47-48: (d1-d0, d1); merge(0), trim(0,0)): the device
conversions are bit-exact with the unmodified reference's materialized
tensors (DCSC: the nonempty columns, then the rows of each; DIA-variant:
the diagonals over a zero-filled column panel), SpMV / SpMM agree within
the tolerance, DCSC is a conversion source like CSC, and the container
bytes equal the reference's."""
import filecmp

import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL, assert_same_materialized, check_spmv, dense_abs_bound
from test_gpu_dia_csb import CASES, _pair

pytestmark = pytest.mark.gpu

FMTS = ["DCSC", "DIA-variant"]


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("case", list(CASES))
def test_matches_reference(ctx, ref, fmt, case):
    d, p, _ = _pair(ctx, ref, case)
    got = ctx.convert(d, fmt).download()
    want = ref.convert(p, fmt).download()
    assert_same_materialized(got, want, (fmt, case))
    assert got.explain() == want.explain() == sfg.storage_explain(fmt)


@pytest.mark.parametrize("fmt", FMTS)
def test_compute(ctx, ref, fmt):
    d, p, (m, n, r, c, v) = _pair(ctx, ref, "banded")
    a = ctx.convert(d, fmt)
    ra = ref.convert(p, fmt)
    x = np.random.default_rng(0).uniform(-1, 1, n).astype(np.float32)
    check_spmv(ctx.spmv(a, x), ref.spmv(ra, x.astype(np.float64)), dense_abs_bound(r, c, v, m, x.astype(np.float64)),
               fmt)
    for nd in (1, 32, 128, 9):
        b = np.random.default_rng(nd).uniform(-1, 1, (n, nd)).astype(np.float32)
        got, want = ctx.spmm(a, b), ref.spmm(ra, b.astype(np.float64))
        bound = np.zeros((m, nd))
        np.add.at(bound, r, np.abs(v)[:, None] * np.abs(b.astype(np.float64)[c]))
        assert np.all(np.abs(got - want) <= TOL * bound + 1e-30), (fmt, nd)


@pytest.mark.parametrize("dst", ["COO", "CSR", "CSC", "DCSR", "DCSC", "ELL", "BCSR(2,2)", "DIA"])
@pytest.mark.parametrize("case", ["random", "banded", "tall", "wide"])
def test_dcsc_as_source(ctx, ref, dst, case):
    """planner.hpp:95-252 from DCSC: Split(0) Swap(0,1) [Sort] + the target's
    ops (to CSC: Fill(0))."""
    d, p, _ = _pair(ctx, ref, case)
    f, a, b = (dst, 0, 0) if not dst.startswith("BCSR") else ("BCSR", 2, 2)
    got = ctx.convert(ctx.convert(d, "DCSC"), dst).download()
    want = ref.convert_from(p, "DCSC", f, a, b).download()
    assert_same_materialized(got, want, (dst, case))


def test_dia_variant_not_a_conversion_source(ctx, ref):
    d, _, _ = _pair(ctx, ref, "random")
    with pytest.raises(sfg.SfgError) as ei:
        ctx.convert(ctx.convert(d, "DIA-variant"), "CSR")
    assert ei.value.kind == "UnsupportedSource"


@pytest.mark.parametrize("fmt", FMTS)
def test_container_matches_reference(ctx, ref, tmp_path, fmt):
    d, p, _ = _pair(ctx, ref, "random")
    dev = ctx.convert(d, fmt)
    ours, theirs = tmp_path / "ours.uspt", tmp_path / "ref.uspt"
    ctx.write_container(dev, str(ours))
    ref.write_container(p, fmt, str(theirs))
    assert filecmp.cmp(ours, theirs, shallow=False), fmt
    back = ctx.read_container(str(theirs), fmt)
    assert_same_materialized(back.download(), dev.download(), ("read", fmt))


@pytest.mark.parametrize("src", ["CSR", "DCSR", "BCSR(2,2)"])
@pytest.mark.parametrize("case", ["random", "banded", "wide"])
def test_dia_variant_from_sources(ctx, ref, src, case):
    d, p, _ = _pair(ctx, ref, case)
    s, a, b = (src, 0, 0) if not src.startswith("BCSR") else ("BCSR", 2, 2)
    got = ctx.convert(ctx.convert(d, src), "DIA-variant").download()
    want = ref.convert_from(p, s, "DIA-variant", 0, 0, a, b).download()
    assert_same_materialized(got, want, (src, case))


@pytest.mark.parametrize("src", ["CSC", "DCSC"])
def test_dia_variant_from_column_major_rejected(ctx, ref, src):
    """The reference's plan from a column-major source (Skew(1,0,-1)
    Skew(0,1,1)) widens the column level to [-(m-1), n+m-2]; the device
    does not model that panel and says so."""
    d, p, (m, n, _, _, _) = _pair(ctx, ref, "random")
    with pytest.raises(sfg.SfgError) as ei:
        ctx.convert(ctx.convert(d, src), "DIA-variant")
    assert ei.value.kind == "UnsupportedSource"
    want = ref.convert_from(p, src, "DIA-variant").download()
    assert (want.levels[1].lo, want.levels[1].hi) == (-(m - 1), n + m - 2)
