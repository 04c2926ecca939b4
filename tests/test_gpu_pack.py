"""The value-layout formats: Pack(0,1) (operators.hpp:424-430) over COO (DOK,
formats.hpp:40) and CSR (LIL, formats.hpp:45). The device stores them as
records (AoS); downloaded, they equal the unmodified reference's
MaterializedTensor field for field, layout tag included (storage.hpp:128-133),
compute exactly what the unpacked formats compute, and round-trip through
the container byte-identically to the reference's write_container
(io.hpp:262-268)."""
import filecmp

import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL, assert_same_materialized, check_spmv, dense_abs_bound
from matrices import power_law_coo, random_coo

pytestmark = pytest.mark.gpu

CASES = [
    ("random", lambda: random_coo(0, 37, 29, 0.2, zeros=0.1)),
    ("power_law", lambda: power_law_coo(2, 3000, 2000, avg=9, alpha=1.3)),
    ("odd_nnz", lambda: random_coo(5, 5, 7, 0.5)),  # nnz not a multiple of 4
    ("one", lambda: ([3], [4], [2.5])),
]
SHAPES = {"random": (37, 29), "power_law": (3000, 2000), "odd_nnz": (5, 7), "one": (6, 9)}


def _mk(ctx, ref, case):
    r, c, v = dict(CASES)[case]()
    m, n = SHAPES[case]
    v = np.asarray(v, np.float32).astype(np.float64)
    return ctx.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v), (m, n, r, c, v)


@pytest.mark.parametrize("fmt", ["DOK", "LIL"])
@pytest.mark.parametrize("case", [c for c, _ in CASES])
def test_pack_matches_reference(ctx, ref, fmt, case):
    d, p, _ = _mk(ctx, ref, case)
    dev = ctx.convert(d, fmt)
    assert dev.kind == fmt
    got, want = dev.download(), ref.convert(p, fmt).download()
    assert want.layout == (0, 1) and got.layout == (0, 1), (got.layout, want.layout)
    assert_same_materialized(got, want, (fmt, case))
    assert got.explain() == want.explain() == sfg.storage_explain(fmt)


@pytest.mark.parametrize("fmt,base", [("DOK", "COO"), ("LIL", "CSR")])
def test_packed_compute_equals_unpacked(ctx, ref, fmt, base):
    """The records hold the same entries in the same order: SpMV / SpMM are
    bit-identical to the SoA format's, and within the tolerance of the
    reference on the packed tensor."""
    d, p, (m, n, r, c, v) = _mk(ctx, ref, "power_law")
    a, b = ctx.convert(d, fmt), ctx.convert(d, base)
    x = np.random.default_rng(1).uniform(-1, 1, n).astype(np.float32)
    ya, yb = ctx.spmv(a, x), ctx.spmv(b, x)
    np.testing.assert_array_equal(ya, yb)
    check_spmv(ya, ref.spmv(ref.convert(p, fmt), x.astype(np.float64)),
               dense_abs_bound(r, c, v, m, x.astype(np.float64)), fmt)
    for nd in (1, 32, 40):
        bm = np.random.default_rng(nd).uniform(-1, 1, (n, nd)).astype(np.float32)
        ca, cb = ctx.spmm(a, bm), ctx.spmm(b, bm)
        np.testing.assert_array_equal(ca, cb)
        cr = ref.spmm(ref.convert(p, fmt), bm.astype(np.float64))
        bound = np.zeros((m, nd))
        np.add.at(bound, np.asarray(r), np.abs(np.asarray(v))[:, None] * np.abs(bm.astype(np.float64)[np.asarray(c)]))
        assert np.all(np.abs(ca - cr) <= TOL * bound + 1e-30), (fmt, nd)


@pytest.mark.parametrize("fmt", ["DOK", "LIL"])
def test_packed_container_matches_reference(ctx, ref, tmp_path, fmt):
    d, p, (m, n, r, c, v) = _mk(ctx, ref, "random")
    dev = ctx.convert(d, fmt)
    ours, theirs = tmp_path / "ours.uspt", tmp_path / "ref.uspt"
    ctx.write_container(dev, str(ours))
    ref.write_container(p, fmt, str(theirs))
    assert filecmp.cmp(ours, theirs, shallow=False), fmt
    for f in (fmt, None):  # named, or inferred from the levels + the AoS tag
        back = ctx.read_container(str(theirs), f) if f else ctx.read_container(str(theirs))
        assert back.kind == fmt
        assert_same_materialized(back.download(), dev.download(), ("read", fmt))
        assert back.download().layout == (0, 1)


def test_packed_sources_are_rejected_like_the_reference(ctx, ref):
    """planner.hpp:98-99: conversion from a format with a value layout."""
    d, p, _ = _mk(ctx, ref, "random")
    for fmt in ("DOK", "LIL"):
        with pytest.raises(sfg.SfgError) as ei:
            ctx.convert(ctx.convert(d, fmt), "CSR")
        assert ei.value.kind == "UnsupportedSource"
        with pytest.raises(Exception) as er:
            ref.convert_from(p, fmt, "CSR")
        assert "value layout" in str(er.value) and "value layout" in str(ei.value)


def test_packed_spgemm(ctx):
    """SpGEMM takes packed operands (the layout is storage only)."""
    r, c, v = random_coo(3, 30, 40, 0.2)
    r2, c2, v2 = random_coo(4, 40, 20, 0.2)
    a, b = ctx.from_coo(30, 40, r, c, v), ctx.from_coo(40, 20, r2, c2, v2)
    want = ctx.spgemm(ctx.convert(a, "CSR"), ctx.convert(b, "CSR"))
    got = ctx.spgemm(ctx.convert(a, "DOK"), ctx.convert(b, "LIL"))
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-6)
