"""Blocked ELL, BELL(b) (formats.hpp:79-85): the
device conversion from canonical COO is bit-exact with the unmodified
reference's materialized tensor (slot-major cells, zero-padded slots and
edge blocks), SpMV / SpMM walk every stored slot like run_kernel and agree
within the tolerance, and the container round-trips byte-identically."""
import filecmp

import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL, assert_same_materialized, check_spmv, dense_abs_bound
from matrices import power_law_coo, random_coo

pytestmark = pytest.mark.gpu

SHAPES = [(37, 29, 0.2), (64, 64, 0.05), (5, 5, 0.4), (1, 3, 0.9), (3, 1, 0.9), (200, 150, 0.02)]


def _pair(ctx, ref, m, n, r, c, v):
    v = np.asarray(v, np.float32).astype(np.float64)
    return ctx.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v)


@pytest.mark.parametrize("b", [2, 3, 4, 16])
@pytest.mark.parametrize("shape", SHAPES)
def test_bell_matches_reference(ctx, ref, b, shape):
    m, n, dens = shape
    r, c, v = random_coo(b + m, m, n, dens)
    if len(v) == 0:
        return
    d, p = _pair(ctx, ref, m, n, r, c, v)
    got = ctx.convert(d, f"BELL({b})").download()
    want = ref.convert(p, "BELL", b).download()
    assert_same_materialized(got, want, (b, shape))


@pytest.mark.parametrize("b", [2, 4])
def test_bell_power_law(ctx, ref, b):
    """Ragged block rows: K is set by the densest block row, the rest pad."""
    m, n = 2000, 1500
    r, c, v = power_law_coo(7, m, n, avg=8, alpha=1.2)
    d, p = _pair(ctx, ref, m, n, r, c, v)
    dev = ctx.convert(d, f"BELL({b})")
    assert_same_materialized(dev.download(), ref.convert(p, "BELL", b).download(), b)
    x = np.random.default_rng(b).uniform(-1, 1, n).astype(np.float32)
    check_spmv(ctx.spmv(dev, x), ref.spmv(ref.convert(p, "BELL", b), x.astype(np.float64)),
               dense_abs_bound(r, c, v, m, x.astype(np.float64)), ("spmv", b))
    for nd in (1, 32, 64, 128, 7):
        bm = np.random.default_rng(nd).uniform(-1, 1, (n, nd)).astype(np.float32)
        got = ctx.spmm(dev, bm)
        want = ref.spmm(ref.convert(p, "BELL", b), bm.astype(np.float64))
        bound = np.zeros((m, nd))
        np.add.at(bound, np.asarray(r), np.abs(np.asarray(v, np.float64))[:, None] * np.abs(bm.astype(np.float64)[c]))
        assert np.all(np.abs(got - want) <= TOL * bound + 1e-30), (b, nd)


def test_bell_explicit_zeros_rejected(ctx):
    """Explicit zeros take the slot query's start-offset path (a block split
    over slots); the device path does not model it and says so."""
    d = ctx.from_coo(4, 4, [0, 0, 1], [0, 1, 2], [1.0, 0.0, 2.0])
    with pytest.raises(sfg.SfgError) as ei:
        ctx.convert(d, "BELL(2)")
    assert ei.value.kind == "UnsupportedSource"


def test_bell_container_matches_reference(ctx, ref, tmp_path):
    m, n = 37, 29
    r, c, v = random_coo(3, m, n, 0.2)
    d, p = _pair(ctx, ref, m, n, r, c, v)
    dev = ctx.convert(d, "BELL(3)")
    ours, theirs = tmp_path / "ours.uspt", tmp_path / "ref.uspt"
    ctx.write_container(dev, str(ours))
    ref.write_container(p, "BELL", str(theirs), 3)
    assert filecmp.cmp(ours, theirs, shallow=False)
    back = ctx.read_container(str(theirs), "BELL(3)")
    assert_same_materialized(back.download(), dev.download(), "read")
    x = np.linspace(-1, 1, n).astype(np.float32)
    np.testing.assert_array_equal(ctx.spmv(back, x), ctx.spmv(dev, x))


def test_bell_from_compressed_source(ctx, ref):
    """CSR -> BELL: dematerialize, then the COO path (planner.hpp:95-252)."""
    m, n = 40, 33
    r, c, v = random_coo(9, m, n, 0.15)
    d, p = _pair(ctx, ref, m, n, r, c, v)
    got = ctx.convert(ctx.convert(d, "CSR"), "BELL(4)").download()
    want = ref.convert_from(p, "CSR", "BELL", 4).download()
    assert_same_materialized(got, want, "csr->bell")
