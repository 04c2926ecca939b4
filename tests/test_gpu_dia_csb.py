"""DIA (formats.hpp:46), BDIA(b) (76-79), CSB(r,c) (54-57) and C2SR(k)
(62-66, Partition(0): per-class value ranges), §8f rank 2: the
device conversions from canonical COO are bit-exact with the unmodified
reference's materialized tensors (DIA: ascending diagonals, zero-filled
diagonal-major panel; CSB: the dense block grid's ptr and the in-block
coordinates), SpMV / SpMM agree within the tolerance, and the container
round-trips byte-identically. Neither is taken as a conversion source (the
reference's expansion gives them skewed / tile-grid level bounds)."""
import filecmp

import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL, assert_same_materialized, check_spmv, dense_abs_bound
from matrices import random_coo

pytestmark = pytest.mark.gpu


def banded(seed, m, n, width, zeros=0.0):
    rng = np.random.default_rng(seed)
    r, c = [], []
    for i in range(m):
        for d in range(-width, width + 1):
            if 0 <= i + d < n and rng.random() < 0.7:
                r.append(i)
                c.append(i + d)
    r, c = np.array(r, np.int64), np.array(c, np.int64)
    v = (0.5 + rng.random(len(r))).astype(np.float32).astype(np.float64)
    if zeros:
        v[rng.random(len(r)) < zeros] = 0.0
    return r, c, v


CASES = {
    "random": (37, 29, lambda: random_coo(1, 37, 29, 0.15, zeros=0.1)),
    "banded": (300, 280, lambda: banded(2, 300, 280, 5, zeros=0.05)),
    "tall": (50, 3, lambda: random_coo(3, 50, 3, 0.3)),
    "wide": (2, 40, lambda: random_coo(4, 2, 40, 0.3)),
    "one": (1, 3, lambda: ([0], [2], [7.0])),
}


def _pair(ctx, ref, case):
    m, n, gen = CASES[case]
    r, c, v = gen()
    v = np.asarray(v, np.float32).astype(np.float64)
    return ctx.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v), (m, n, np.asarray(r), np.asarray(c), v)


def _ref_fmt(fmt):
    if fmt.startswith("CSB"):
        a = [int(t) for t in fmt[4:-1].split(",")]
        return "CSB", a[0], a[1] if len(a) > 1 else a[0]
    if fmt.startswith("BDIA"):
        return "BDIA", int(fmt[5:-1]), 0
    if fmt.startswith("C2SR"):
        return "C2SR", int(fmt[5:-1]), 0
    return fmt, 0, 0


@pytest.mark.parametrize("fmt", ["DIA", "CSB(2)", "CSB(2,3)", "CSB(16)", "BDIA(2)", "BDIA(3)", "BDIA(16)",
                                 "C2SR(2)", "C2SR(3)", "C2SR(64)"])
@pytest.mark.parametrize("case", list(CASES))
def test_matches_reference(ctx, ref, fmt, case):
    d, p, _ = _pair(ctx, ref, case)
    got = ctx.convert(d, fmt).download()
    want = ref.convert(p, *_ref_fmt(fmt)).download()
    assert_same_materialized(got, want, (fmt, case))
    assert got.partitions == want.partitions, (fmt, case)
    assert got.explain() == want.explain() == sfg.storage_explain(fmt)


@pytest.mark.parametrize("fmt", ["DIA", "CSB(4)", "CSB(3,2)", "BDIA(4)", "BDIA(3)", "C2SR(2)", "C2SR(5)"])
def test_compute(ctx, ref, fmt):
    d, p, (m, n, r, c, v) = _pair(ctx, ref, "banded")
    a = ctx.convert(d, fmt)
    ra = ref.convert(p, *_ref_fmt(fmt))
    x = np.random.default_rng(0).uniform(-1, 1, n).astype(np.float32)
    check_spmv(ctx.spmv(a, x), ref.spmv(ra, x.astype(np.float64)), dense_abs_bound(r, c, v, m, x.astype(np.float64)),
               fmt)
    for nd in (1, 32, 128, 9):
        b = np.random.default_rng(nd).uniform(-1, 1, (n, nd)).astype(np.float32)
        got, want = ctx.spmm(a, b), ref.spmm(ra, b.astype(np.float64))
        bound = np.zeros((m, nd))
        np.add.at(bound, r, np.abs(v)[:, None] * np.abs(b.astype(np.float64)[c]))
        assert np.all(np.abs(got - want) <= TOL * bound + 1e-30), (fmt, nd)


@pytest.mark.parametrize("src", ["DIA", "CSB(2)", "CSB(2,3)", "BDIA(2)"])
def test_not_a_conversion_source(ctx, ref, src):
    """The reference expands a DIA source through its skewed map (its column
    level comes back as [-(m-1), n+m-2]) and a CSB source with tile-grid
    extents; the device does not model those bounds and says so."""
    d, p, _ = _pair(ctx, ref, "random")
    with pytest.raises(sfg.SfgError) as ei:
        ctx.convert(ctx.convert(d, src), "CSR")
    assert ei.value.kind == "UnsupportedSource"
    s, sr, sc = _ref_fmt(src)
    want = ref.convert_from(p, s, "COO", 0, 0, sr, sc).download()
    assert (want.levels[1].lo, want.levels[1].hi) != (0, 28) or want.levels[0].node_count != len(want.values)


@pytest.mark.parametrize("fmt", ["DIA", "CSB(2,3)", "BDIA(3)", "C2SR(3)"])
def test_container_matches_reference(ctx, ref, tmp_path, fmt):
    d, p, (m, n, r, c, v) = _pair(ctx, ref, "random")
    dev = ctx.convert(d, fmt)
    ours, theirs = tmp_path / "ours.uspt", tmp_path / "ref.uspt"
    ctx.write_container(dev, str(ours))
    f, a, b = _ref_fmt(fmt)
    ref.write_container(p, f, str(theirs), a, b)
    assert filecmp.cmp(ours, theirs, shallow=False), fmt
    for f in (fmt, None):  # named, or inferred from the stored levels
        back = ctx.read_container(str(theirs), f)
        assert_same_materialized(back.download(), dev.download(), ("read", fmt, f))
        assert back.download().partitions == dev.download().partitions


def test_dia_capacity_error(ctx):
    """A DIA panel of (diagonals x rows) beyond the device's capacity is
    refused, not truncated."""
    m = n = 1 << 17
    r, c, v = random_coo(9, 64, 64, 0.5)
    d = ctx.from_coo(m, n, np.concatenate([r, [m - 1]]), np.concatenate([c * 2000, [0]]),
                     np.concatenate([v, [1.0]]))
    try:
        ctx.convert(d, "DIA")
    except sfg.SfgError as e:
        assert e.kind == "InvalidOperation"
