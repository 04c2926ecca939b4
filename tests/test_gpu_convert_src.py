"""Conversions from compressed sources: a tensor held
in CSR / DCSR / CSC / BCSR converted to every target, bit-exact against the
unmodified reference's convert_structure from that source (planner.hpp:95:
normalize — split, trim every untrimmed level — realign, regrow), through
the oracle shim. The matrices carry explicit zeros, all-zero rows and
columns and empty rows: exactly what the reference's Trim(l) treats
specially (operators.hpp:302-345)."""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import assert_same_materialized

pytestmark = pytest.mark.gpu

SOURCES = ["CSR", "DCSR", "CSC", "BCSR(2,2)", "BCSR(3,2)"]
TARGETS = ["COO", "CSR", "DCSR", "CSC", "ELL", "BCSR(2,2)", "BCSR(4,4)"]


def split_fmt(f):
    if f.startswith("BCSR"):
        r, c = (int(t) for t in f[5:-1].split(","))
        return "BCSR", r, c
    return f, 0, 0


def matrix(seed, m=37, n=29):
    rng = np.random.default_rng(seed)
    dense = (rng.random((m, n)) < 0.25) * (rng.integers(1, 9, (m, n)) * 0.5)
    dense[rng.random((m, n)) < 0.08] = 0.0  # some stored zeros below
    keep = (rng.random((m, n)) < 0.3) | (dense != 0)
    keep[3, :] = False                       # empty row
    keep[5, ::4] = True; dense[5, :] = 0.0   # a row of stored zeros only
    keep[:, 7] = False
    keep[::3, 11] = True; dense[:, 11] = 0.0  # a column of stored zeros only
    r, c = np.nonzero(keep)
    return m, n, r, c, dense[r, c]


@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("dst", TARGETS)
@pytest.mark.parametrize("src", SOURCES)
def test_convert_from_compressed_source(ctx, ref, src, dst, seed):
    m, n, r, c, v = matrix(seed)
    d = ctx.from_coo(m, n, r, c, v)
    s = ctx.convert(d, src)
    out = ctx.convert(s, dst).download()
    sk, sr, sc = split_fmt(src)
    dk, dr, dc = split_fmt(dst)
    want = ref.convert_from(ref.from_coo(m, n, r, c, v), sk, dk, dr, dc, sr, sc).download()
    assert_same_materialized(out, want, (src, dst, seed))


@pytest.mark.parametrize("dst", ["COO", "CSR", "HYB(3)"])
def test_ell_source_is_unsupported(ctx, dst):
    d = ctx.from_coo(4, 4, [0, 1, 2], [1, 2, 3], [1.0, 2.0, 3.0])
    with pytest.raises(sfg.SfgError) as ei:
        ctx.convert(ctx.convert(d, "ELL"), dst)
    assert ei.value.kind == "UnsupportedSource"


def test_compressed_round_trip_spmv(ctx, port):
    """CSR -> CSC -> DCSR -> COO keeps the operator (no stored zeros here)."""
    rng = np.random.default_rng(3)
    m, n = 300, 200
    keep = rng.random((m, n)) < 0.05
    r, c = np.nonzero(keep)
    v = rng.random(len(r)) + 0.5
    t = ctx.from_coo(m, n, r, c, v)
    for f in ["CSR", "CSC", "DCSR", "BCSR(4,4)", "COO"]:
        t = ctx.convert(t, f)
    rr, cc, vv = t.coo_arrays()
    assert rr.tolist() == r.tolist() and cc.tolist() == c.tolist()
    np.testing.assert_array_equal(vv, v.astype(np.float32))
