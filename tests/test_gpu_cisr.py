"""CISR(k) and CISR-plus(k) (formats.hpp:67-72; the count, reorder and
schedule queries, query_engine.hpp:202-273): the device conversions are
bit-exact with the unmodified reference's materialized tensors — the
partitions holding entries, their rows, the rows' columns, the values and
the Partition(0) value ranges — SpMV / SpMM agree within the tolerance, the
container bytes equal the reference's, and CISR is refused as a
conversion source (indirect level) like the reference."""
import filecmp

import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL, assert_same_materialized, check_spmv, dense_abs_bound
from matrices import power_law_coo, random_coo
from test_gpu_dia_csb import CASES, _pair

pytestmark = pytest.mark.gpu

FMTS = ["CISR(2)", "CISR(3)", "CISR(7)", "CISR-plus(2)", "CISR-plus(3)", "CISR-plus(16)"]


def _ref(fmt):
    name, k = fmt.split("(")
    return name, int(k[:-1])


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("case", list(CASES) + ["power_law"])
def test_matches_reference(ctx, ref, fmt, case):
    if case == "power_law":
        m, n = 300, 250
        r, c, v = power_law_coo(3, m, n, avg=6, alpha=1.2)
        v = np.asarray(v, np.float32).astype(np.float64)
        v[::7] = 0.0  # explicit zeros: stored, but weigh nothing in the schedule
        d, p = ctx.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v)
    else:
        d, p, _ = _pair(ctx, ref, case)
    got = ctx.convert(d, fmt).download()
    want = ref.convert(p, *_ref(fmt)).download()
    assert_same_materialized(got, want, (fmt, case))
    assert got.partitions == want.partitions, (fmt, case)
    assert sfg.storage_explain(fmt) == ref.explain(fmt)


@pytest.mark.parametrize("fmt", ["CISR(3)", "CISR-plus(4)"])
def test_compute(ctx, ref, fmt):
    d, p, (m, n, r, c, v) = _pair(ctx, ref, "banded")
    a = ctx.convert(d, fmt)
    ra = ref.convert(p, *_ref(fmt))
    x = np.random.default_rng(0).uniform(-1, 1, n).astype(np.float32)
    check_spmv(ctx.spmv(a, x), ref.spmv(ra, x.astype(np.float64)), dense_abs_bound(r, c, v, m, x.astype(np.float64)),
               fmt)
    for nd in (1, 32, 128, 9):
        b = np.random.default_rng(nd).uniform(-1, 1, (n, nd)).astype(np.float32)
        got, want = ctx.spmm(a, b), ref.spmm(ra, b.astype(np.float64))
        bound = np.zeros((m, nd))
        np.add.at(bound, r, np.abs(v)[:, None] * np.abs(b.astype(np.float64)[c]))
        assert np.all(np.abs(got - want) <= TOL * bound + 1e-30), (fmt, nd)


@pytest.mark.parametrize("src", ["CSR", "DCSR", "CSC", "BCSR(2,2)"])
def test_from_compressed_sources(ctx, ref, src):
    d, p, _ = _pair(ctx, ref, "random")
    s, a, b = (src, 0, 0) if not src.startswith("BCSR") else ("BCSR", 2, 2)
    for fmt in ("CISR(3)", "CISR-plus(2)"):
        name, k = _ref(fmt)
        got = ctx.convert(ctx.convert(d, src), fmt).download()
        want = ref.convert_from(p, s, name, k, 0, a, b).download()
        assert_same_materialized(got, want, (src, fmt))
        assert got.partitions == want.partitions


def test_not_a_conversion_source(ctx, ref):
    d, _, _ = _pair(ctx, ref, "random")
    with pytest.raises(sfg.SfgError) as ei:
        ctx.convert(ctx.convert(d, "CISR(2)"), "CSR")
    assert ei.value.kind == "UnsupportedSource"


@pytest.mark.parametrize("fmt", ["CISR(3)", "CISR-plus(2)"])
def test_container_matches_reference(ctx, ref, tmp_path, fmt):
    d, p, _ = _pair(ctx, ref, "random")
    dev = ctx.convert(d, fmt)
    ours, theirs = tmp_path / "ours.uspt", tmp_path / "ref.uspt"
    ctx.write_container(dev, str(ours))
    name, k = _ref(fmt)
    ref.write_container(p, name, str(theirs), k)
    assert filecmp.cmp(ours, theirs, shallow=False), fmt
    back = ctx.read_container(str(theirs), fmt)
    assert_same_materialized(back.download(), dev.download(), ("read", fmt))
    assert back.download().partitions == dev.download().partitions


def test_large_schedule(ctx, ref):
    """A larger R-MAT-like matrix: the host schedule over every row, the
    device ordering and moves, against the reference."""
    m, n = 20000, 20000
    r, c, v = power_law_coo(11, m, n, avg=8, alpha=1.1)
    v = np.asarray(v, np.float32).astype(np.float64)
    d, p = ctx.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v)
    for fmt in ("CISR(8)", "CISR-plus(8)"):
        got = ctx.convert(d, fmt).download()
        want = ref.convert(p, *_ref(fmt)).download()
        assert_same_materialized(got, want, fmt)
        assert got.partitions == want.partitions


@pytest.mark.parametrize("fmt", ["CISR(2)", "CISR-plus(3)", "DCSC", "DIA-variant", "DIA", "BELL(2)", "HBELL(2,2)"])
def test_empty_matrix(ctx, ref, fmt):
    """No entries: the empty levels and bounds the reference materializes
    (HBELL: both parts empty)."""
    m, n = 5, 4
    e = np.array([], np.int64)
    d = ctx.from_coo(m, n, e, e, np.array([], np.float64))
    got = ctx.convert(d, fmt)
    x = np.ones(n, np.float32)
    assert np.all(ctx.spmv(got, x) == 0)
    if fmt.startswith("HBELL"):
        return
    if "(" in fmt and not fmt.startswith("BELL"):
        name, k = _ref(fmt)
        want = ref.convert(ref.from_coo(m, n, e, e, np.array([], np.float64)), name, k).download()
    elif fmt.startswith("BELL"):
        want = ref.convert(ref.from_coo(m, n, e, e, np.array([], np.float64)), "BELL", 2).download()
    else:
        want = ref.convert(ref.from_coo(m, n, e, e, np.array([], np.float64)), fmt).download()
    assert_same_materialized(got.download(), want, fmt)
