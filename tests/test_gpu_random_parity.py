"""Seeded random sweep over every named format: random shapes (1..700 ×
1..700), densities from 0.1 % to 20 %, some inputs with explicit zeros —
each conversion from canonical COO bit-exact with the unmodified
reference's materialized tensor (levels, bounds, node counts, values,
partitions), and the SpMV of every format within the fp32 tolerance."""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL, assert_same_materialized

pytestmark = pytest.mark.gpu

FMTS = ["COO", "CSR", "CSC", "DCSR", "DCSC", "ELL", "BCSR(2,2)", "BCSR(3,5)", "BELL(2)", "BELL(3)", "DIA",
        "DIA-variant", "BDIA(3)", "CSB(2,3)", "C2SR(4)", "CISR(3)", "CISR-plus(5)", "DOK", "LIL"]


def _ref_fmt(f):
    if "(" not in f:
        return f, 0, 0
    name, args = f.split("(")
    a = [int(x) for x in args[:-1].split(",")]
    return name, a[0], a[1] if len(a) > 1 else (a[0] if name in ("BCSR", "CSB") else 0)


@pytest.mark.parametrize("seed", range(12))
def test_random_matrices_all_formats(ctx, ref, seed):
    rng = np.random.default_rng(1000 + seed)
    m, n = int(rng.integers(1, 700)), int(rng.integers(1, 700))
    dens = float(rng.choice([0.001, 0.01, 0.05, 0.2]))
    key = np.unique(rng.integers(0, m * n, max(1, int(m * n * dens))))
    r, c = key // n, key % n
    v = (rng.random(len(r)) * 2 - 1).astype(np.float32).astype(np.float64)
    zeros = seed % 3 == 0
    if zeros:
        v[rng.random(len(v)) < 0.2] = 0.0
    d, p = ctx.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v)
    x = rng.uniform(-1, 1, n).astype(np.float32)
    A = np.zeros((m, n))
    A[r, c] = v
    bound = np.abs(A) @ np.abs(x.astype(np.float64))
    for f in FMTS:
        if f.startswith("BELL") and zeros:
            continue  # BELL over explicit zeros is refused (row +2)
        t = ctx.convert(d, f)
        want = ref.convert(p, *_ref_fmt(f)).download()
        got = t.download()
        assert_same_materialized(got, want, (seed, f, m, n, dens))
        assert got.partitions == want.partitions, (seed, f)
        y = ctx.spmv(t, x).astype(np.float64)
        assert np.all(np.abs(y - A @ x.astype(np.float64)) <= TOL * bound + 1e-30), (seed, f)


SOURCES = ["CSR", "DCSR", "CSC", "DCSC", "BCSR(2,2)"]
TARGETS = ["COO", "CSR", "CSC", "DCSR", "DCSC", "ELL", "BCSR(2,3)", "BELL(2)", "CSB(2,2)", "C2SR(3)", "CISR(2)", "DOK",
           "LIL"]


@pytest.mark.parametrize("seed", range(6))
def test_random_conversions_from_sources(ctx, ref, seed):
    """planner.hpp:95-252 from each compressed source to each target,
    bit-exact with the reference's convert_structure."""
    rng = np.random.default_rng(2000 + seed)
    m, n = int(rng.integers(2, 300)), int(rng.integers(2, 300))
    key = np.unique(rng.integers(0, m * n, max(1, int(m * n * 0.05))))
    r, c = key // n, key % n
    v = (rng.random(len(r)) * 2 - 1).astype(np.float32).astype(np.float64)
    d, p = ctx.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v)
    for s in SOURCES:
        src = ctx.convert(d, s)
        sn, sa, sb = _ref_fmt(s)
        for f in TARGETS:
            fn, fa, fb = _ref_fmt(f)
            got = ctx.convert(src, f).download()
            want = ref.convert_from(p, sn, fn, fa, fb, sa, sb).download()
            assert_same_materialized(got, want, (seed, s, f))
            assert got.partitions == want.partitions, (seed, s, f)


@pytest.mark.parametrize("seed", range(6))
def test_random_spmm_all_formats(ctx, seed):
    """SpMM over every format for widths 1, 3, 32, 64, 128 (fp32 B) against
    the f64 dense product."""
    rng = np.random.default_rng(3000 + seed)
    m, n = int(rng.integers(1, 400)), int(rng.integers(1, 400))
    key = np.unique(rng.integers(0, m * n, max(1, int(m * n * 0.03))))
    r, c = key // n, key % n
    v = (rng.random(len(r)) * 2 - 1).astype(np.float32).astype(np.float64)
    d = ctx.from_coo(m, n, r, c, v)
    A = np.zeros((m, n))
    A[r, c] = v
    for f in FMTS + ["HYB(4)", "HBELL(2,2)", "BCSR(16,16)", "BCSR(4,4)"]:
        t = ctx.convert(d, f)
        for nd in (1, 3, 32, 64, 128):
            b = rng.uniform(-1, 1, (n, nd)).astype(np.float32)
            got = ctx.spmm(t, b).astype(np.float64)
            bound = np.abs(A) @ np.abs(b.astype(np.float64))
            assert np.all(np.abs(got - A @ b.astype(np.float64)) <= TOL * bound + 1e-30), (seed, f, nd)
