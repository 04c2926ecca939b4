"""Hybrid BELL/COO — the paper's GPU format (PAPER.md, Hybrid BELL/COO; the
BELL part built by the block count query, decompose.hpp:30-63): decompose by
r x c blocks is bit-exact with the unmodified reference's decompose under
the block rule (both parts, input order kept), the BELL part equals the
reference's BELL of the selected entries, and SpMV / SpMM over the pair
match the dense product."""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL, assert_same_materialized
from matrices import power_law_coo, random_coo

pytestmark = pytest.mark.gpu


def blocky(seed, m, n, b, dens_blocks=0.15, fill_dense=0.9, scatter=0.01):
    """Dense-ish b x b blocks plus scattered entries."""
    rng = np.random.default_rng(seed)
    a = np.zeros((m, n))
    for bi in range(0, m, b):
        for bj in range(0, n, b):
            if rng.random() < dens_blocks:
                blk = rng.random((min(b, m - bi), min(b, n - bj))) < fill_dense
                a[bi:bi + b, bj:bj + b][blk] = 1.0
    a[rng.random((m, n)) < scatter] = 1.0
    r, c = np.nonzero(a)
    v = (0.5 + rng.random(len(r))).astype(np.float32).astype(np.float64) * np.where(rng.random(len(r)) < .5, -1, 1)
    return r, c, v


@pytest.mark.parametrize("b,t", [(2, 2), (4, 8), (4, 1), (8, 40), (16, 100)])
@pytest.mark.parametrize("case", ["blocky", "random", "power_law"])
def test_decompose_blocks_matches_reference(ctx, ref, case, b, t):
    m, n = 150, 130
    if case == "blocky":
        r, c, v = blocky(b, m, n, b)
    elif case == "random":
        r, c, v = random_coo(b, m, n, 0.1)
    else:
        r, c, v = power_law_coo(b, m, n, avg=10, alpha=1.3)
    d, p = ctx.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v)
    ds, dr = ctx.decompose_blocks(d, b, b, t)
    ps, pr = ref.decompose_blocks(p, b, b, t)
    for dd, pp, what in ((ds, ps, "selected"), (dr, pr, "remainder")):
        assert_same_materialized(ctx.convert(dd, "COO").download(), ref.convert(pp, "COO").download(), (case, b, t, what))
    if ps.nnz:  # the BELL part: the reference's BELL of the selected entries
        hb = ctx.convert(d, f"HBELL({b},{t})")
        bell, coo = hb.parts()
        assert bell.kind == "BELL" and coo.kind == "COO"
        assert_same_materialized(bell.download(), ref.convert(ps, "BELL", b).download(), (case, b, t, "bell"))


@pytest.mark.parametrize("case", ["zeros", "wide"])
def test_decompose_blocks_paths(ctx, ref, case):
    """Explicit zeros (the count rule counts only nonzero values) and a block
    grid wider than the device's shared counters (the radix-order path)."""
    b, t = 2, 2
    if case == "zeros":
        m, n = 150, 130
        r, c, v = blocky(3, m, n, b)
        v = v.copy()
        v[np.random.default_rng(1).random(len(v)) < 0.3] = 0.0
    else:
        m, n = 40, 200_000
        rng = np.random.default_rng(2)
        r = rng.integers(0, m, 3000)
        c = np.concatenate([rng.integers(0, n, 1500), rng.integers(0, 200, 1500)])
        key = np.unique(r * n + c)
        r, c = key // n, key % n
        v = (0.5 + rng.random(len(r))).astype(np.float32).astype(np.float64)
    d, p = ctx.from_coo(m, n, r, c, v), ref.from_coo(m, n, r, c, v)
    ds, dr = ctx.decompose_blocks(d, b, b, t)
    ps, pr = ref.decompose_blocks(p, b, b, t)
    assert 0 < ps.nnz < len(v)
    for dd, pp, what in ((ds, ps, "selected"), (dr, pr, "remainder")):
        assert_same_materialized(ctx.convert(dd, "COO").download(), ref.convert(pp, "COO").download(), (case, what))


@pytest.mark.parametrize("b,t", [(4, 8), (16, 128)])
def test_hbell_spmv_spmm(ctx, b, t):
    m, n = 1000, 900
    r, c, v = blocky(7, m, n, b, scatter=0.003)
    a = ctx.convert(ctx.from_coo(m, n, r, c, v), f"HBELL({b},{t})")
    A = np.zeros((m, n)); A[r, c] = v
    x = np.random.default_rng(0).uniform(-1, 1, n).astype(np.float32)
    y = ctx.spmv(a, x).astype(np.float64)
    assert np.all(np.abs(y - A @ x) <= TOL * (np.abs(A) @ np.abs(x)) + 1e-30)
    for nd in (32, 128, 3):
        bm = np.random.default_rng(nd).uniform(-1, 1, (n, nd)).astype(np.float32)
        got = ctx.spmm(a, bm).astype(np.float64)
        assert np.all(np.abs(got - A @ bm) <= TOL * (np.abs(A) @ np.abs(bm)) + 1e-30), nd


def test_hbell_names_and_plan():
    f = sfg.resolve_format("HBELL(4, 10)")
    assert (f.kind, f.block_r, f.threshold) == (sfg.KINDS["HBELL"], 4, 10)
    lines = sfg.plan_lines("COO", "HBELL(4,10)")
    assert lines[0].startswith("Decompose(sum(value) groupBy (d0, d1) -> (d0/4, d1/4)")
    assert lines[1:] == ["selected: " + l for l in sfg.plan_lines("COO", "BELL(4)")]
