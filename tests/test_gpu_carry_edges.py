"""Edge cases of the atomic-free reductions (merge-path CSR SpMM, COO SpMV /
SpMM with per-chunk carry slots and the log-32 carry tree): no entries at
all, one row spanning every chunk, rows ending exactly on chunk boundaries,
empty rows between long ones, accumulate — against the f64 dense product."""
import numpy as np
import pytest
import torch

from gpu_common import TOL

pytestmark = pytest.mark.gpu


def _dense(m, n, r, c, v):
    a = np.zeros((m, n))
    a[r, c] = v
    return a


def _cases():
    rng = np.random.default_rng(0)
    out = {}
    out["no_entries"] = (50, 40, np.zeros(0, int), np.zeros(0, int), np.zeros(0))
    n = 70000  # one row longer than ~60 merge-path chunks and ~180 COO chunks
    out["one_long_row"] = (3, n, np.full(n, 1), np.arange(n), rng.uniform(0.5, 1.5, n))
    # rows of exactly 1024 - 1 entries: row ends land on merge-path chunk edges
    m, L = 40, 1023
    r = np.repeat(np.arange(m), L)
    c = np.tile(np.arange(L), m)
    out["chunk_aligned"] = (m, L, r, c, rng.uniform(-1, 1, len(r)))
    # long rows separated by runs of empty rows, plus a long last row
    rows, cols = [], []
    for i in (0, 5000, 5001, 9999):
        k = 3000 if i != 5001 else 1
        rows.append(np.full(k, i))
        cols.append(np.sort(rng.choice(4000, k, replace=False)))
    out["sparse_long_rows"] = (10000, 4000, np.concatenate(rows), np.concatenate(cols),
                               rng.uniform(-1, 1, sum(len(x) for x in rows)))
    return out


CASES = _cases()


@pytest.mark.parametrize("fmt", ["COO", "CSR", "DOK", "LIL", "HYB(4)"])
@pytest.mark.parametrize("case", list(CASES))
def test_spmv_edges(ctx, fmt, case):
    m, n, r, c, v = CASES[case]
    v = np.asarray(v, np.float32).astype(np.float64)
    a = ctx.convert(ctx.from_coo(m, n, r, c, v), fmt)
    x = np.random.default_rng(1).uniform(-1, 1, n).astype(np.float32)
    A = _dense(m, n, r, c, v)
    want, bound = A @ x.astype(np.float64), np.abs(A) @ np.abs(x.astype(np.float64))
    got = ctx.spmv(a, x).astype(np.float64)
    assert np.all(np.abs(got - want) <= TOL * bound + 1e-30), (fmt, case)


@pytest.mark.parametrize("nd", [32, 64, 128, 5])
@pytest.mark.parametrize("fmt", ["COO", "CSR", "LIL"])
@pytest.mark.parametrize("case", list(CASES))
def test_spmm_edges(ctx, fmt, case, nd):
    m, n, r, c, v = CASES[case]
    v = np.asarray(v, np.float32).astype(np.float64)
    a = ctx.convert(ctx.from_coo(m, n, r, c, v), fmt)
    b = np.random.default_rng(nd).uniform(-1, 1, (n, nd)).astype(np.float32)
    A = _dense(m, n, r, c, v)
    want = A @ b.astype(np.float64)
    bound = np.abs(A) @ np.abs(b.astype(np.float64))
    got = ctx.spmm(a, b).astype(np.float64)
    assert np.all(np.abs(got - want) <= TOL * bound + 1e-30), (fmt, case, nd)
    # accumulate on top of a non-zero C, and the same bits on every run
    c0 = torch.rand(m * nd, device="cuda")
    bd = torch.from_numpy(b).cuda()
    outs = []
    for _ in range(3):
        cc = c0.clone()
        ctx.spmm_device(a, bd.data_ptr(), 0, nd, cc.data_ptr(), accumulate=True)
        outs.append(cc)
    torch.cuda.synchronize()
    acc = outs[0].cpu().numpy().reshape(m, nd).astype(np.float64)
    base = c0.cpu().numpy().reshape(m, nd).astype(np.float64)
    assert np.all(np.abs(acc - (want + base)) <= TOL * (bound + np.abs(base)) + 1e-30), (fmt, case, nd, "acc")
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
