"""Row partitioning on the device without a multi-GPU box.

* sfg_row_partition against the host rule (sfgx_row_bounds_host and the
  Python restatement rowpart.row_bounds) for P in {2, 4, 8} on R-MAT s20;
* sfg_coo_slice_rows against a numpy slice of the canonical COO;
* a P-block simulation on one device: every block is sliced, converted and
  multiplied through the row-partitioned entry points (sfg_rowpart_spmv /
  sfg_rowpart_spmm, one-rank communicator, no gather) into its chunk of one
  output buffer; the reassembled product equals the unpartitioned one and
  the f64 oracle within the north-star tolerance. The all-gather between
  real ranks is the one step this cannot run (one GPU per box)."""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL
from paper_2403_05802_b200.rowpart import row_bounds

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rmat20(ctx):
    coo = ctx.gen_rmat(7, 20, 16 << 20)
    return coo, coo.coo_arrays()


@pytest.fixture(scope="module")
def comm(ctx):
    c = ctx.comm_create(1, 0, sfg.comm_unique_id())
    yield c
    c.close()


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_row_partition_matches_host_rule(ctx, rmat20, parts):
    coo, (r, c, v) = rmat20
    m = coo.shape[0]
    b = ctx.row_partition(coo, parts)
    assert b == sfg.row_bounds_host(r, m, parts) == row_bounds(r, m, parts)
    counts = np.diff(np.searchsorted(r, b))
    heaviest = np.bincount(r).max()
    assert all(abs(int(k) - len(r) / parts) <= heaviest for k in counts), counts


@pytest.mark.parametrize("r0,r1", [(0, 1), (0, 1024), (1000, 5000), (1 << 19, 1 << 20), (77, 77)])
def test_coo_slice_rows(ctx, rmat20, r0, r1):
    coo, (r, c, v) = rmat20
    s = ctx.slice_rows(coo, r0, r1)
    assert s.shape == (r1 - r0, coo.shape[1])
    sel = (r >= r0) & (r < r1)
    sr, sc, sv = s.coo_arrays()
    np.testing.assert_array_equal(sr, r[sel] - r0)
    np.testing.assert_array_equal(sc, c[sel])
    np.testing.assert_array_equal(sv.view(np.uint32), v[sel].view(np.uint32))


def _bound_rows(r, c, v, m, x):
    return np.bincount(r, weights=np.abs(v.astype(np.float64)) * np.abs(x[c]), minlength=m)


@pytest.mark.parametrize("parts", [2, 4, 8])
@pytest.mark.parametrize("fmt", ["CSR", "HYB(8)", "DCSR"])
def test_pblock_spmv_simulation(ctx, port, comm, rmat20, parts, fmt):
    coo, (r, c, v) = rmat20
    m, n = coo.shape
    x = port.gen_dense(3, n)
    xb = sfg.DeviceBuffer(ctx, n * 4).upload(x.astype(np.float32))
    b = ctx.row_partition(coo, parts)
    chunk = max(b[p + 1] - b[p] for p in range(parts))
    yb = sfg.DeviceBuffer(ctx, parts * chunk * 4).upload(np.full(parts * chunk, np.nan, np.float32))
    for p in range(parts):
        a = ctx.convert(ctx.slice_rows(coo, b[p], b[p + 1]), fmt)
        ctx.rowpart_spmv(comm, a, xb.ptr, yb.ptr + p * chunk * 4, chunk, gather=False)
    y = yb.download(np.float32, parts * chunk)
    y = np.concatenate([y[p * chunk: p * chunk + b[p + 1] - b[p]] for p in range(parts)])
    whole = ctx.spmv(ctx.convert(coo, fmt), x.astype(np.float32))
    want = port.spmv(port.convert(port.from_coo(m, n, r, c, v), "CSR"), x)
    bound = _bound_rows(r, c, v, m, x)
    assert np.all(np.abs(y - want) <= TOL * bound + 1e-30)
    assert np.all(np.abs(whole - want) <= TOL * bound + 1e-30)


@pytest.mark.parametrize("parts", [2, 8])
def test_pblock_spmm_simulation(ctx, port, comm, rmat20, parts):
    coo, (r, c, v) = rmat20
    m, n = coo.shape
    nd = 32
    bdev = sfg.DeviceBuffer(ctx, n * nd * 4)
    ctx.gen_dense(3, n * nd, bdev.ptr)
    bh = bdev.download(np.float32, n * nd).reshape(n, nd).astype(np.float64)
    bnd = ctx.row_partition(coo, parts)
    chunk = max(bnd[p + 1] - bnd[p] for p in range(parts))
    cb = sfg.DeviceBuffer(ctx, parts * chunk * nd * 4).upload(np.full(parts * chunk * nd, np.nan, np.float32))
    for p in range(parts):
        a = ctx.convert(ctx.slice_rows(coo, bnd[p], bnd[p + 1]), "CSR")
        ctx.rowpart_spmm(comm, a, bdev.ptr, sfg.F32, nd, cb.ptr + p * chunk * nd * 4, chunk, gather=False)
    out = cb.download(np.float32, parts * chunk * nd).reshape(parts * chunk, nd)
    out = np.concatenate([out[p * chunk: p * chunk + bnd[p + 1] - bnd[p]] for p in range(parts)])
    pa = port.convert(port.from_coo(m, n, r, c, v), "CSR")
    want = port.spmm(pa, bh)
    bound = port.spmm(port.convert(port.from_coo(m, n, r, c, np.abs(v.astype(np.float64))), "CSR"), np.abs(bh))
    assert np.all(np.abs(out - want) <= TOL * bound + 1e-30)
