"""Row-partitioned path through the C-ABI: sfg_comm_create,
sfg_rowpart_spmv / sfg_rowpart_spmm, sfg_allgather_chunks.

The box has one GPU, so the communicator here has one rank: the product
must land in chunk 0 exactly as the plain SpMV / SpMM computes it, the
all-gather is the identity, and the size checks hold. The multi-rank chunk
layout and the reassembly are covered on CPU (tests/test_multirank.py,
gloo, world size 2)."""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm(ctx):
    c = ctx.comm_create(1, 0, sfg.comm_unique_id())
    yield c
    c.close()


def test_rowpart_spmv_one_rank(ctx, comm, port):
    coo = ctx.gen_rmat(7, 12, 16 << 12)
    m, n = coo.shape
    x = port.gen_dense(3, n).astype(np.float32)
    for fmt in ("CSR", "HYB(8)", "DCSR"):
        a = ctx.convert(coo, fmt)
        chunk = m + 37  # padding rows past the block stay untouched
        xb = sfg.DeviceBuffer(ctx, n * 4).upload(x)
        yb = sfg.DeviceBuffer(ctx, chunk * 4).upload(np.full(chunk, -7.0, np.float32))
        ctx.rowpart_spmv(comm, a, xb.ptr, yb.ptr, chunk)
        y = yb.download(np.float32, chunk)
        # the COO half of HYB adds with atomics: equal up to summation order
        np.testing.assert_allclose(y[:m], ctx.spmv(a, x), rtol=1e-5, atol=1e-5, err_msg=fmt)
        assert np.all(y[m:] == -7.0)


def test_rowpart_spmm_one_rank(ctx, comm, port):
    coo = ctx.gen_hypersparse(5, 5000, 3000, 12000)
    m, n = coo.shape
    nd = 64
    b = port.gen_dense(4, n * nd).astype(np.float32).reshape(n, nd)
    a = ctx.convert(coo, "DCSR")
    bb = sfg.DeviceBuffer(ctx, b.nbytes).upload(b)
    cb = sfg.DeviceBuffer(ctx, m * nd * 4)
    ctx.rowpart_spmm(comm, a, bb.ptr, sfg.F32, nd, cb.ptr, m)
    np.testing.assert_array_equal(cb.download(np.float32, m * nd).reshape(m, nd), ctx.spmm(a, b))


def test_rowpart_checks(ctx, comm):
    coo = ctx.gen_uniform(1, 256, 256, 4)
    a = ctx.convert(coo, "CSR")
    xb = sfg.DeviceBuffer(ctx, 256 * 4)
    yb = sfg.DeviceBuffer(ctx, 256 * 4)
    with pytest.raises(sfg.SfgError) as ei:
        ctx.rowpart_spmv(comm, a, xb.ptr, yb.ptr, 255)  # block larger than its chunk
    assert ei.value.kind == "InvalidOperation"
    ctx.allgather_chunks(comm, yb.ptr, 256)  # one rank: identity
    with pytest.raises(sfg.SfgError) as ei:
        ctx.comm_create(2, 2, sfg.comm_unique_id())
    assert ei.value.kind == "InvalidOperation"
