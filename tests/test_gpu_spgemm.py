"""Two sparse operands: run_kernel(spgemm_kernel(),
{A, B}) (kernel.hpp:53, 424-567) into a dense C, against the unmodified
reference (both its co-iterate and probe modes) within
|C_hat - C| <= 1e-5 * sum_k |a_ik| |b_kj|."""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import TOL
from matrices import random_coo

pytestmark = pytest.mark.gpu

FMTS = ["COO", "CSR", "DCSR", "CSC", "BCSR(2,2)"]


def split(f):
    if f.startswith("BCSR"):
        r, c = (int(t) for t in f[5:-1].split(","))
        return "BCSR", r, c
    return f, 0, 0


@pytest.mark.parametrize("fb", FMTS)
@pytest.mark.parametrize("fa", FMTS)
def test_spgemm_matches_reference(ctx, ref, fa, fb):
    m, k, n = 36, 28, 22
    ra, ca, va = random_coo(3, m, k, 0.2, zeros=0.1)
    rb, cb, vb = random_coo(4, k, n, 0.25, zeros=0.1)
    da = ctx.convert(ctx.from_coo(m, k, ra, ca, va), fa)
    db = ctx.convert(ctx.from_coo(k, n, rb, cb, vb), fb)
    got = ctx.spgemm(da, db)
    ka, ar, ac = split(fa)
    kb, br, bc = split(fb)
    want, mode = ref.spgemm(ref.convert(ref.from_coo(m, k, ra, ca, va), ka, ar, ac),
                            ref.convert(ref.from_coo(k, n, rb, cb, vb), kb, br, bc))
    A = np.zeros((m, k)); A[ra, ca] = va
    B = np.zeros((k, n)); B[rb, cb] = vb
    bound = np.abs(A) @ np.abs(B)
    err = np.abs(got.astype(np.float64) - want)
    assert (err <= TOL * bound + 1e-30).all(), (fa, fb, mode, err.max())


def test_spgemm_power_law_and_accumulate(ctx):
    rng = np.random.default_rng(1)
    m = k = n = 400
    A = (rng.random((m, k)) < 0.03) * rng.random((m, k))
    A[7, :] = rng.random(k)  # one dense row
    B = (rng.random((k, n)) < 0.03) * rng.random((k, n))
    ra, ca = np.nonzero(A)
    rb, cb = np.nonzero(B)
    da = ctx.convert(ctx.from_coo(m, k, ra, ca, A[ra, ca]), "CSR")
    db = ctx.convert(ctx.from_coo(k, n, rb, cb, B[rb, cb]), "DCSR")
    c0 = rng.random((m, n)).astype(np.float32)
    buf = ctx.buffer(c0.nbytes).upload(c0)
    ctx.spgemm_device(da, db, buf.ptr, accumulate=True)
    got = buf.download(np.float32, m * n).reshape(m, n).astype(np.float64)
    want = A @ B + c0
    bound = np.abs(A) @ np.abs(B) + np.abs(c0)
    assert (np.abs(got - want) <= TOL * bound + 1e-30).all()


def test_spgemm_errors(ctx):
    a = ctx.convert(ctx.from_coo(3, 4, [0], [1], [1.0]), "CSR")
    b = ctx.convert(ctx.from_coo(5, 2, [0], [1], [1.0]), "CSR")
    with pytest.raises(sfg.SfgError) as ei:
        ctx.spgemm(a, b)
    assert ei.value.kind == "InvalidOperation"



EXTRA = ["ELL", "HYB(2)", "DOK", "LIL", "BELL(2)", "DIA", "CSB(2,3)", "BDIA(3)", "C2SR(3)", "DCSC", "DIA-variant", "HBELL(2,2)",
         "CISR(3)", "CISR-plus(2)"]


@pytest.mark.parametrize("fb", ["CSR"] + EXTRA)
@pytest.mark.parametrize("fa", ["CSR"] + EXTRA)
def test_spgemm_indirect_hybrid_packed_operands(ctx, fa, fb):
    """ELL / hybrid operands (their zero slots add nothing), packed (AoS) and
    blocked-ELL operands: the same product as the dense f64 one."""
    m, k, n = 40, 31, 27
    ra, ca, va = random_coo(5, m, k, 0.2)
    rb, cb, vb = random_coo(6, k, n, 0.2)
    da = ctx.convert(ctx.from_coo(m, k, ra, ca, va), fa)
    db = ctx.convert(ctx.from_coo(k, n, rb, cb, vb), fb)
    got = ctx.spgemm(da, db).astype(np.float64)
    A = np.zeros((m, k)); A[ra, ca] = va
    B = np.zeros((k, n)); B[rb, cb] = vb
    bound = np.abs(A) @ np.abs(B)
    assert (np.abs(got - A @ B) <= TOL * bound + 1e-30).all(), (fa, fb)
