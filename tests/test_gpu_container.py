"""USPT container (io.hpp:202-334): files written from
device tensors are byte-identical to the unmodified reference's
write_container of the same materialized tensor, and reading a
reference-written file gives back the same tensor (bit-exact levels and
values)."""
import filecmp

import numpy as np
import pytest

import paper_2403_05802_b200 as sfg
from gpu_common import assert_same_materialized
from matrices import random_coo

pytestmark = pytest.mark.gpu

FORMATS = ["COO", "CSR", "CSC", "DCSR", "ELL", "BCSR(2,2)", "BCSR(4,3)"]


def ref_args(fmt):
    if fmt.startswith("BCSR"):
        r, c = (int(t) for t in fmt[5:-1].split(","))
        return "BCSR", r, c
    return fmt, 0, 0


@pytest.mark.parametrize("seed", [0, 1])
@pytest.mark.parametrize("fmt", FORMATS)
def test_container_matches_reference(ctx, ref, tmp_path, fmt, seed):
    m, n = [(37, 29), (64, 64)][seed]
    r, c, v = random_coo(seed, m, n, 0.2, zeros=0.1)
    v = np.asarray(v, np.float32).astype(np.float64)  # fp32-exact values: identical f64 payloads
    d = ctx.convert(ctx.from_coo(m, n, r, c, v), fmt)
    ours, theirs = tmp_path / "ours.uspt", tmp_path / "ref.uspt"
    ctx.write_container(d, str(ours))
    k, br, bc = ref_args(fmt)
    rc = ref.from_coo(m, n, r, c, v)
    ref.write_container(rc, k, str(theirs), br, bc)
    assert filecmp.cmp(ours, theirs, shallow=False), fmt
    back = ctx.read_container(str(theirs), fmt)
    assert_same_materialized(back.download(), d.download(), ("read", fmt))
    # and it computes: SpMV through the re-read tensor
    x = np.linspace(-1, 1, n).astype(np.float32)
    np.testing.assert_allclose(ctx.spmv(back, x), ctx.spmv(d, x), rtol=1e-6, atol=1e-6)


def test_container_errors(ctx, tmp_path):
    p = tmp_path / "bad.uspt"
    p.write_bytes(b"NOPE")
    with pytest.raises(sfg.SfgError) as ei:
        ctx.read_container(str(p), "CSR")
    assert ei.value.kind == "Io" and "bad magic" in str(ei.value)
    d = ctx.convert(ctx.from_coo(4, 4, [0, 1], [1, 2], [1.0, 2.0]), "CSR")
    ctx.write_container(d, str(p))
    raw = p.read_bytes()
    (tmp_path / "cut.uspt").write_bytes(raw[:-9])
    with pytest.raises(sfg.SfgError) as ei:
        ctx.read_container(str(tmp_path / "cut.uspt"), "CSR")
    assert ei.value.kind == "Io"
    with pytest.raises(sfg.SfgError) as ei:  # a CSR container read as COO
        ctx.read_container(str(p), "COO")
    assert ei.value.kind == "InvalidOperation"
    with pytest.raises(sfg.SfgError) as ei:
        ctx.read_container(str(tmp_path / "missing.uspt"), "CSR")
    assert ei.value.kind == "Io"
