"""Shared helpers for the GPU parity tests (device path vs CPU oracle)."""
import numpy as np
import pytest

import paper_2403_05802_b200 as sfg

TOL = 1e-5  # north_star: SpMV/SpMM within 1e-5 relative (fp32 vs f64 oracle)


def assert_same_materialized(dev, ora, ctx=""):
    """Bit-exact: every level's storage flags, bounds, node count, idx, ptr,
    and the values (fp32 widened to f64 == the f64 oracle)."""
    assert len(dev.levels) == len(ora.levels), ctx
    for i, (a, b) in enumerate(zip(dev.levels, ora.levels)):
        assert (a.flags, a.lo, a.hi, a.node_count) == (b.flags, b.lo, b.hi, b.node_count), (ctx, i)
        np.testing.assert_array_equal(a.idx, b.idx, err_msg=f"{ctx} L{i} idx")
        np.testing.assert_array_equal(a.ptr, b.ptr, err_msg=f"{ctx} L{i} ptr")
    np.testing.assert_array_equal(dev.values, ora.values, err_msg=f"{ctx} values")


def check_spmv(y_dev, y_ref, bound, ctx=""):
    """|y_hat - y| <= 1e-5 * sum_j |a_ij||x_j| per row."""
    err = np.abs(y_dev.astype(np.float64) - y_ref)
    ok = err <= TOL * bound + 1e-30
    if not np.all(ok):
        i = int(np.argmax(err - TOL * bound))
        raise AssertionError(f"{ctx}: row {i} dev={y_dev[i]!r} ref={y_ref[i]!r} "
                             f"err={err[i]:.3e} bound={TOL * bound[i]:.3e}")


def dense_abs_bound(r, c, v, m, x):
    """sum_j |a_ij| |x_j| from COO arrays (numpy, f64)."""
    w = np.abs(np.asarray(v, np.float64)) * np.abs(x[np.asarray(c, np.int64)])
    return np.bincount(np.asarray(r, np.int64), weights=w, minlength=m)
