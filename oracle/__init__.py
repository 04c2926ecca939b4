"""CPU ORACLE — test infrastructure only.

ctypes front-ends for
  * ``Port``: the C restatement of the reference hot path (oracle/sfo.c,
    built to oracle/_build/libsfo.so), and
  * ``Ref``:  the unmodified reference headers behind a C-ABI shim
    (oracle/ref_shim.cpp, built to oracle/_ref/libsfref.so in the build
    container, where /root/reference exists).

Both expose the same methods, so parity checks read the same against either.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libsfo.so")
REF_SO = os.path.join(HERE, "_ref", "libsfref.so")

FORMATS = {"COO": 0, "CSR": 1, "CSC": 2, "DCSR": 3, "ELL": 4, "BCSR": 5}
SIZE, PTR, IDX, DENSE_VECTOR = 1, 2, 4, 8

# 1 + ErrorKind ordinal (errors.hpp:10-21)
ERROR_KINDS = [
    "Parse", "NonAffine", "NonIntegral", "UnsupportedSource", "UnsupportedHeader",
    "DuplicateCoordinate", "Collision", "InvalidOperation", "Singular", "Io",
]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        kind = ERROR_KINDS[status - 1] if 1 <= status <= len(ERROR_KINDS) else f"status{status}"
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.status = status


def build(quiet: bool = True) -> None:
    """Compile the port (and the reference shim when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{out.stdout}\n{out.stderr}")
    if not quiet:
        print(out.stdout)


P64 = C.POINTER(C.c_int64)
PF64 = C.POINTER(C.c_double)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(P64)


def _pf64(a: np.ndarray):
    return a.ctypes.data_as(PF64)


@dataclass
class Level:
    flags: int
    lo: int
    hi: int
    node_count: int
    idx: np.ndarray
    ptr: np.ndarray

    def explain(self) -> str:
        parts = [n for f, n in ((SIZE, "size"), (PTR, "ptr"), (IDX, "idx"),
                               (DENSE_VECTOR, "dense_vector")) if self.flags & f]
        return ", ".join(parts)


@dataclass
class Materialized:
    """Host copy of a MaterializedTensor (storage.hpp:77-91), int64 / f64."""
    fmt: str
    shape: tuple
    levels: list = field(default_factory=list)
    values: np.ndarray = None
    layout: tuple = None  # AoS span (aos_start, aos_end) of a packed format; None: SoA
    partitions: list = field(default_factory=list)  # Partition: (begin, end) value ranges

    def explain(self) -> str:
        text = " | ".join(f"L{i}: {lv.explain()}" for i, lv in enumerate(self.levels)) + " | val"
        text += f" | pack({self.layout[0]},{self.layout[1]})" if self.layout else ""
        return text + (" | partition(0)" if self.fmt.startswith("C2SR") else "")  # the one partitioned format


class _Coo:
    def __init__(self, lib, handle, prefix, shape):
        self._lib, self.h, self._p, self.shape = lib, handle, prefix, shape

    def __del__(self):
        try:
            getattr(self._lib, self._p + "coo_free")(self.h)
        except Exception:
            pass

    @property
    def nnz(self) -> int:
        return int(getattr(self._lib, self._p + "coo_nnz")(self.h))

    def arrays(self):
        n = self.nnz
        r, c, v = np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n, np.float64)
        getattr(self._lib, self._p + "coo_get")(self.h, _p64(r), _p64(c), _pf64(v))
        return r, c, v


class _Mat:
    def __init__(self, lib, handle, prefix, fmt, shape):
        self._lib, self.h, self._p, self.fmt, self.shape = lib, handle, prefix, fmt, shape

    def __del__(self):
        try:
            getattr(self._lib, self._p + "mat_free")(self.h)
        except Exception:
            pass

    def download(self) -> Materialized:
        f = lambda n: getattr(self._lib, self._p + n)
        out = Materialized(self.fmt, self.shape)
        for l in range(f("mat_nlevels")(self.h)):
            info = np.zeros(6, np.int64)
            f("mat_level_info")(self.h, l, _p64(info))
            idx, ptr = np.zeros(int(info[4]), np.int64), np.zeros(int(info[5]), np.int64)
            f("mat_level_idx")(self.h, l, _p64(idx))
            f("mat_level_ptr")(self.h, l, _p64(ptr))
            out.levels.append(Level(int(info[0]), int(info[1]), int(info[2]), int(info[3]), idx, ptr))
        vals = np.zeros(int(f("mat_nvals")(self.h)), np.float64)
        f("mat_values")(self.h, _pf64(vals))
        out.values = vals
        if hasattr(self._lib, self._p + "mat_layout"):  # the reference shim only
            lay = np.zeros(3, np.int64)
            f("mat_layout")(self.h, _p64(lay))
            if lay[0] == 1:
                out.layout = (int(lay[1]), int(lay[2]))
            np_ = int(f("mat_npartitions")(self.h))
            if np_:
                pr = np.zeros(2 * np_, np.int64)
                f("mat_partitions")(self.h, _p64(pr))
                out.partitions = [(int(pr[2 * i]), int(pr[2 * i + 1])) for i in range(np_)]
        return out


class _Base:
    prefix = ""
    so = ""

    def __init__(self):
        if not os.path.exists(self.so):
            raise FileNotFoundError(f"{self.so} missing: run oracle.build() / make -C oracle")
        self.lib = C.CDLL(self.so)
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p
        getattr(self.lib, self.prefix + "coo_nnz").restype = C.c_int64
        getattr(self.lib, self.prefix + "mat_nvals").restype = C.c_int64
        if hasattr(self.lib, self.prefix + "mat_npartitions"):
            getattr(self.lib, self.prefix + "mat_npartitions").restype = C.c_int64
        for n in ("coo_free", "mat_free"):
            getattr(self.lib, self.prefix + n).restype = None

    def _check(self, st):
        if st != 0:
            raise OracleError(st, getattr(self.lib, self.prefix + "last_error")().decode())

    def from_coo(self, m, n, row, col, val, sum_duplicates=False):
        row = np.ascontiguousarray(row, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        h = C.c_void_p()
        self._check(getattr(self.lib, self.prefix + "from_coo")(
            C.c_int64(m), C.c_int64(n), C.c_int64(len(val)), _p64(row), _p64(col), _pf64(val),
            C.c_int(1 if sum_duplicates else 0), C.byref(h)))
        return _Coo(self.lib, h, self.prefix, (m, n))

    def spmv(self, mat, x, threads=1):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(mat.shape[0], np.float64)
        self._check(self._spmv(mat, x, y, threads))
        return y

    def spmm(self, mat, b, threads=1):
        b = np.ascontiguousarray(b, np.float64)
        c = np.zeros((mat.shape[0], b.shape[1]), np.float64)
        self._check(self._spmm(mat, b, c, threads))
        return c

    def decompose_rows(self, coo, min_sum):
        s, r = C.c_void_p(), C.c_void_p()
        tot = np.zeros(coo.shape[0], np.int64)
        self._check(getattr(self.lib, self.prefix + "decompose_rows")(
            coo.h, C.c_int64(min_sum), C.byref(s), C.byref(r), _p64(tot)))
        return (_Coo(self.lib, s, self.prefix, coo.shape), _Coo(self.lib, r, self.prefix, coo.shape), tot)


def _fmt_text(fmt, r=None, c=None):
    if fmt == "BCSR":
        return f"BCSR({r},{c})"
    if fmt in ("BELL", "BDIA", "C2SR", "CISR", "CISR-plus"):  # formats.hpp:62-85: one argument
        return f"{fmt}({r})"
    if fmt == "CSB":  # formats.hpp:54-57: CSB(r, c)
        return f"CSB({r},{c})"
    return fmt


class Port(_Base):
    """The C restatement (oracle/sfo.c)."""
    prefix = "sfo_"
    so = PORT_SO

    def convert(self, coo, fmt, r=0, c=0):
        h = C.c_void_p()
        self._check(self.lib.sfo_convert(coo.h, C.c_int(FORMATS[fmt]), C.c_int64(r), C.c_int64(c),
                                         C.byref(h)))
        return _Mat(self.lib, h, self.prefix, _fmt_text(fmt, r, c), coo.shape)

    def _spmv(self, mat, x, y, threads):
        return self.lib.sfo_spmv(mat.h, _pf64(x), _pf64(y))

    def _spmm(self, mat, b, c, threads):
        return self.lib.sfo_spmm(mat.h, _pf64(b), C.c_int64(b.shape[1]), _pf64(c))

    # Synthetic inputs; identical to the GPU generators.
    def gen_uniform(self, seed, m, n, per_row):
        h = C.c_void_p()
        self._check(self.lib.sfo_gen_uniform(C.c_uint64(seed), C.c_int64(m), C.c_int64(n),
                                             C.c_int(per_row), C.byref(h)))
        return _Coo(self.lib, h, self.prefix, (m, n))

    def gen_rmat(self, seed, scale, edges):
        h = C.c_void_p()
        self._check(self.lib.sfo_gen_rmat(C.c_uint64(seed), C.c_int(scale), C.c_int64(edges),
                                          C.byref(h)))
        return _Coo(self.lib, h, self.prefix, (1 << scale, 1 << scale))

    def gen_hypersparse(self, seed, m, n, draws):
        h = C.c_void_p()
        self._check(self.lib.sfo_gen_hypersparse(C.c_uint64(seed), C.c_int64(m), C.c_int64(n),
                                                 C.c_int64(draws), C.byref(h)))
        return _Coo(self.lib, h, self.prefix, (m, n))

    def gen_block_sparse(self, seed, m, n, r, c, density):
        h = C.c_void_p()
        thresh = min(int(density * 2 ** 32), 2 ** 32 - 1)
        self._check(self.lib.sfo_gen_block_sparse(C.c_uint64(seed), C.c_int64(m), C.c_int64(n), C.c_int64(r),
                                                  C.c_int64(c), C.c_uint32(thresh), C.byref(h)))
        return _Coo(self.lib, h, self.prefix, (m, n))

    def gen_dense(self, seed, count):
        out = np.empty(count, np.float64)
        self.lib.sfo_gen_dense(C.c_uint64(seed), C.c_int64(count), _pf64(out))
        return out


class Ref(_Base):
    """The unmodified reference headers (oracle/_ref/libsfref.so)."""
    prefix = "sfr_"
    so = REF_SO

    def convert(self, coo, fmt, r=0, c=0):
        h = C.c_void_p()
        text = _fmt_text(fmt, r, c)
        self._check(self.lib.sfr_convert(coo.h, text.encode(), C.byref(h)))
        return _Mat(self.lib, h, self.prefix, text, coo.shape)

    def _spmv(self, mat, x, y, threads):
        return self.lib.sfr_spmv(mat.h, _pf64(x), _pf64(y), C.c_int(threads))

    def _spmm(self, mat, b, c, threads):
        return self.lib.sfr_spmm(mat.h, _pf64(b), C.c_int64(b.shape[1]), _pf64(c), C.c_int(threads))

    def convert_from(self, coo, mid, fmt, r=0, c=0, mr=0, mc=0):
        """A tensor first converted to `mid`, then from `mid` to `fmt`
        (convert_structure from a non-COO source, planner.hpp:95)."""
        h = C.c_void_p()
        text = _fmt_text(fmt, r, c)
        mtext = _fmt_text(mid, mr, mc)
        self._check(self.lib.sfr_convert_from(coo.h, mtext.encode(), text.encode(), C.byref(h)))
        return _Mat(self.lib, h, self.prefix, text, coo.shape)

    def spgemm(self, ma, mb):
        """run_kernel(spgemm_kernel(), {A, B}) -> (dense C f64, plan mode)."""
        c = np.zeros((ma.shape[0], mb.shape[1]), np.float64)
        buf = C.create_string_buffer(64)
        self._check(self.lib.sfr_spgemm(ma.h, mb.h, _pf64(c), buf, C.c_int64(64)))
        return c, buf.value.decode()

    def write_container(self, coo, fmt, path, r=0, c=0):
        """write_container (io.hpp:240) of the materialized `fmt` form."""
        self._check(self.lib.sfr_write_container(coo.h, _fmt_text(fmt, r, c).encode(), os.fsencode(path)))

    def read_mm(self, path, sum_duplicates=False):
        """read_matrix_market + from_coo (io.hpp:50, tensor.hpp:118)."""
        h = C.c_void_p()
        self._check(self.lib.sfr_read_mm(os.fsencode(path), C.c_int(1 if sum_duplicates else 0), C.byref(h)))
        m, n = C.c_int64(), C.c_int64()
        self.lib.sfr_coo_shape(h, C.byref(m), C.byref(n))
        return _Coo(self.lib, h, self.prefix, (m.value, n.value))

    def decompose_blocks(self, coo, r, c, min_sum):
        s, rem = C.c_void_p(), C.c_void_p()
        self._check(self.lib.sfr_decompose_blocks(coo.h, C.c_int64(r), C.c_int64(c), C.c_int64(min_sum),
                                                  C.byref(s), C.byref(rem)))
        return _Coo(self.lib, s, self.prefix, coo.shape), _Coo(self.lib, rem, self.prefix, coo.shape)

    def plan(self, src, dst):
        buf = C.create_string_buffer(4096)
        self._check(self.lib.sfr_plan(src.encode(), dst.encode(), buf, C.c_int64(4096)))
        return [l for l in buf.value.decode().split("\n") if l]

    def explain(self, fmt):
        buf = C.create_string_buffer(4096)
        self._check(self.lib.sfr_storage_explain(fmt.encode(), buf, C.c_int64(4096)))
        return buf.value.decode()


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def rel_error_bound(y_hat, y_ref, abs_sum):
    """|y_hat - y| <= tol * sum_j |a_ij| |x_j| (per output)."""
    err = np.abs(np.asarray(y_hat, np.float64) - y_ref)
    denom = np.maximum(abs_sum, np.finfo(np.float64).tiny)
    return float(np.max(err / denom)) if err.size else 0.0
