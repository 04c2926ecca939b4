"""ctypes binding of the B200 sparse hot path (include/sparseforge_b200.h).

The product is the sm_100a library ``_lib/libsfg.so`` behind a C-ABI; this
module is a thin host binding used by the tests and bench.py. It never
computes anything itself: when the library (or a B200) is missing it raises.

    import paper_2403_05802_b200 as sfg
    ctx = sfg.Context(0)
    coo = ctx.from_coo(m, n, rows, cols, vals)          # from_coo (tensor.hpp:118)
    csr = ctx.convert(coo, "CSR")                        # convert_structure + materialize
    y   = ctx.spmv(csr, x)                               # run_kernel(spmv_kernel(), ...)
"""
from __future__ import annotations

import ctypes as C
import weakref
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libsfg.so")

KINDS = {"COO": 0, "CSR": 1, "CSC": 2, "DCSR": 3, "ELL": 4, "BCSR": 5, "HYB": 6, "DOK": 7, "LIL": 8, "BELL": 9, "DIA": 10, "CSB": 11, "BDIA": 12, "C2SR": 13, "HBELL": 14, "DCSC": 15,
         "DIA-variant": 16, "CISR": 17, "CISR-plus": 18}
KIND_NAMES = {v: k for k, v in KINDS.items()}
F32, BF16 = 0, 1
FLAG_SORTED, FLAG_SUM_DUPLICATES, FLAG_HOST = 1, 2, 4
COMPUTE_HOST, COMPUTE_ACCUMULATE = 1, 2
COMM_ID_BYTES, ROWPART_GATHER = 128, 1
ERROR_KINDS = ["Parse", "NonAffine", "NonIntegral", "UnsupportedSource", "UnsupportedHeader",
               "DuplicateCoordinate", "Collision", "InvalidOperation", "Singular", "Io"]


class SfgError(RuntimeError):
    """Status from the C-ABI: ``kind`` is the reference ErrorKind name
    (errors.hpp:10-21) or "Cuda" / "OutOfMemory" / "Nccl"."""

    def __init__(self, status, msg):
        if 1 <= status <= 10:
            kind = ERROR_KINDS[status - 1]
        else:
            kind = {64: "Cuda", 65: "OutOfMemory", 66: "Nccl"}.get(status, f"status{status}")
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.status = status


class Format(C.Structure):
    _fields_ = [("kind", C.c_int32), ("block_r", C.c_int32), ("block_c", C.c_int32),
                ("value_dtype", C.c_int32), ("threshold", C.c_int64)]


class LevelView(C.Structure):
    _fields_ = [("storage", C.c_uint32), ("lo", C.c_int64), ("hi", C.c_int64),
                ("node_count", C.c_int64), ("idx_len", C.c_int64), ("ptr_len", C.c_int64),
                ("idx", C.c_void_p), ("ptr", C.c_void_p)]


class TensorView(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value_dtype", C.c_int32), ("rows", C.c_int64),
                ("cols", C.c_int64), ("nlevels", C.c_int32), ("level", LevelView * 5),
                ("nvals", C.c_int64), ("values", C.c_void_p), ("parts", C.c_void_p * 2),
                ("layout", C.c_int32), ("aos_start", C.c_int32), ("aos_end", C.c_int32),
                ("record_words", C.c_int32), ("npartitions", C.c_int64),
                ("partitions", C.POINTER(C.c_int64))]


@dataclass
class Level:
    """MaterializedLevel (storage.hpp:77-83) on the host."""
    flags: int
    lo: int
    hi: int
    node_count: int
    idx: np.ndarray
    ptr: np.ndarray

    def explain(self) -> str:
        names = ((1, "size"), (2, "ptr"), (4, "idx"), (8, "dense_vector"))
        return ", ".join(n for f, n in names if self.flags & f)


@dataclass
class Materialized:
    """MaterializedTensor (storage.hpp:85-91) on the host."""
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


_lib = None


def load():
    """Load libsfg.so; fails loudly if it was not built (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: the CUDA extension is not built "
                          "(run __graft_entry__.build() or `make lib`)")
    lib = C.CDLL(LIB_PATH)
    vp, i64, i32, u32 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint32
    pp = C.POINTER(C.c_void_p)
    sig = {
        "sfg_last_error": (C.c_char_p, []),
        "sfg_context_create": (C.c_int, [C.c_int, vp, pp]),
        "sfg_context_set_stream": (C.c_int, [vp, vp]),
        "sfg_context_destroy": (C.c_int, [vp]),
        "sfg_context_synchronize": (C.c_int, [vp]),
        "sfg_context_release_cached": (C.c_int, [vp, C.POINTER(i64)]),
        "sfg_format_resolve": (C.c_int, [C.c_char_p, C.POINTER(Format)]),
        "sfg_plan_text": (C.c_int, [C.POINTER(Format), C.POINTER(Format), C.c_char_p, i64]),
        "sfg_storage_explain": (C.c_int, [C.POINTER(Format), C.c_char_p, i64]),
        "sfg_from_coo": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, u32, pp]),
        "sfg_convert": (C.c_int, [vp, vp, C.POINTER(Format), pp]),
        "sfg_decompose_rows": (C.c_int, [vp, vp, i64, pp, pp, vp]),
        "sfg_decompose_blocks": (C.c_int, [vp, vp, i64, i64, i64, pp, pp]),
        "sfg_tensor_view_get": (C.c_int, [vp, vp, C.POINTER(TensorView)]),
        "sfg_tensor_free": (C.c_int, [vp]),
        "sfg_spmv": (C.c_int, [vp, vp, vp, vp, u32]),
        "sfg_spmm": (C.c_int, [vp, vp, vp, i32, i64, i64, vp, i64, u32]),
        "sfg_row_partition": (C.c_int, [vp, vp, i32, C.POINTER(C.c_int64)]),
        "sfg_coo_slice_rows": (C.c_int, [vp, vp, i64, i64, pp]),
        "sfgx_row_bounds_host": (C.c_int, [vp, i64, i64, i32, C.POINTER(C.c_int64)]),
        "sfg_read_matrix_market": (C.c_int, [vp, C.c_char_p, u32, pp]),
        "sfg_write_container": (C.c_int, [vp, vp, C.c_char_p]),
        "sfg_spgemm": (C.c_int, [vp, vp, vp, vp, i64, u32]),
        "sfg_read_container": (C.c_int, [vp, C.c_char_p, C.POINTER(Format), pp]),
        "sfg_comm_unique_id": (C.c_int, [vp]),
        "sfg_comm_create": (C.c_int, [vp, i32, i32, vp, pp]),
        "sfg_comm_destroy": (C.c_int, [vp]),
        "sfg_rowpart_spmv": (C.c_int, [vp, vp, vp, vp, vp, i64, u32]),
        "sfg_rowpart_spmm": (C.c_int, [vp, vp, vp, vp, i32, i64, i64, vp, i64, u32]),
        "sfg_allgather_chunks": (C.c_int, [vp, vp, vp, i64]),
        "sfgx_gen_uniform": (C.c_int, [vp, C.c_uint64, i64, i64, i32, pp]),
        "sfgx_gen_rmat": (C.c_int, [vp, C.c_uint64, i32, i64, pp]),
        "sfgx_gen_hypersparse": (C.c_int, [vp, C.c_uint64, i64, i64, i64, pp]),
        "sfgx_gen_dense": (C.c_int, [vp, C.c_uint64, i64, vp]),
        "sfgx_gen_block_sparse": (C.c_int, [vp, C.c_uint64, i64, i64, i32, i32, u32, i32, pp]),
        "sfgx_launch_count": (i64, []),
        "sfgx_device_alloc": (C.c_int, [vp, i64, pp]),
        "sfgx_device_free": (C.c_int, [vp, vp]),
        "sfgx_copy": (C.c_int, [vp, vp, vp, i64, i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(st):
    if st != 0:
        raise SfgError(st, _lib.sfg_last_error().decode(errors="replace"))


def row_bounds_host(rows: np.ndarray, m: int, parts: int) -> list[int]:
    """The library's nnz-balanced row split (sfgx_row_bounds_host, the rule
    sfg_row_partition applies on the device) over a host array of the
    row-sorted COO's rows; no GPU needed."""
    lib = load()
    rows = np.ascontiguousarray(rows, np.int32)
    b = (C.c_int64 * (parts + 1))()
    _check(lib.sfgx_row_bounds_host(rows.ctypes.data_as(C.c_void_p), len(rows), m, parts, b))
    return list(b)


def comm_unique_id() -> bytes:
    """ncclGetUniqueId through the C-ABI (rank 0 of the row-partitioned path)."""
    lib = load()
    buf = C.create_string_buffer(COMM_ID_BYTES)
    _check(lib.sfg_comm_unique_id(buf))
    return buf.raw


class Comm:
    """Owns an sfg_comm (NCCL communicator) handle."""

    def __init__(self, h, nranks, rank):
        self.h, self.nranks, self.rank = h, nranks, rank

    def close(self):
        if self.h:
            _lib.sfg_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def resolve_format(text: str) -> Format:
    lib = load()
    f = Format()
    _check(lib.sfg_format_resolve(text.encode(), C.byref(f)))
    return f


def plan_lines(src: str, dst: str):
    lib = load()
    buf = C.create_string_buffer(4096)
    s, d = resolve_format(src), resolve_format(dst)
    _check(lib.sfg_plan_text(C.byref(s), C.byref(d), buf, 4096))
    return [l for l in buf.value.decode().split("\n") if l]


def storage_explain(fmt: str) -> str:
    lib = load()
    buf = C.create_string_buffer(4096)
    f = resolve_format(fmt)
    _check(lib.sfg_storage_explain(C.byref(f), buf, 4096))
    return buf.value.decode()


def launch_count() -> int:
    return int(load().sfgx_launch_count())


class DeviceBuffer:
    """Device allocation owned by a context (stream-ordered)."""

    def __init__(self, ctx: "Context", nbytes: int):
        self.ctx, self.nbytes = ctx, int(nbytes)
        p = C.c_void_p()
        _check(ctx.lib.sfgx_device_alloc(ctx.h, self.nbytes, C.byref(p)))
        self.ptr = p.value

    def free(self):
        if self.ptr:
            self.ctx.lib.sfgx_device_free(self.ctx.h, C.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def upload(self, arr: np.ndarray):
        arr = np.ascontiguousarray(arr)
        assert arr.nbytes <= self.nbytes
        _check(self.ctx.lib.sfgx_copy(self.ctx.h, C.c_void_p(self.ptr), arr.ctypes.data_as(C.c_void_p),
                                      arr.nbytes, 0))
        return self

    def download(self, dtype, count, offset=0) -> np.ndarray:
        """`count` elements from element `offset` on."""
        out = np.empty(int(count), dtype)
        if out.nbytes:
            _check(self.ctx.lib.sfgx_copy(self.ctx.h, out.ctypes.data_as(C.c_void_p),
                                          C.c_void_p(self.ptr + int(offset) * out.itemsize), out.nbytes, 1))
        return out


class Tensor:
    """A device-resident materialized tensor (sfg_tensor handle)."""

    def __init__(self, ctx: "Context", handle, owned=True):
        self.ctx, self.h, self.owned = ctx, handle, owned
        if owned and handle:
            ctx._live.add(self)

    def free(self):
        """Release the device arrays now (also done when collected, and by
        Context.close for tensors still alive then)."""
        if self.owned and self.h and self.ctx.h:
            self.ctx.lib.sfg_tensor_free(self.h)
        self.h = None
        self.ctx._live.discard(self)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def view(self) -> TensorView:
        v = TensorView()
        _check(self.ctx.lib.sfg_tensor_view_get(self.ctx.h, self.h, C.byref(v)))
        return v

    @property
    def kind(self) -> str:
        return KIND_NAMES[self.view().kind]

    @property
    def shape(self):
        v = self.view()
        return (v.rows, v.cols)

    def parts(self):
        v = self.view()
        out = [Tensor(self.ctx, C.c_void_p(p), owned=False) for p in v.parts if p]
        for t in out:
            t._parent = self  # the parts live in (and die with) this tensor
        return out

    def _dl(self, ptr, dtype, count, stride=1):
        """count elements from device pointer ptr, element i at ptr[i * stride]
        (stride > 1: a field of packed records)."""
        out = np.empty(int(count) * int(stride), dtype)
        nbytes = (int(count) - 1) * int(stride) * out.itemsize + out.itemsize if count else 0
        if nbytes:
            _check(self.ctx.lib.sfgx_copy(self.ctx.h, out.ctypes.data_as(C.c_void_p), C.c_void_p(ptr),
                                          nbytes, 1))
        return np.ascontiguousarray(out[::int(stride)][:int(count)])

    def download(self):
        """Host copy shaped like the reference MaterializedTensor
        (storage.hpp:77-91): int64 idx/ptr and f64 values, field for field
        the layout the oracle returns."""
        v = self.view()
        out = Materialized(KIND_NAMES[v.kind], (v.rows, v.cols))
        rw = v.record_words if v.layout == 1 else 1
        if v.layout == 1:
            out.layout = (int(v.aos_start), int(v.aos_end))
        for i in range(v.nlevels):
            lv = v.level[i]
            packed = v.layout == 1 and v.aos_start <= i <= v.aos_end
            idx = self._dl(lv.idx, np.int32, lv.idx_len, rw if packed else 1).astype(np.int64)
            ptr = self._dl(lv.ptr, np.int32, lv.ptr_len).astype(np.int64)
            out.levels.append(Level(int(lv.storage), int(lv.lo), int(lv.hi),
                                           int(lv.node_count), idx, ptr))
        if v.value_dtype == BF16:
            raw = self._dl(v.values, np.uint16, v.nvals).astype(np.uint32) << 16
            out.values = raw.view(np.float32).astype(np.float64)
        else:
            out.values = self._dl(v.values, np.float32, v.nvals, rw).astype(np.float64)
        if v.npartitions:
            out.partitions = [(int(v.partitions[2 * i]), int(v.partitions[2 * i + 1])) for i in range(v.npartitions)]
        return out

    def coo_arrays(self):
        v = self.view()
        assert v.kind == KINDS["COO"]
        return (self._dl(v.level[0].idx, np.int32, v.level[0].idx_len),
                self._dl(v.level[1].idx, np.int32, v.level[1].idx_len),
                self._dl(v.values, np.float32, v.nvals))


class Context:
    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = load()
        h = C.c_void_p()
        self._live = weakref.WeakSet()  # owned tensors: freed before the context goes
        _check(self.lib.sfg_context_create(device, C.c_void_p(stream or 0), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            # a tensor collected after this point must not touch the deleted
            # context: free the live ones now, their handles become null
            for t in list(self._live):
                t.free()
            self.lib.sfg_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: int):
        _check(self.lib.sfg_context_set_stream(self.h, C.c_void_p(stream)))

    def synchronize(self):
        _check(self.lib.sfg_context_synchronize(self.h))

    def release_cached(self) -> int:
        """Return the context's cached device blocks to the driver pool;
        returns how many bytes were cached."""
        b = C.c_int64()
        _check(self.lib.sfg_context_release_cached(self.h, C.byref(b)))
        return b.value

    def buffer(self, nbytes) -> DeviceBuffer:
        return DeviceBuffer(self, nbytes)

    # ---------------------------------------------------------------- ingest
    def from_coo(self, m, n, row, col, val, sorted=False, sum_duplicates=False) -> Tensor:
        """from_coo (tensor.hpp:118) from host arrays."""
        row = np.ascontiguousarray(row, np.int32)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float32)
        flags = FLAG_HOST | (FLAG_SORTED if sorted else 0) | (FLAG_SUM_DUPLICATES if sum_duplicates else 0)
        h = C.c_void_p()
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        _check(self.lib.sfg_from_coo(self.h, m, n, len(val), vp(row), vp(col), vp(val), flags, C.byref(h)))
        return Tensor(self, h)

    def download_ptr(self, ptr: int, dtype, count, offset=0) -> np.ndarray:
        """Host copy of `count` elements at device address ptr + offset elements."""
        out = np.empty(int(count), dtype)
        if out.nbytes:
            _check(self.lib.sfgx_copy(self.h, out.ctypes.data_as(C.c_void_p),
                                      C.c_void_p(int(ptr) + int(offset) * out.itemsize), out.nbytes, 1))
        return out

    def copy_device(self, dst_ptr: int, src_ptr: int, nbytes: int):
        """Device-to-device copy on the context's stream."""
        _check(self.lib.sfgx_copy(self.h, C.c_void_p(dst_ptr), C.c_void_p(src_ptr), nbytes, 2))

    def from_coo_device(self, m, n, nnz, row_ptr, col_ptr, val_ptr, flags=0) -> Tensor:
        h = C.c_void_p()
        _check(self.lib.sfg_from_coo(self.h, m, n, nnz, C.c_void_p(row_ptr), C.c_void_p(col_ptr),
                                     C.c_void_p(val_ptr), flags, C.byref(h)))
        return Tensor(self, h)

    # ------------------------------------------------------------ conversion
    def convert(self, src: Tensor, fmt: str, value_dtype: int = F32) -> Tensor:
        f = resolve_format(fmt)
        f.value_dtype = value_dtype
        h = C.c_void_p()
        _check(self.lib.sfg_convert(self.h, src.h, C.byref(f), C.byref(h)))
        return Tensor(self, h)

    def decompose_rows(self, coo: Tensor, min_sum: int, totals_ptr: int = 0):
        s, r = C.c_void_p(), C.c_void_p()
        _check(self.lib.sfg_decompose_rows(self.h, coo.h, min_sum, C.byref(s), C.byref(r),
                                           C.c_void_p(totals_ptr)))
        return Tensor(self, s), Tensor(self, r)

    def decompose_blocks(self, coo: Tensor, r: int, c: int, min_sum: int):
        """decompose by r x c blocks (the block count rule): (selected, remainder)."""
        s, rem = C.c_void_p(), C.c_void_p()
        _check(self.lib.sfg_decompose_blocks(self.h, coo.h, r, c, min_sum, C.byref(s), C.byref(rem)))
        return Tensor(self, s), Tensor(self, rem)

    def row_partition(self, coo: Tensor, parts: int):
        b = (C.c_int64 * (parts + 1))()
        _check(self.lib.sfg_row_partition(self.h, coo.h, parts, b))
        return list(b)

    def read_matrix_market(self, path: str, sum_duplicates: bool = False) -> Tensor:
        """read_matrix_market + from_coo (io.hpp:50, tensor.hpp:118), parsed
        on the device."""
        h = C.c_void_p()
        _check(self.lib.sfg_read_matrix_market(self.h, os.fsencode(path),
                                               FLAG_SUM_DUPLICATES if sum_duplicates else 0, C.byref(h)))
        return Tensor(self, h)

    def spgemm(self, a: Tensor, b: Tensor) -> np.ndarray:
        """Dense C = A B over two sparse operands (run_kernel(spgemm_kernel(),
        {A, B}), kernel.hpp:424); host result."""
        m, n = a.shape[0], b.shape[1]
        c = np.zeros((m, n), np.float32)
        _check(self.lib.sfg_spgemm(self.h, a.h, b.h, c.ctypes.data_as(C.c_void_p), n, COMPUTE_HOST))
        return c

    def spgemm_device(self, a: Tensor, b: Tensor, c_ptr: int, ldc=None, accumulate=False):
        _check(self.lib.sfg_spgemm(self.h, a.h, b.h, C.c_void_p(c_ptr), ldc or b.shape[1],
                                   COMPUTE_ACCUMULATE if accumulate else 0))

    def write_container(self, t: Tensor, path: str):
        """write_container (io.hpp:240): the USPT file of t's levels."""
        _check(self.lib.sfg_write_container(self.h, t.h, os.fsencode(path)))

    def read_container(self, path: str, fmt: str | None = None, value_dtype: int = F32) -> Tensor:
        """read_container (io.hpp:279) into a device tensor of format `fmt`
        (None: the format the stored levels and layout tag name)."""
        h = C.c_void_p()
        if fmt is None:
            _check(self.lib.sfg_read_container(self.h, os.fsencode(path), None, C.byref(h)))
        else:
            f = resolve_format(fmt)
            f.value_dtype = value_dtype
            _check(self.lib.sfg_read_container(self.h, os.fsencode(path), C.byref(f), C.byref(h)))
        return Tensor(self, h)

    def slice_rows(self, coo: Tensor, r0: int, r1: int) -> Tensor:
        h = C.c_void_p()
        _check(self.lib.sfg_coo_slice_rows(self.h, coo.h, r0, r1, C.byref(h)))
        return Tensor(self, h)

    # ------------------------------------------- row-partitioned multi-GPU
    def comm_create(self, nranks: int, rank: int, unique_id: bytes) -> "Comm":
        """NCCL communicator of the row-partitioned path (sfg_comm_create);
        `unique_id` from comm_unique_id() on rank 0, shared by any channel."""
        assert len(unique_id) == COMM_ID_BYTES
        h = C.c_void_p()
        buf = C.create_string_buffer(unique_id, COMM_ID_BYTES)
        _check(self.lib.sfg_comm_create(self.h, nranks, rank, buf, C.byref(h)))
        return Comm(h, nranks, rank)

    def rowpart_spmv(self, comm: "Comm", a_block: Tensor, x_ptr: int, y_ptr: int, chunk_rows: int,
                     gather=True):
        """y chunk `rank` = A_block x, then the in-place all-gather of the
        P chunks (sfg_rowpart_spmv)."""
        _check(self.lib.sfg_rowpart_spmv(self.h, comm.h, a_block.h, C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                         chunk_rows, ROWPART_GATHER if gather else 0))

    def rowpart_spmm(self, comm: "Comm", a_block: Tensor, b_ptr: int, b_dtype: int, nd: int, c_ptr: int,
                     chunk_rows: int, ldb=None, gather=True):
        _check(self.lib.sfg_rowpart_spmm(self.h, comm.h, a_block.h, C.c_void_p(b_ptr), b_dtype, nd, ldb or nd,
                                         C.c_void_p(c_ptr), chunk_rows, ROWPART_GATHER if gather else 0))

    def allgather_chunks(self, comm: "Comm", buf_ptr: int, chunk_elems: int):
        _check(self.lib.sfg_allgather_chunks(self.h, comm.h, C.c_void_p(buf_ptr), chunk_elems))

    # --------------------------------------------------------------- compute
    def spmv(self, a: Tensor, x: np.ndarray) -> np.ndarray:
        """y = A x from host x (copies inside, like the reference API)."""
        x = np.ascontiguousarray(x, np.float32)
        y = np.zeros(a.shape[0], np.float32)
        _check(self.lib.sfg_spmv(self.h, a.h, x.ctypes.data_as(C.c_void_p),
                                 y.ctypes.data_as(C.c_void_p), COMPUTE_HOST))
        return y

    def spmv_device(self, a: Tensor, x_ptr: int, y_ptr: int, accumulate=False):
        _check(self.lib.sfg_spmv(self.h, a.h, C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                 COMPUTE_ACCUMULATE if accumulate else 0))

    def spmm(self, a: Tensor, b: np.ndarray, b_dtype=F32) -> np.ndarray:
        if b_dtype == F32:
            b = np.ascontiguousarray(b, np.float32)
        else:
            b = np.ascontiguousarray(b, np.uint16)  # raw bf16 bits
        nd = b.shape[1]
        c = np.zeros((a.shape[0], nd), np.float32)
        _check(self.lib.sfg_spmm(self.h, a.h, b.ctypes.data_as(C.c_void_p), b_dtype, nd, nd,
                                 c.ctypes.data_as(C.c_void_p), nd, COMPUTE_HOST))
        return c

    def spmm_device(self, a: Tensor, b_ptr: int, b_dtype: int, nd: int, c_ptr: int,
                    ldb=None, ldc=None, accumulate=False):
        _check(self.lib.sfg_spmm(self.h, a.h, C.c_void_p(b_ptr), b_dtype, nd, ldb or nd,
                                 C.c_void_p(c_ptr), ldc or nd, COMPUTE_ACCUMULATE if accumulate else 0))

    # ------------------------------------------------------------ generators
    def gen_uniform(self, seed, m, n, per_row) -> Tensor:
        h = C.c_void_p()
        _check(self.lib.sfgx_gen_uniform(self.h, seed, m, n, per_row, C.byref(h)))
        return Tensor(self, h)

    def gen_rmat(self, seed, scale, edges) -> Tensor:
        h = C.c_void_p()
        _check(self.lib.sfgx_gen_rmat(self.h, seed, scale, edges, C.byref(h)))
        return Tensor(self, h)

    def gen_hypersparse(self, seed, m, n, draws) -> Tensor:
        h = C.c_void_p()
        _check(self.lib.sfgx_gen_hypersparse(self.h, seed, m, n, draws, C.byref(h)))
        return Tensor(self, h)

    def gen_block_sparse(self, seed, m, n, r, c, density, value_dtype=F32) -> Tensor:
        h = C.c_void_p()
        thresh = min(int(density * 2 ** 32), 2 ** 32 - 1)
        _check(self.lib.sfgx_gen_block_sparse(self.h, seed, m, n, r, c, thresh, value_dtype, C.byref(h)))
        return Tensor(self, h)

    def gen_dense(self, seed, count, out_ptr):
        _check(self.lib.sfgx_gen_dense(self.h, seed, count, C.c_void_p(out_ptr)))
