// container.cu — the USPT binary container:
// write_container / read_container (io.hpp:202-334) for device tensors.
//
// Layout (little-endian): "USPT", u16 version 1, u8 rank, i64 extents,
// u8 level count, per level {u8 kind (1 size, 2 idx, 4 ptr, 8 dense
// vector), i64 lo, i64 hi, u64 n + i64 idx[n], u64 n + i64 ptr[n]}, u64 n +
// f64 values[n], u8 layout tag (0 SoA), u32 partition count (0 here).
//
// The device widens the int32 index arrays and the fp32 / bf16 values to
// the container's i64 / f64 in aligned device buffers; each lands in pinned
// staging at its (unaligned) file offset with one D2H copy, the small
// headers are filled on the host, and the file is written with parallel
// pwrites. Reading goes the other way: parallel preads, host header walk,
// H2D of each payload, narrowing kernels (range-checked indices).
// Tensors written here are byte-identical to the reference's
// write_container of the same materialized tensor (tests/test_gpu_container.py).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include <cuda_bf16.h>

#include "devutil.cuh"
#include "internal.cuh"

extern "C" int sfg_tensor_view_get(sfg_context* ctx, const sfg_tensor* t, sfg_tensor_view* out);

namespace sfg {

namespace {

constexpr int kBlock = 256;
constexpr uint8_t kUSize = 1, kUIdx = 2, kUPtr = 4, kUDense = 8;

__global__ void k_widen_i32(const int32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

template <typename T>
__global__ void k_widen_val(const T* __restrict__ in, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)(float)in[i];
}

__global__ void k_narrow_i64(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out,
                             int* __restrict__ bad) {
  bool b = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = in[i];
    b |= v < INT32_MIN || v > INT32_MAX;
    out[i] = (int32_t)v;
  }
  if (__any_sync(kFull, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

template <typename T>
__global__ void k_narrow_val(const double* __restrict__ in, int64_t n, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)(float)in[i];
}

template <>
__global__ void k_narrow_val<__nv_bfloat16>(const double* __restrict__ in, int64_t n, __nv_bfloat16* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn((float)in[i]);
}

void put(std::vector<uint8_t>& b, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) b.push_back((uint8_t)(v >> (8 * i)));
}

uint8_t usp_kind(uint32_t storage) {
  uint8_t k = 0;
  if (storage & SFG_LEVEL_SIZE) k |= kUSize;
  if (storage & SFG_LEVEL_IDX) k |= kUIdx;
  if (storage & SFG_LEVEL_PTR) k |= kUPtr;
  if (storage & SFG_LEVEL_DENSE_VECTOR) k |= kUDense;
  return k;
}

// The expected level kinds of each format (storage.hpp:97-234 as materialized).
std::vector<uint8_t> expected_kinds(int kind) {
  switch (kind) {
    case SFG_COO: return {kUIdx, kUIdx};
    case SFG_CSR:
    case SFG_CSC: return {kUSize, kUIdx | kUPtr};
    case SFG_DCSR:
    case SFG_DCSC: return {kUIdx, kUIdx | kUPtr};  // (DCSC: read with the format given)
    case SFG_ELL: return {kUIdx, kUSize, kUIdx};
    case SFG_BCSR: return {kUSize, kUIdx | kUPtr, kUSize | kUDense, kUSize | kUDense};
    case SFG_BELL: return {kUIdx, kUSize, kUIdx, kUSize | kUDense, kUSize | kUDense};
    case SFG_DIA:
    case SFG_DIAV: return {kUIdx, kUSize | kUDense};  // (DIA-variant: read with the format given)
    case SFG_BDIA: return {kUSize, kUIdx | kUPtr, kUSize | kUDense};
    case SFG_C2SR: return {kUSize, kUSize, kUIdx | kUPtr};
    case SFG_CISR:
    case SFG_CISRP: return {kUIdx, kUIdx | kUPtr, kUIdx | kUPtr};  // (-plus: read with the format given)
    case SFG_CSB: return {kUSize, kUSize, kUIdx | kUPtr, kUIdx};
    case SFG_DOK: return {kUIdx, kUIdx};           // COO + pack(0,1)
    case SFG_LIL: return {kUSize, kUIdx | kUPtr};  // CSR + pack(0,1)
  }
  return {};
}

void write_all(const std::string& path, const char* data, int64_t size) {
  const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) raise(SFG_ERR_IO, "cannot write " + path);
  constexpr int64_t kChunk = 32 << 20;
  const int64_t nchunks = (size + kChunk - 1) / kChunk;
  std::atomic<int64_t> next{0};
  std::atomic<bool> bad{false};
  std::vector<std::thread> pool;
  for (int w = 0; w < (int)std::min<int64_t>(std::max<int64_t>(nchunks, 1), 8); ++w)
    pool.emplace_back([&] {
      for (int64_t k = next++; k < nchunks; k = next++) {
        const int64_t off = k * kChunk, len = std::min(kChunk, size - off);
        int64_t done = 0;
        while (done < len) {
          ssize_t put = ::pwrite(fd, data + off + done, (size_t)(len - done), off + done);
          if (put <= 0) {
            bad = true;
            return;
          }
          done += put;
        }
      }
    });
  for (auto& t : pool) t.join();
  if (::close(fd) != 0 || bad) raise(SFG_ERR_IO, "write failed: " + path);
}

}  // namespace

void write_container(sfg_context* ctx, const sfg_tensor* t, const char* path_c) {
  const std::string path(path_c);
  if (t->kind == SFG_HYB || t->kind == SFG_HBELL) raise(SFG_ERR_INVALID_OPERATION, "the hybrid pair is two tensors: write each part");
  sfg_tensor_view v;
  if (int st = sfg_tensor_view_get(ctx, t, &v)) raise(st, "tensor view");
  // a packed (AoS) tensor is written like its SoA base plus the layout tag
  // (io.hpp:262-268): its records are split into plain arrays first
  const void* values = t->val;
  int32_t *ur = nullptr, *ui = nullptr;
  float* uv = nullptr;
  struct Unpacked {
    sfg_context* ctx;
    std::vector<void*> p;
    ~Unpacked() {
      for (void* q : p) dfree(ctx, q);
    }
  } unpacked{ctx, {}};
  if (v.layout == 1) {
    aos_unpack(ctx, t, &ur, &ui, &uv);
    unpacked.p = {ur, ui, uv};
    if (t->kind == SFG_DOK) v.level[0].idx = ur;
    v.level[1].idx = ui;
    values = uv;
  }
  // layout: header bytes per piece, payload offsets
  struct Piece {
    int64_t off, n;
    const int32_t* src;
  };
  std::vector<uint8_t> head;
  std::vector<std::pair<int64_t, std::vector<uint8_t>>> heads;  // (offset, bytes)
  std::vector<Piece> arrays;
  int64_t off = 0;
  auto emit = [&](std::vector<uint8_t>& h) {
    heads.push_back({off, h});
    off += (int64_t)h.size();
    h.clear();
  };
  head.insert(head.end(), {'U', 'S', 'P', 'T'});
  put(head, 1, 2);
  put(head, 2, 1);
  put(head, (uint64_t)t->m, 8);
  put(head, (uint64_t)t->n, 8);
  put(head, (uint64_t)v.nlevels, 1);
  for (int l = 0; l < v.nlevels; ++l) {
    const sfg_level_view& lv = v.level[l];
    put(head, usp_kind(lv.storage), 1);
    put(head, (uint64_t)lv.lo, 8);
    put(head, (uint64_t)lv.hi, 8);
    put(head, (uint64_t)lv.idx_len, 8);
    emit(head);
    arrays.push_back({off, lv.idx_len, lv.idx});
    off += 8 * lv.idx_len;
    put(head, (uint64_t)lv.ptr_len, 8);
    emit(head);
    arrays.push_back({off, lv.ptr_len, lv.ptr});
    off += 8 * lv.ptr_len;
  }
  put(head, (uint64_t)v.nvals, 8);
  emit(head);
  const int64_t voff = off;
  off += 8 * v.nvals;
  if (v.layout == 1) {  // AoS over levels [aos_start, aos_end]
    put(head, 1, 1);
    put(head, (uint64_t)v.aos_start, 1);
    put(head, (uint64_t)v.aos_end, 1);
  } else {
    put(head, 0, 1);  // SoA
  }
  put(head, (uint64_t)v.npartitions, 4);  // partitions: (begin, end) value ranges
  for (int64_t q = 0; q < 2 * v.npartitions; ++q) put(head, (uint64_t)v.partitions[q], 8);
  emit(head);
  const int64_t size = off;

  if ((size_t)size + 1 > ctx->staging_bytes) {
    cudaStreamSynchronize(ctx->stream);
    if (ctx->staging) cudaFreeHost(ctx->staging);
    ctx->staging = nullptr;
    ctx->staging_bytes = 0;
    const size_t want = (size_t)size + 1 + ((size_t)size >> 3);
    if (cudaMallocHost(&ctx->staging, want) != cudaSuccess) {
      cudaGetLastError();
      raise(SFG_ERR_OOM, "pinned staging of " + std::to_string(want) + " bytes failed");
    }
    ctx->staging_bytes = want;
  } else {
    cudaStreamSynchronize(ctx->stream);
  }
  char* host = ctx->staging;
  // payloads: widen on the device, copy to their file offsets
  int64_t maxn = v.nvals;
  for (auto& a : arrays) maxn = std::max(maxn, a.n);
  std::vector<void*> temps;
  try {
    for (auto& a : arrays) {
      if (a.n == 0) continue;
      auto* w = dalloc_n<int64_t>(ctx, a.n);
      temps.push_back(w);
      SFG_LAUNCH(k_widen_i32, stream_grid(ctx, a.n, kBlock, 4, 8), kBlock, 0, ctx->stream, a.src, a.n, w);
      SFG_CUDA(cudaMemcpyAsync(host + a.off, w, 8 * a.n, cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (v.nvals) {
      auto* w = dalloc_n<double>(ctx, v.nvals);
      temps.push_back(w);
      if (t->dtype == SFG_BF16)
        SFG_LAUNCH(k_widen_val<__nv_bfloat16>, stream_grid(ctx, v.nvals, kBlock, 4, 8), kBlock, 0, ctx->stream,
                   static_cast<const __nv_bfloat16*>(values), v.nvals, w);
      else
        SFG_LAUNCH(k_widen_val<float>, stream_grid(ctx, v.nvals, kBlock, 4, 8), kBlock, 0, ctx->stream,
                   static_cast<const float*>(values), v.nvals, w);
      SFG_CUDA(cudaMemcpyAsync(host + voff, w, 8 * v.nvals, cudaMemcpyDeviceToHost, ctx->stream));
    }
    SFG_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    for (void* p : temps) dfree(ctx, p);
    throw;
  }
  for (void* p : temps) dfree(ctx, p);
  for (auto& [o, b] : heads) std::memcpy(host + o, b.data(), b.size());
  write_all(path, host, size);
}

sfg_tensor* read_container(sfg_context* ctx, const char* path_c, const sfg_format* fmt_in) {
  const std::string path(path_c);
  int64_t size = 0;
  const char* host = read_file_pinned(ctx, path_c, &size, nullptr);
  int64_t pos = 0;
  auto get = [&](int n) -> uint64_t {
    if (pos + n > size) raise(SFG_ERR_IO, "truncated container");
    uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= (uint64_t)(uint8_t)host[pos + i] << (8 * i);
    pos += n;
    return v;
  };
  if (size < 4 || std::memcmp(host, "USPT", 4) != 0) raise(SFG_ERR_IO, path + ": bad magic");
  pos = 4;
  const uint64_t version = get(2);
  if (version != 1) raise(SFG_ERR_IO, path + ": unsupported container version " + std::to_string(version));
  const uint64_t rank = get(1);
  std::vector<int64_t> ext;
  for (uint64_t k = 0; k < rank; ++k) ext.push_back((int64_t)get(8));
  struct Lvl {
    uint8_t kind;
    int64_t lo, hi;
    int64_t nidx, idx_off, nptr, ptr_off;
  };
  std::vector<Lvl> lv(get(1));
  for (auto& l : lv) {
    l.kind = (uint8_t)get(1);
    l.lo = (int64_t)get(8);
    l.hi = (int64_t)get(8);
    l.nidx = (int64_t)get(8);
    l.idx_off = pos;
    if (pos + 8 * l.nidx > size) raise(SFG_ERR_IO, "truncated container");
    pos += 8 * l.nidx;
    l.nptr = (int64_t)get(8);
    l.ptr_off = pos;
    if (pos + 8 * l.nptr > size) raise(SFG_ERR_IO, "truncated container");
    pos += 8 * l.nptr;
  }
  const int64_t nvals = (int64_t)get(8);
  const int64_t voff = pos;
  if (pos + 8 * nvals > size) raise(SFG_ERR_IO, "truncated container");
  pos += 8 * nvals;
  const uint64_t tag = get(1);
  if (tag > 1) raise(SFG_ERR_IO, path + ": bad layout tag");
  uint64_t aos_start = 0, aos_end = 0;
  if (tag == 1) {
    aos_start = get(1);
    aos_end = get(1);
    // the device's packed formats: DOK / LIL, Pack(0,1) (formats.hpp:40,45)
    if (aos_start != 0 || aos_end != 1)
      raise(SFG_ERR_UNSUPPORTED_SOURCE, path + ": only the Pack(0,1) value layout (DOK / LIL) is held on the device");
  }
  const uint64_t nparts = get(4);
  std::vector<int64_t> parts;
  for (uint64_t q = 0; q < 2 * nparts; ++q) parts.push_back((int64_t)get(8));

  // the requested format must match the stored structure; without one, the
  // level kinds name it (CSR and CSC look alike: CSR is taken)
  sfg_format fmt{};
  if (fmt_in) {
    fmt = *fmt_in;
  } else {
    fmt.value_dtype = SFG_F32;
    int found = -1;
    for (int k : {SFG_COO, SFG_CSR, SFG_DCSR, SFG_ELL, SFG_BCSR, SFG_BELL, SFG_DIA, SFG_CSB, SFG_BDIA, SFG_C2SR,
                  SFG_CISR}) {
      const auto w = expected_kinds(k);
      bool same = w.size() == lv.size();
      for (size_t l = 0; same && l < lv.size(); ++l) same = lv[l].kind == w[l];
      if (same) found = k;
    }
    if (found < 0) raise(SFG_ERR_UNSUPPORTED_SOURCE, path + ": no device format has these levels");
    if (tag == 1) {
      if (found == SFG_COO) found = SFG_DOK;
      else if (found == SFG_CSR) found = SFG_LIL;
      else raise(SFG_ERR_UNSUPPORTED_SOURCE, path + ": packed layout over a format the device does not pack");
    }
    fmt.kind = found;
    if (found == SFG_BCSR) {
      fmt.block_r = lv[2].hi - lv[2].lo + 1;
      fmt.block_c = lv[3].hi - lv[3].lo + 1;
    } else if (found == SFG_BELL) {
      fmt.block_r = fmt.block_c = lv[3].hi - lv[3].lo + 1;
    } else if (found == SFG_C2SR || found == SFG_CISR) {
      fmt.block_r = fmt.block_c = lv[0].hi - lv[0].lo + 1;  // k (C2SR: min(k, m) when k > m)
    } else if (found == SFG_BDIA) {
      fmt.block_r = fmt.block_c = lv[2].hi - lv[2].lo + 1;
    } else if (found == SFG_CSB) {
      fmt.block_r = lv[2].hi - lv[2].lo + 1;  // the in-block extents (one-tile edges shrink them)
      fmt.block_c = lv[3].hi - lv[3].lo + 1;
    }
  }
  const auto want = expected_kinds(fmt.kind);
  bool ok = rank == 2 && lv.size() == want.size();
  for (size_t l = 0; ok && l < lv.size(); ++l) ok = lv[l].kind == want[l];
  if (ok) ok = (tag == 1) == (fmt.kind == SFG_DOK || fmt.kind == SFG_LIL);
  if (ok && nparts && fmt.kind != SFG_C2SR && fmt.kind != SFG_CISR && fmt.kind != SFG_CISRP)
    raise(SFG_ERR_UNSUPPORTED_SOURCE, path + ": partitions are held on the device for C2SR and CISR only");
  if (!ok) raise(SFG_ERR_INVALID_OPERATION, path + ": the container does not hold this format");
  const int64_t m = ext[0], n = ext[1];
  if (m >= INT32_MAX || n >= INT32_MAX || nvals >= INT32_MAX)
    raise(SFG_ERR_INVALID_OPERATION, "extent or nnz exceeds the int32 index range");

  sfg_tensor* t = new_tensor(ctx, fmt.kind, m, n);
  int* bad = static_cast<int*>(scratch(ctx, 64));
  try {
    SFG_CUDA(cudaMemsetAsync(bad, 0, 4, ctx->stream));
    auto load_i = [&](int64_t off, int64_t cnt) -> int32_t* {
      int32_t* out = dalloc_n<int32_t>(ctx, cnt);
      if (cnt) {
        auto* tmp = dalloc_n<int64_t>(ctx, cnt);
        SFG_CUDA(cudaMemcpyAsync(tmp, host + off, 8 * cnt, cudaMemcpyHostToDevice, ctx->stream));
        SFG_LAUNCH(k_narrow_i64, stream_grid(ctx, cnt, kBlock, 4, 8), kBlock, 0, ctx->stream, tmp, cnt, out, bad);
        dfree(ctx, tmp);
      }
      return out;
    };
    const bool bf16 = fmt.kind == SFG_BCSR && fmt.value_dtype == SFG_BF16;
    t->dtype = bf16 ? SFG_BF16 : SFG_F32;
    {
      auto* tmp = dalloc_n<double>(ctx, std::max<int64_t>(nvals, 1));
      if (nvals) SFG_CUDA(cudaMemcpyAsync(tmp, host + voff, 8 * nvals, cudaMemcpyHostToDevice, ctx->stream));
      if (bf16) {
        t->val = dalloc(ctx, std::max<int64_t>(nvals, 1) * 2);
        if (nvals)
          SFG_LAUNCH(k_narrow_val<__nv_bfloat16>, stream_grid(ctx, nvals, kBlock, 4, 8), kBlock, 0, ctx->stream, tmp,
                     nvals, static_cast<__nv_bfloat16*>(t->val));
      } else {
        t->val = dalloc_n<float>(ctx, nvals);
        if (nvals)
          SFG_LAUNCH(k_narrow_val<float>, stream_grid(ctx, nvals, kBlock, 4, 8), kBlock, 0, ctx->stream, tmp, nvals,
                     static_cast<float*>(t->val));
      }
      dfree(ctx, tmp);
    }
    switch (fmt.kind) {
      case SFG_DOK:
      case SFG_LIL: {
        const bool dok = fmt.kind == SFG_DOK;
        t->nnz = lv[1].nidx;
        int32_t* r = dok ? load_i(lv[0].idx_off, lv[0].nidx) : nullptr;
        if (!dok) t->ptr = load_i(lv[1].ptr_off, lv[1].nptr);
        int32_t* c = load_i(lv[1].idx_off, lv[1].nidx);
        float* vals = static_cast<float*>(t->val);
        t->val = dalloc_n<int32_t>(ctx, t->nnz * (dok ? 3 : 2));
        aos_pack_into(ctx, t, r, c, vals);
        dfree(ctx, r);
        dfree(ctx, c);
        dfree(ctx, vals);
        break;
      }
      case SFG_DIA:
      case SFG_DIAV:
        t->k = lv[0].nidx;
        t->nnz = t->k * (fmt.kind == SFG_DIAV ? n : m);
        t->slots = load_i(lv[0].idx_off, lv[0].nidx);
        break;
      case SFG_C2SR:
        t->br = t->bc = fmt.block_r;
        t->nbr = lv[0].hi - lv[0].lo + 1;
        t->k = lv[1].hi - lv[1].lo + 1;
        t->nnz = lv[2].nidx;
        t->ptr = load_i(lv[2].ptr_off, lv[2].nptr);
        t->idx = load_i(lv[2].idx_off, lv[2].nidx);
        t->partitions = parts;
        break;
      case SFG_BDIA:
        t->br = t->bc = fmt.block_r;
        t->nbr = lv[0].hi - lv[0].lo + 1;
        t->rb = lv[2].hi - lv[2].lo + 1;
        t->k = lv[1].nidx;
        t->nnz = t->k * t->rb;
        t->ptr = load_i(lv[1].ptr_off, lv[1].nptr);
        t->idx = load_i(lv[1].idx_off, lv[1].nidx);
        break;
      case SFG_CSB:
        t->br = fmt.block_r;
        t->bc = fmt.block_c;
        t->nbr = lv[0].hi - lv[0].lo + 1;
        t->nbc = lv[1].hi - lv[1].lo + 1;
        t->rb = lv[2].hi - lv[2].lo + 1;
        t->cb = lv[3].hi - lv[3].lo + 1;
        t->nnz = lv[2].nidx;
        t->ptr = load_i(lv[2].ptr_off, lv[2].nptr);
        t->row = load_i(lv[2].idx_off, lv[2].nidx);
        t->idx = load_i(lv[3].idx_off, lv[3].nidx);
        break;
      case SFG_BELL:
        t->br = t->bc = fmt.block_r;
        t->k = lv[0].nidx;
        t->nbr = lv[1].hi - lv[1].lo + 1;
        t->nbc = lv[2].hi - lv[2].lo + 1;
        t->rb = lv[3].hi - lv[3].lo + 1;
        t->cb = lv[4].hi - lv[4].lo + 1;
        t->nnz = lv[2].nidx;
        t->slots = load_i(lv[0].idx_off, lv[0].nidx);
        t->idx = load_i(lv[2].idx_off, lv[2].nidx);
        break;
      case SFG_COO:
        t->nnz = lv[0].nidx;
        t->row = load_i(lv[0].idx_off, lv[0].nidx);
        t->idx = load_i(lv[1].idx_off, lv[1].nidx);
        break;
      case SFG_CSR:
      case SFG_CSC:
        t->nnz = lv[1].nidx;
        t->ptr = load_i(lv[1].ptr_off, lv[1].nptr);
        t->idx = load_i(lv[1].idx_off, lv[1].nidx);
        break;
      case SFG_CISR:
      case SFG_CISRP:
        t->br = t->bc = fmt.block_r;
        t->k = lv[0].nidx;
        t->nnr = lv[1].nidx;
        t->nnz = lv[2].nidx;
        t->slots = load_i(lv[0].idx_off, lv[0].nidx);
        t->ptr1 = load_i(lv[1].ptr_off, lv[1].nptr);
        t->row = load_i(lv[1].idx_off, lv[1].nidx);
        t->ptr = load_i(lv[2].ptr_off, lv[2].nptr);
        t->idx = load_i(lv[2].idx_off, lv[2].nidx);
        t->partitions = parts;
        break;
      case SFG_DCSR:
      case SFG_DCSC:
        t->nnr = lv[0].nidx;
        t->nnz = lv[1].nidx;
        t->row = load_i(lv[0].idx_off, lv[0].nidx);
        t->ptr = load_i(lv[1].ptr_off, lv[1].nptr);
        t->idx = load_i(lv[1].idx_off, lv[1].nidx);
        break;
      case SFG_ELL:
        t->k = lv[0].nidx;
        t->nnz = lv[2].nidx;
        t->slots = load_i(lv[0].idx_off, lv[0].nidx);
        t->idx = load_i(lv[2].idx_off, lv[2].nidx);
        break;
      case SFG_BCSR:
        t->br = fmt.block_r;
        t->bc = fmt.block_c;
        t->nbr = lv[0].hi - lv[0].lo + 1;
        t->nbc = lv[1].hi - lv[1].lo + 1;
        t->rb = lv[2].hi - lv[2].lo + 1;
        t->cb = lv[3].hi - lv[3].lo + 1;
        t->nnz = lv[1].nidx;
        t->ptr = load_i(lv[1].ptr_off, lv[1].nptr);
        t->idx = load_i(lv[1].idx_off, lv[1].nidx);
        break;
    }
    t->has_zeros = -1;
    int b = 0;
    read_back(ctx, bad, 4, &b);
    if (b) raise(SFG_ERR_INVALID_OPERATION, "container index exceeds the int32 range");
  } catch (...) {
    free_tensor_arrays(t);
    delete t;
    throw;
  }
  return t;
}

}  // namespace sfg
