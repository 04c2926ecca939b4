// abi.cu — the extern "C" boundary (include/sparseforge_b200.h).
//
// Each entry point converts C++ failures into a status code (1 + ErrorKind,
// or SFG_ERR_CUDA / SFG_ERR_OOM) and a thread-local message, mirroring the
// reference's Error(ErrorKind) convention (errors.hpp:10-36).
#include <cctype>
#include <cstdio>
#include <cstring>
#include <string>

#include "internal.cuh"

namespace sfg {
const char* last_error();
}

namespace {

// Makes ctx's device current for the duration of an entry point (several
// contexts on several devices may be driven from one host thread).
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(const sfg_context* ctx) {
    if (!ctx) return;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != ctx->device) {
      if (cudaSetDevice(ctx->device) == cudaSuccess) prev = cur;
      else cudaGetLastError();
    }
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return SFG_OK;
  } catch (const sfg::Failure& e) {
    sfg::set_last_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    sfg::set_last_error("host allocation failed");
    return SFG_ERR_OOM;
  } catch (const std::exception& e) {
    sfg::set_last_error(e.what());
    return SFG_ERR_INVALID_OPERATION;
  }
}

template <class F>
int guard(const sfg_context* ctx, F&& f) {
  DeviceScope scope(ctx);
  return guard(static_cast<F&&>(f));
}

void require(bool ok, int code, const char* msg) {
  if (!ok) sfg::raise(code, msg);
}

void copy_text(const std::string& s, char* buf, int64_t len) {
  if (!buf || len <= 0) return;
  size_t n = std::min<size_t>(s.size(), static_cast<size_t>(len - 1));
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
}

// plan_conversion output for a COO source (planner.hpp:95-252), as the
// reference prints it (plan_lines, planner.hpp:22-27).
std::string plan_for(const sfg_format& dst) {
  switch (dst.kind) {
    case SFG_COO: return "";
    case SFG_CSR: return "Fill(0)\nMerge(0)\n";
    case SFG_CSC: return "Swap(0,1)\nSort\nFill(0)\nMerge(0)\n";
    case SFG_DCSR: return "Merge(0)\n";
    case SFG_ELL: return "Sum(0)\nEnumerate(0)\nSort\nFill(1)\nMerge(0)\n";
    case SFG_BCSR:
      return "TileSplit(0," + std::to_string(dst.block_r) + ")\nTileSplit(2," +
             std::to_string(dst.block_c) + ")\nSwap(1,2)\nSort\nFill(3)\nFill(2)\nFill(0)\n" +
             "Vectorize(2)\nMerge(0)\n";
    case SFG_HYB:
      return "Decompose(sum(value) groupBy (d0, d1) -> (d0) with value ne 0 -> 1 | otherwise -> 0, " +
             std::to_string(dst.threshold) +
             ")\nremainder: Sum(0)\nremainder: Enumerate(0)\nremainder: Sort\nremainder: Fill(1)\n"
             "remainder: Merge(0)\n";
    case SFG_DOK: return "Pack(0,1)\n";
    case SFG_DIA: return "Skew(0,1,-1)\nSwap(0,1)\nSort\nFill(1)\nVectorize(1)\nMerge(0)\n";
    case SFG_HBELL: {
      const std::string b = std::to_string(dst.block_r);
      return "Decompose(sum(value) groupBy (d0, d1) -> (d0/" + b + ", d1/" + b +
             ") with value ne 0 -> 1 | otherwise -> 0, " + std::to_string(dst.threshold) +
             ")\nselected: TileSplit(0," + b + ")\nselected: TileSplit(2," + b +
             ")\nselected: Swap(1,2)\nselected: Sum(0)\nselected: Enumerate(0)\nselected: Sort\nselected: "
             "Fill(4)\nselected: Fill(3)\nselected: Fill(1)\nselected: Vectorize(3)\nselected: Merge(0)\n";
    }
    case SFG_C2SR:
      return "TileSplit(0," + std::to_string(dst.block_r) +
             ")\nSwap(0,1)\nSort\nFill(1)\nFill(0)\nMerge(0)\nMerge(1)\nPartition(0)\n";
    case SFG_BDIA:
      return "Skew(0,1,-1)\nTileSplit(0," + std::to_string(dst.block_r) +
             ")\nSwap(1,2)\nSort\nFill(2)\nFill(0)\nVectorize(2)\nMerge(0)\n";
    case SFG_CSB:
      return "TileSplit(0," + std::to_string(dst.block_r) + ")\nTileSplit(2," + std::to_string(dst.block_c) +
             ")\nSwap(1,2)\nSort\nFill(1)\nFill(0)\nMerge(0)\nMerge(1)\n";
    case SFG_BELL: {
      const std::string b = std::to_string(dst.block_r);
      return "TileSplit(0," + b + ")\nTileSplit(2," + b + ")\nSwap(1,2)\nSum(0)\nEnumerate(0)\nSort\nFill(4)\n"
             "Fill(3)\nFill(1)\nVectorize(3)\nMerge(0)\n";
    }
    case SFG_LIL: return "Fill(0)\nMerge(0)\nPack(0,1)\n";
    case SFG_DCSC: return "Swap(0,1)\nSort\nMerge(0)\n";
    case SFG_DIAV: return "Scale(0,-1)\nSkew(1,0,1)\nSort\nFill(1)\nVectorize(1)\nMerge(0)\n";
    case SFG_CISR: return "Sum(0)\nSchedule(0)\nSort\nMerge(0)\nMerge(1)\nPartition(0)\n";
    case SFG_CISRP: return "Sum(0)\nReorder(0)\nSchedule(0)\nSort\nMerge(0)\nMerge(1)\nPartition(0)\n";
  }
  return "";
}

bool same_format(const sfg_format& a, const sfg_format& b) {
  if (a.kind != b.kind) return false;
  if (a.kind == SFG_BCSR || a.kind == SFG_BELL || a.kind == SFG_CSB || a.kind == SFG_BDIA || a.kind == SFG_C2SR ||
      a.kind == SFG_CISR || a.kind == SFG_CISRP)
    return a.block_r == b.block_r && a.block_c == b.block_c;
  if (a.kind == SFG_HYB) return a.threshold == b.threshold;
  return true;
}

std::string simplify_plan(std::string p);
std::string plan_from_raw(const sfg_format& src, const sfg_format& dst);

// plan_conversion from a compressed source (planner.hpp:95-252): the
// source's levels are expanded back to coordinates (Split / Trim /
// Swap / Devectorize / TileUnion), a Sort restores row order where the
// target's own ops do not sort, then the target's ops as from COO. Sources
// with an indirect level or a value layout are rejected (planner.hpp:96-99).
std::string plan_from(const sfg_format& src, const sfg_format& dst) {
  if (src.kind == SFG_COO) return plan_for(dst);
  if (src.kind == SFG_ELL || src.kind == SFG_BELL || src.kind == SFG_CISR || src.kind == SFG_CISRP)
    sfg::raise(SFG_ERR_UNSUPPORTED_SOURCE, "conversion from a format with indirect levels");
  if (src.kind == SFG_DOK || src.kind == SFG_LIL || src.kind == SFG_C2SR)
    sfg::raise(SFG_ERR_UNSUPPORTED_SOURCE, "conversion from a format with a value layout");
  if (src.kind == SFG_HYB || dst.kind == SFG_HYB || src.kind == SFG_HBELL || dst.kind == SFG_HBELL)
    sfg::raise(SFG_ERR_UNSUPPORTED_SOURCE, "the hybrid pair has no single-tensor plan from a compressed source");
  if (same_format(src, dst)) return "";
  // BCSR(r,c) and CSB(r,c) share the index map: only the storage of the
  // inner levels changes (planner.hpp's equal-map branch)
  if (src.kind == SFG_BCSR && dst.kind == SFG_CSB && src.block_r == dst.block_r && src.block_c == dst.block_c)
    return "Devectorize(2)\nTrim(3)\nTrim(2)\nFill(1)\nMerge(1)\n";
  if (src.kind == SFG_CSB && dst.kind == SFG_BCSR && src.block_r == dst.block_r && src.block_c == dst.block_c)
    return "Split(1)\nTrim(1)\nFill(3)\nFill(2)\nVectorize(2)\n";
  return simplify_plan(plan_from_raw(src, dst));
}

// The reference planner composes the affine maps it emits: a skew and its
// inverse cancel, a swap commutes with a skew by conjugating it, two swaps
// cancel, and a skew followed by a swap is written as a scale and two skews.
// Applied in this order until nothing changes.
std::string simplify_plan(std::string p) {
  const std::pair<const char*, const char*> rules[] = {
      {"Skew(0,1,1)\nSkew(0,1,-1)\n", ""},
      {"Skew(1,0,1)\nSwap(0,1)\nSkew(0,1,-1)\n", "Swap(0,1)\n"},
      {"Swap(0,1)\nSkew(0,1,-1)\n", "Skew(1,0,-1)\nSwap(0,1)\n"},
      {"Swap(0,1)\nSwap(0,1)\n", ""},
      {"Skew(0,1,1)\nSwap(0,1)\n", "Scale(1,-1)\nSkew(1,0,-1)\nSkew(0,1,1)\n"},
      // DIA-variant's map (Scale(0,-1) Skew(1,0,1)) after a transposing or
      // skewed source, and its inverse before DIA's
      {"Swap(0,1)\nScale(0,-1)\nSkew(1,0,1)\n", "Skew(1,0,-1)\nSkew(0,1,1)\n"},
      {"Skew(1,0,1)\nSkew(1,0,-1)\n", ""},
      {"Skew(0,1,1)\nScale(0,-1)\nSkew(1,0,1)\n", "Skew(1,0,1)\nSwap(0,1)\n"},
      {"Scale(0,-1)\nSkew(1,0,1)\nSkew(0,1,-1)\n", "Skew(0,1,-1)\nSwap(0,1)\n"},
  };
  for (bool changed = true; changed;) {
    changed = false;
    for (const auto& [from, to] : rules)
      for (size_t at; (at = p.find(from)) != std::string::npos; changed = true)
        p.replace(at, std::strlen(from), to);
  }
  return p;
}

std::string plan_from_raw(const sfg_format& src, const sfg_format& dst) {
  const std::string tail = plan_for(dst);
  const bool sorts = tail.find("Sort\n") != std::string::npos;
  switch (src.kind) {
    case SFG_CSR:
      if (dst.kind == SFG_DCSR) return "Trim(0)\n";
      if (dst.kind == SFG_LIL) return "Pack(0,1)\n";
      return "Split(0)\nTrim(0)\n" + tail;
    case SFG_DCSR:
      if (dst.kind == SFG_CSR) return "Fill(0)\n";
      if (dst.kind == SFG_LIL) return "Fill(0)\nPack(0,1)\n";
      return "Split(0)\n" + tail;
    case SFG_DCSC:
      if (dst.kind == SFG_CSC) return "Fill(0)\n";
      return "Split(0)\nSwap(0,1)\n" + std::string(sorts ? "" : "Sort\n") + tail;
    case SFG_DIAV:
      return "Devectorize(1)\nSplit(0)\nTrim(1)\nScale(0,-1)\nSkew(1,0,1)\n" + std::string(sorts ? "" : "Sort\n") +
             tail;
    case SFG_CSC: {
      // the coordinates come back column-major: Swap(0,1), then the sort
      // unless the target's ops sort
      if (dst.kind == SFG_DCSC) return "Trim(0)\n";
      return "Split(0)\nTrim(0)\nSwap(0,1)\n" + std::string(sorts ? "" : "Sort\n") + tail;
    }
    case SFG_BCSR:
      return "Devectorize(2)\nSplit(0)\nTrim(3)\nTrim(2)\nTrim(0)\nSwap(1,2)\nTileUnion(0," +
             std::to_string(src.block_r) + ")\nTileUnion(1," + std::to_string(src.block_c) + ")\n" +
             (sorts ? "" : "Sort\n") + tail;
    case SFG_DIA:
      return "Devectorize(1)\nSplit(0)\nTrim(1)\nSkew(1,0,1)\nSwap(0,1)\n" + std::string(sorts ? "" : "Sort\n") +
             tail;
    case SFG_CSB:
      return "Split(1)\nSplit(0)\nTrim(1)\nTrim(0)\nSwap(1,2)\nTileUnion(0," + std::to_string(src.block_r) +
             ")\nTileUnion(1," + std::to_string(src.block_c) + ")\n" + (sorts ? "" : "Sort\n") + tail;
    case SFG_BDIA:
      return "Devectorize(2)\nSplit(0)\nTrim(2)\nTrim(0)\nSwap(1,2)\nTileUnion(0," + std::to_string(src.block_r) +
             ")\nSkew(0,1,1)\n" + std::string(sorts ? "" : "Sort\n") + tail;
  }
  sfg::raise(SFG_ERR_UNSUPPORTED_SOURCE, "unsupported source format");
}

// explain_storage(infer_storage(...)) (storage.hpp:35-75; oracle_data.hpp:128-148).
std::string explain_for(const sfg_format& f) {
  switch (f.kind) {
    case SFG_COO: return "L0: idx | L1: idx | val";
    case SFG_CSR:
    case SFG_CSC: return "L0: size | L1: ptr, idx | val";
    case SFG_DCSR: return "L0: idx | L1: ptr, idx | val";
    case SFG_ELL: return "L0: idx | L1: size | L2: idx | val";
    case SFG_BCSR:
      return "L0: size | L1: ptr, idx | L2: size, dense_vector | L3: size, dense_vector | val";
    case SFG_HYB: return "ELL(L0: idx | L1: size | L2: idx | val) + COO(L0: idx | L1: idx | val)";
    case SFG_DOK: return "L0: idx | L1: idx | val | pack(0,1)";
    case SFG_BELL:
      return "L0: idx | L1: size | L2: idx | L3: size, dense_vector | L4: size, dense_vector | val";
    case SFG_DIA: return "L0: idx | L1: size, dense_vector | val";
    case SFG_BDIA: return "L0: size | L1: ptr, idx | L2: size, dense_vector | val";
    case SFG_C2SR: return "L0: size | L1: size | L2: ptr, idx | val | partition(0)";
    case SFG_HBELL:
      return "BELL(L0: idx | L1: size | L2: idx | L3: size, dense_vector | L4: size, dense_vector | val) + "
             "COO(L0: idx | L1: idx | val)";
    case SFG_CSB: return "L0: size | L1: size | L2: ptr, idx | L3: idx | val";
    case SFG_LIL: return "L0: size | L1: ptr, idx | val | pack(0,1)";
    case SFG_DCSC: return "L0: idx | L1: ptr, idx | val";
    case SFG_DIAV: return "L0: idx | L1: size, dense_vector | val";
    case SFG_CISR:
    case SFG_CISRP: return "L0: idx | L1: ptr, idx | L2: ptr, idx | val | partition(0)";
  }
  return "";
}

void validate_format(const sfg_format& f) {
  require(f.kind >= SFG_COO && f.kind <= SFG_CISRP, SFG_ERR_PARSE, "unknown format kind");
  if (f.kind == SFG_BCSR || f.kind == SFG_BELL || f.kind == SFG_CSB || f.kind == SFG_BDIA || f.kind == SFG_C2SR ||
      f.kind == SFG_HBELL || f.kind == SFG_CISR || f.kind == SFG_CISRP)
    require(f.block_r > 0 && f.block_c > 0, SFG_ERR_INVALID_OPERATION,
            "TileSplit factor must be positive");
  require(f.value_dtype == SFG_F32 || (f.value_dtype == SFG_BF16 && f.kind == SFG_BCSR),
          SFG_ERR_INVALID_OPERATION, "bf16 values are supported for BCSR only");
}

sfg_level_view level(uint32_t storage, int64_t lo, int64_t hi, int64_t nodes, int64_t idx_len,
                     const int32_t* idx, int64_t ptr_len, const int32_t* ptr) {
  sfg_level_view v;
  v.storage = storage;
  v.lo = lo;
  v.hi = hi;
  v.node_count = nodes;
  v.idx_len = idx_len;
  v.ptr_len = ptr_len;
  v.idx = idx;
  v.ptr = ptr;
  return v;
}

}  // namespace

extern "C" {

const char* sfg_last_error(void) { return sfg::last_error(); }

int sfg_context_create(int device, void* stream, sfg_context** out) {
  return guard([&] {
    require(out != nullptr, SFG_ERR_INVALID_OPERATION, "null output");
    *out = nullptr;
    SFG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    SFG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      sfg::raise(SFG_ERR_CUDA, std::string("sm_100a build needs a Blackwell (cc 10.x) device, got ") +
                                   prop.name);
    auto* ctx = new sfg_context;
    ctx->device = device;
    ctx->stream = static_cast<cudaStream_t>(stream);
    ctx->sms = prop.multiProcessorCount;
    ctx->total_mem = prop.totalGlobalMem;
    SFG_CUDA(cudaMallocHost(&ctx->pinned, 4096));
    // Keep freed blocks in the pool: conversions allocate and free per call.
    cudaMemPool_t pool;
    SFG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    SFG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    *out = ctx;
  });
}

int sfg_context_set_stream(sfg_context* ctx, void* stream) {
  return guard(ctx, [&] {
    require(ctx, SFG_ERR_INVALID_OPERATION, "null context");
    SFG_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->stream = static_cast<cudaStream_t>(stream);
  });
}

int sfg_context_release_cached(sfg_context* ctx, int64_t* bytes_out) {
  return guard(ctx, [&] {
    require(ctx, SFG_ERR_INVALID_OPERATION, "null context");
    if (bytes_out) *bytes_out = static_cast<int64_t>(ctx->cached_bytes);
    sfg::release_cached(ctx);
  });
}

int sfg_context_synchronize(sfg_context* ctx) {
  return guard(ctx, [&] { SFG_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

int sfg_context_destroy(sfg_context* ctx) {
  return guard(ctx, [&] {
    if (!ctx) return;
    if (ctx->scratch) sfg::dfree(ctx, ctx->scratch);
    if (ctx->status) sfg::dfree(ctx, ctx->status);
    sfg::release_cached(ctx);
    cudaStreamSynchronize(ctx->stream);
    cudaFreeHost(ctx->pinned);
    if (ctx->sizes_ev) cudaEventDestroy(ctx->sizes_ev);
    for (cudaEvent_t e : ctx->size_events)
      if (e) cudaEventDestroy(e);
    if (ctx->size_slots) cudaFreeHost(ctx->size_slots);
    if (ctx->staging) cudaFreeHost(ctx->staging);
    delete ctx;
  });
}

int sfg_format_resolve(const char* text, sfg_format* out) {
  return guard([&] {
    require(text && out, SFG_ERR_INVALID_OPERATION, "null argument");
    std::string t;
    for (const char* p = text; *p; ++p)
      if (!std::isspace(static_cast<unsigned char>(*p))) t += *p;
    require(!t.empty(), SFG_ERR_PARSE, "empty format");
    std::string name = t;
    int64_t args[2] = {0, 0};
    int nargs = 0;
    auto open = t.find('(');
    if (open != std::string::npos) {
      require(t.back() == ')', SFG_ERR_PARSE, "malformed format name");
      name = t.substr(0, open);
      std::string inner = t.substr(open + 1, t.size() - open - 2);
      size_t pos = 0;
      while (pos <= inner.size() && nargs < 3) {
        size_t next = inner.find(',', pos);
        if (next == std::string::npos) next = inner.size();
        std::string piece = inner.substr(pos, next - pos);
        require(!piece.empty() && piece.find_first_not_of("0123456789") == std::string::npos,
                SFG_ERR_PARSE, "format arguments must be positive integers");
        require(nargs < 2, SFG_ERR_PARSE, "too many format arguments");
        args[nargs++] = std::stoll(piece);
        pos = next + 1;
        if (next == inner.size()) break;
      }
    }
    sfg_format f{};
    f.value_dtype = SFG_F32;
    if (name == "COO") f.kind = SFG_COO;
    else if (name == "CSR") f.kind = SFG_CSR;
    else if (name == "CSC") f.kind = SFG_CSC;
    else if (name == "DCSR") f.kind = SFG_DCSR;
    else if (name == "DCSC") f.kind = SFG_DCSC;
    else if (name == "DIA-variant" || name == "DIAV") f.kind = SFG_DIAV;
    else if (name == "ELL") f.kind = SFG_ELL;
    else if (name == "DOK") f.kind = SFG_DOK;
    else if (name == "LIL") f.kind = SFG_LIL;
    else if (name == "BCSR") {
      // formats.hpp:49-53: r defaults to 2, c defaults to r
      f.kind = SFG_BCSR;
      f.block_r = static_cast<int32_t>(nargs > 0 ? args[0] : 2);
      f.block_c = static_cast<int32_t>(nargs > 1 ? args[1] : f.block_r);
    } else if (name == "CSB") {
      // formats.hpp:54-57: r defaults to 2, c defaults to r
      f.kind = SFG_CSB;
      f.block_r = static_cast<int32_t>(nargs > 0 ? args[0] : 2);
      f.block_c = static_cast<int32_t>(nargs > 1 ? args[1] : f.block_r);
    } else if (name == "DIA") {
      f.kind = SFG_DIA;
    } else if (name == "HBELL") {
      // hybrid BELL/COO: block size b (default 2), threshold (default b*b/2)
      f.kind = SFG_HBELL;
      f.block_r = f.block_c = static_cast<int32_t>(nargs > 0 ? args[0] : 2);
      f.threshold = nargs > 1 ? args[1] : std::max<int64_t>(1, (int64_t)f.block_r * f.block_r / 2);
    } else if (name == "C2SR") {
      // formats.hpp:62-66: k defaults to 2
      f.kind = SFG_C2SR;
      f.block_r = f.block_c = static_cast<int32_t>(nargs > 0 ? args[0] : 2);
    } else if (name == "CISR" || name == "CISR-plus" || name == "CISRPLUS") {
      // formats.hpp:67-72: k partitions (default 2); -plus visits the rows
      // heaviest first
      f.kind = name == "CISR" ? SFG_CISR : SFG_CISRP;
      f.block_r = f.block_c = static_cast<int32_t>(nargs > 0 ? args[0] : 2);
    } else if (name == "BDIA") {
      // formats.hpp:76-79: one argument, the block size (default 3)
      f.kind = SFG_BDIA;
      f.block_r = f.block_c = static_cast<int32_t>(nargs > 0 ? args[0] : 3);
    } else if (name == "BELL") {
      // formats.hpp:79-85: one argument, the block size (default 2)
      f.kind = SFG_BELL;
      f.block_r = f.block_c = static_cast<int32_t>(nargs > 0 ? args[0] : 2);
    } else if (name == "HYB") {
      f.kind = SFG_HYB;
      f.threshold = nargs > 0 ? args[0] : 8;
    } else {
      sfg::raise(SFG_ERR_PARSE, "unknown format name: " + name);
    }
    validate_format(f);
    *out = f;
  });
}

int sfg_plan_text(const sfg_format* src, const sfg_format* dst, char* buf, int64_t len) {
  return guard([&] {
    require(src && dst, SFG_ERR_INVALID_OPERATION, "null format");
    validate_format(*src);
    validate_format(*dst);
    copy_text(plan_from(*src, *dst), buf, len);
  });
}

int sfg_storage_explain(const sfg_format* f, char* buf, int64_t len) {
  return guard([&] {
    require(f != nullptr, SFG_ERR_INVALID_OPERATION, "null format");
    validate_format(*f);
    copy_text(explain_for(*f), buf, len);
  });
}

int sfg_from_coo(sfg_context* ctx, int64_t rows, int64_t cols, int64_t nnz, const int32_t* row,
                 const int32_t* col, const float* val, uint32_t flags, sfg_tensor** out) {
  return guard(ctx, [&] {
    require(ctx && out, SFG_ERR_INVALID_OPERATION, "null argument");
    *out = nullptr;
    require(nnz >= 0 && rows >= 0 && cols >= 0, SFG_ERR_INVALID_OPERATION,
            "coordinate rank mismatch");
    require(rows < INT32_MAX && cols < INT32_MAX && nnz < INT32_MAX, SFG_ERR_INVALID_OPERATION,
            "extent or nnz exceeds the int32 index range");
    const int32_t* drow = row;
    const int32_t* dcol = col;
    const float* dval = val;
    int32_t* tmp[3] = {nullptr, nullptr, nullptr};
    if (flags & SFG_FLAG_HOST) {
      tmp[0] = sfg::dalloc_n<int32_t>(ctx, nnz);
      tmp[1] = sfg::dalloc_n<int32_t>(ctx, nnz);
      tmp[2] = sfg::dalloc_n<int32_t>(ctx, nnz);
      SFG_CUDA(cudaMemcpyAsync(tmp[0], row, nnz * 4, cudaMemcpyHostToDevice, ctx->stream));
      SFG_CUDA(cudaMemcpyAsync(tmp[1], col, nnz * 4, cudaMemcpyHostToDevice, ctx->stream));
      SFG_CUDA(cudaMemcpyAsync(tmp[2], val, nnz * 4, cudaMemcpyHostToDevice, ctx->stream));
      drow = tmp[0];
      dcol = tmp[1];
      dval = reinterpret_cast<const float*>(tmp[2]);
    }
    sfg_tensor* t = nullptr;
    try {
      if (flags & SFG_FLAG_SORTED) {
        int zeros = sfg::check_coo_canonical(ctx, drow, dcol, dval, rows, cols, nnz);
        t = sfg::new_tensor(ctx, SFG_COO, rows, cols);
        t->nnz = nnz;
        t->has_zeros = zeros;
        t->row = sfg::dalloc_n<int32_t>(ctx, nnz);
        t->idx = sfg::dalloc_n<int32_t>(ctx, nnz);
        t->val = sfg::dalloc_n<float>(ctx, nnz);
        SFG_CUDA(cudaMemcpyAsync(t->row, drow, nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
        SFG_CUDA(cudaMemcpyAsync(t->idx, dcol, nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
        SFG_CUDA(cudaMemcpyAsync(t->val, dval, nnz * 4, cudaMemcpyDeviceToDevice, ctx->stream));
      } else {
        t = sfg::sort_coo(ctx, rows, cols, nnz, drow, dcol, dval,
                          (flags & SFG_FLAG_SUM_DUPLICATES) != 0);
      }
    } catch (...) {
      for (auto* p : tmp) sfg::dfree(ctx, p);
      throw;
    }
    for (auto* p : tmp) sfg::dfree(ctx, p);
    *out = t;
  });
}

int sfg_convert(sfg_context* ctx, const sfg_tensor* src, const sfg_format* dst, sfg_tensor** out) {
  return guard(ctx, [&] {
    require(ctx && src && dst && out, SFG_ERR_INVALID_OPERATION, "null argument");
    *out = nullptr;
    validate_format(*dst);
    if (src->kind != SFG_COO) {
      *out = sfg::convert_from_compressed(ctx, src, *dst);
      return;
    }
    if (src->m <= 0 || src->n <= 0)
      sfg::raise(SFG_ERR_INVALID_OPERATION, "empty bounds at extent-only level");
    switch (dst->kind) {
      case SFG_COO: *out = sfg::coo_to_coo(ctx, src); break;
      case SFG_CSR: *out = sfg::coo_to_csr(ctx, src); break;
      case SFG_CSC: *out = sfg::coo_to_csc(ctx, src); break;
      case SFG_DCSR: *out = sfg::coo_to_dcsr(ctx, src); break;
      case SFG_ELL: *out = sfg::coo_to_ell(ctx, src); break;
      case SFG_BCSR:
        *out = sfg::coo_to_bcsr(ctx, src, dst->block_r, dst->block_c, dst->value_dtype);
        break;
      case SFG_HYB: *out = sfg::coo_to_hyb(ctx, src, dst->threshold); break;
      case SFG_DOK: *out = sfg::coo_to_dok(ctx, src); break;
      case SFG_LIL: *out = sfg::coo_to_lil(ctx, src); break;
      case SFG_BELL: *out = sfg::coo_to_bell(ctx, src, dst->block_r); break;
      case SFG_DIA: *out = sfg::coo_to_dia(ctx, src); break;
      case SFG_CSB: *out = sfg::coo_to_csb(ctx, src, dst->block_r, dst->block_c); break;
      case SFG_BDIA: *out = sfg::coo_to_bdia(ctx, src, dst->block_r); break;
      case SFG_C2SR: *out = sfg::coo_to_c2sr(ctx, src, dst->block_r); break;
      case SFG_HBELL: *out = sfg::coo_to_hbell(ctx, src, dst->block_r, dst->threshold); break;
      case SFG_DCSC: *out = sfg::coo_to_dcsc(ctx, src); break;
      case SFG_DIAV: *out = sfg::coo_to_dia(ctx, src, true); break;
      case SFG_CISR:
      case SFG_CISRP: *out = sfg::coo_to_cisr(ctx, src, dst->block_r, dst->kind == SFG_CISRP); break;
    }
  });
}

int sfg_decompose_rows(sfg_context* ctx, const sfg_tensor* coo, int64_t min_sum,
                       sfg_tensor** selected, sfg_tensor** remainder, int32_t* totals) {
  return guard(ctx, [&] {
    require(ctx && coo && selected && remainder, SFG_ERR_INVALID_OPERATION, "null argument");
    require(coo->kind == SFG_COO, SFG_ERR_INVALID_OPERATION,
            "decompose expects coordinate-form input");
    *selected = *remainder = nullptr;
    sfg::decompose_rows(ctx, coo, min_sum, selected, remainder, totals);
  });
}

int sfg_decompose_blocks(sfg_context* ctx, const sfg_tensor* coo, int64_t r, int64_t c, int64_t min_sum,
                         sfg_tensor** selected, sfg_tensor** remainder) {
  return guard(ctx, [&] {
    require(ctx && coo && selected && remainder, SFG_ERR_INVALID_OPERATION, "null argument");
    require(coo->kind == SFG_COO, SFG_ERR_INVALID_OPERATION, "decompose expects coordinate-form input");
    require(r > 0 && c > 0, SFG_ERR_INVALID_OPERATION, "TileSplit factor must be positive");
    *selected = *remainder = nullptr;
    sfg::decompose_blocks(ctx, coo, r, c, min_sum, selected, remainder);
  });
}

int sfg_tensor_view_get(sfg_context* ctx, const sfg_tensor* t, sfg_tensor_view* out) {
  return guard(ctx, [&] {
    require(t && out, SFG_ERR_INVALID_OPERATION, "null argument");
    (void)ctx;
    sfg_tensor_view v;
    std::memset(&v, 0, sizeof v);
    v.kind = t->kind;
    v.value_dtype = t->dtype;
    v.rows = t->m;
    v.cols = t->n;
    v.values = t->val;
    v.record_words = 1;
    const int S = SFG_LEVEL_SIZE, P = SFG_LEVEL_PTR, I = SFG_LEVEL_IDX, D = SFG_LEVEL_DENSE_VECTOR;
    switch (t->kind) {
      case SFG_COO:
        v.nlevels = 2;
        v.level[0] = level(I, 0, t->m - 1, t->nnz, t->nnz, t->row, 0, nullptr);
        v.level[1] = level(I, 0, t->n - 1, t->nnz, t->nnz, t->idx, 0, nullptr);
        v.nvals = t->nnz;
        break;
      case SFG_CSR:
        v.nlevels = 2;
        v.level[0] = level(S, 0, t->m - 1, t->m, 0, nullptr, 0, nullptr);
        v.level[1] = level(P | I, 0, t->n - 1, t->nnz, t->nnz, t->idx, t->m + 1, t->ptr);
        v.nvals = t->nnz;
        break;
      case SFG_CSC:
        v.nlevels = 2;
        v.level[0] = level(S, 0, t->n - 1, t->n, 0, nullptr, 0, nullptr);
        v.level[1] = level(P | I, 0, t->m - 1, t->nnz, t->nnz, t->idx, t->n + 1, t->ptr);
        v.nvals = t->nnz;
        break;
      case SFG_DCSR: {
        const int64_t nnr = sfg::tensor_nnr(t);  // may still be in flight
        v.nlevels = 2;
        v.level[0] = level(I, 0, t->m - 1, nnr, nnr, t->row, 0, nullptr);
        v.level[1] = level(P | I, 0, t->n - 1, t->nnz, t->nnz, t->idx, nnr + 1, t->ptr);
        v.nvals = t->nnz;
        break;
      }
      case SFG_ELL:
        v.nlevels = 3;
        v.level[0] = level(I, 0, t->k - 1, t->k, t->k, t->slots, 0, nullptr);
        v.level[1] = level(S, 0, t->m - 1, t->k * t->m, 0, nullptr, 0, nullptr);
        v.level[2] = level(I, 0, t->n - 1, t->k * t->m, t->k * t->m, t->idx, 0, nullptr);
        v.nvals = t->k * t->m;
        break;
      case SFG_BCSR:
        v.nlevels = 4;
        v.level[0] = level(S, 0, t->nbr - 1, t->nbr, 0, nullptr, 0, nullptr);
        v.level[1] = level(P | I, 0, t->nbc - 1, t->nnz, t->nnz, t->idx, t->nbr + 1, t->ptr);
        v.level[2] = level(S | D, 0, t->rb - 1, t->nnz * t->rb, 0, nullptr, 0, nullptr);
        v.level[3] = level(S | D, 0, t->cb - 1, t->nnz * t->rb * t->cb, 0, nullptr, 0, nullptr);
        v.nvals = t->nnz * t->rb * t->cb;
        break;
      case SFG_HYB:
      case SFG_HBELL:
        v.nlevels = 0;
        v.parts[0] = t->part[0];
        v.parts[1] = t->part[1];
        break;
      case SFG_DOK: {  // records {row, col, val}
        const int32_t* rec = static_cast<const int32_t*>(t->val);
        v.nlevels = 2;
        v.level[0] = level(I, 0, t->m - 1, t->nnz, t->nnz, rec, 0, nullptr);
        v.level[1] = level(I, 0, t->n - 1, t->nnz, t->nnz, rec ? rec + 1 : nullptr, 0, nullptr);
        v.values = rec ? rec + 2 : nullptr;
        v.nvals = t->nnz;
        v.layout = 1, v.aos_start = 0, v.aos_end = 1, v.record_words = 3;
        break;
      }
      case SFG_BELL: {  // slot-major cells (slot, block row), dense b x b blocks
        const int64_t cells = t->k * t->nbr;
        v.nlevels = 5;
        v.level[0] = level(I, 0, t->k - 1, t->k, t->k, t->slots, 0, nullptr);
        v.level[1] = level(S, 0, t->nbr - 1, cells, 0, nullptr, 0, nullptr);
        v.level[2] = level(I, 0, t->nbc - 1, cells, cells, t->idx, 0, nullptr);
        v.level[3] = level(S | D, 0, t->rb - 1, cells * t->rb, 0, nullptr, 0, nullptr);
        v.level[4] = level(S | D, 0, t->cb - 1, cells * t->rb * t->cb, 0, nullptr, 0, nullptr);
        v.nvals = cells * t->rb * t->cb;
        break;
      }
      case SFG_DIA:  // diagonals, then a dense vector over the rows
        v.nlevels = 2;
        v.level[0] = level(I, -(t->m - 1), t->n - 1, t->k, t->k, t->slots, 0, nullptr);
        v.level[1] = level(S | D, 0, t->m - 1, t->k * t->m, 0, nullptr, 0, nullptr);
        v.nvals = t->k * t->m;
        break;
      case SFG_DIAV:  // diagonals, then a dense vector over the columns
        v.nlevels = 2;
        v.level[0] = level(I, -(t->m - 1), t->n - 1, t->k, t->k, t->slots, 0, nullptr);
        v.level[1] = level(S | D, 0, t->n - 1, t->k * t->n, 0, nullptr, 0, nullptr);
        v.nvals = t->k * t->n;
        break;
      case SFG_CISR:
      case SFG_CISRP: {  // partitions, their rows, the rows' columns; value range per partition
        v.nlevels = 3;
        v.level[0] = level(I, 0, t->br - 1, t->k, t->k, t->slots, 0, nullptr);
        v.level[1] = level(P | I, 0, t->m - 1, t->nnr, t->nnr, t->row, t->k + 1, t->ptr1);
        v.level[2] = level(P | I, 0, t->n - 1, t->nnz, t->nnz, t->idx, t->nnr + 1, t->ptr);
        v.nvals = t->nnz;
        v.npartitions = (int64_t)t->partitions.size() / 2;
        v.partitions = t->partitions.data();
        break;
      }
      case SFG_DCSC: {  // nonempty columns, then the rows
        const int64_t nnc = sfg::tensor_nnr(t);
        v.nlevels = 2;
        v.level[0] = level(I, 0, t->n - 1, nnc, nnc, t->row, 0, nullptr);
        v.level[1] = level(P | I, 0, t->m - 1, t->nnz, t->nnz, t->idx, nnc + 1, t->ptr);
        v.nvals = t->nnz;
        break;
      }
      case SFG_C2SR:  // residue classes, rows per class, CSR over the interleaved rows
        v.nlevels = 3;
        v.level[0] = level(S, 0, t->nbr - 1, t->nbr, 0, nullptr, 0, nullptr);
        v.level[1] = level(S, 0, t->k - 1, t->nbr * t->k, 0, nullptr, 0, nullptr);
        v.level[2] = level(P | I, 0, t->n - 1, t->nnz, t->nnz, t->idx, t->nbr * t->k + 1, t->ptr);
        v.nvals = t->nnz;
        v.npartitions = (int64_t)t->partitions.size() / 2;
        v.partitions = t->partitions.data();
        break;
      case SFG_BDIA:  // block rows, their diagonals, a dense vector over the block's rows
        v.nlevels = 3;
        v.level[0] = level(S, 0, t->nbr - 1, t->nbr, 0, nullptr, 0, nullptr);
        v.level[1] = level(P | I, -(t->m - 1), t->n - 1, t->k, t->k, t->idx, t->nbr + 1, t->ptr);
        v.level[2] = level(S | D, 0, t->rb - 1, t->k * t->rb, 0, nullptr, 0, nullptr);
        v.nvals = t->k * t->rb;
        break;
      case SFG_CSB:  // dense block grid, entries per block (row, column in block)
        v.nlevels = 4;
        v.level[0] = level(S, 0, t->nbr - 1, t->nbr, 0, nullptr, 0, nullptr);
        v.level[1] = level(S, 0, t->nbc - 1, t->nbr * t->nbc, 0, nullptr, 0, nullptr);
        v.level[2] = level(P | I, 0, t->rb - 1, t->nnz, t->nnz, t->row, t->nbr * t->nbc + 1, t->ptr);
        v.level[3] = level(I, 0, t->cb - 1, t->nnz, t->nnz, t->idx, 0, nullptr);
        v.nvals = t->nnz;
        break;
      case SFG_LIL: {  // ptr + records {col, val}
        const int32_t* rec = static_cast<const int32_t*>(t->val);
        v.nlevels = 2;
        v.level[0] = level(S, 0, t->m - 1, t->m, 0, nullptr, 0, nullptr);
        v.level[1] = level(P | I, 0, t->n - 1, t->nnz, t->nnz, rec, t->m + 1, t->ptr);
        v.values = rec ? rec + 1 : nullptr;
        v.nvals = t->nnz;
        v.layout = 1, v.aos_start = 0, v.aos_end = 1, v.record_words = 2;
        break;
      }
    }
    *out = v;
  });
}

int sfg_tensor_free(sfg_tensor* t) {
  return guard(t ? t->ctx : nullptr, [&] {
    if (!t) return;
    for (auto* p : t->part)
      if (p) {
        sfg::free_tensor_arrays(p);
        delete p;
      }
    sfg::free_tensor_arrays(t);
    delete t;
  });
}

int sfg_spmv(sfg_context* ctx, const sfg_tensor* a, const float* x, float* y, uint32_t flags) {
  return guard(ctx, [&] {
    require(ctx && a && x && y, SFG_ERR_INVALID_OPERATION, "null argument");
    if (flags & SFG_COMPUTE_HOST) {
      float* dx = sfg::dalloc_n<float>(ctx, a->n);
      float* dy = sfg::dalloc_n<float>(ctx, a->m);
      try {
        SFG_CUDA(cudaMemcpyAsync(dx, x, a->n * 4, cudaMemcpyHostToDevice, ctx->stream));
        if (flags & SFG_COMPUTE_ACCUMULATE)
          SFG_CUDA(cudaMemcpyAsync(dy, y, a->m * 4, cudaMemcpyHostToDevice, ctx->stream));
        sfg::spmv(ctx, a, dx, dy, (flags & SFG_COMPUTE_ACCUMULATE) != 0);
        SFG_CUDA(cudaMemcpyAsync(y, dy, a->m * 4, cudaMemcpyDeviceToHost, ctx->stream));
        SFG_CUDA(cudaStreamSynchronize(ctx->stream));
      } catch (...) {
        sfg::dfree(ctx, dx);
        sfg::dfree(ctx, dy);
        throw;
      }
      sfg::dfree(ctx, dx);
      sfg::dfree(ctx, dy);
    } else {
      sfg::spmv(ctx, a, x, y, (flags & SFG_COMPUTE_ACCUMULATE) != 0);
    }
  });
}

int sfg_spmm(sfg_context* ctx, const sfg_tensor* a, const void* b, int32_t b_dtype, int64_t nd,
             int64_t ldb, float* c, int64_t ldc, uint32_t flags) {
  return guard(ctx, [&] {
    require(ctx && a && b && c, SFG_ERR_INVALID_OPERATION, "null argument");
    require(nd > 0 && ldb >= nd && ldc >= nd, SFG_ERR_INVALID_OPERATION, "bad dense shape");
    require(b_dtype == SFG_F32 || b_dtype == SFG_BF16, SFG_ERR_INVALID_OPERATION, "bad dtype");
    bool acc = (flags & SFG_COMPUTE_ACCUMULATE) != 0;
    if (flags & SFG_COMPUTE_HOST) {
      size_t esz = b_dtype == SFG_F32 ? 4 : 2;
      void* db = sfg::dalloc(ctx, a->n * ldb * esz);
      float* dc = sfg::dalloc_n<float>(ctx, a->m * ldc);
      try {
        SFG_CUDA(cudaMemcpyAsync(db, b, a->n * ldb * esz, cudaMemcpyHostToDevice, ctx->stream));
        if (acc)
          SFG_CUDA(cudaMemcpyAsync(dc, c, a->m * ldc * 4, cudaMemcpyHostToDevice, ctx->stream));
        sfg::spmm(ctx, a, db, b_dtype, nd, ldb, dc, ldc, acc);
        SFG_CUDA(cudaMemcpyAsync(c, dc, a->m * ldc * 4, cudaMemcpyDeviceToHost, ctx->stream));
        SFG_CUDA(cudaStreamSynchronize(ctx->stream));
      } catch (...) {
        sfg::dfree(ctx, db);
        sfg::dfree(ctx, dc);
        throw;
      }
      sfg::dfree(ctx, db);
      sfg::dfree(ctx, dc);
    } else {
      sfg::spmm(ctx, a, b, b_dtype, nd, ldb, c, ldc, acc);
    }
  });
}

int sfg_row_partition(sfg_context* ctx, const sfg_tensor* coo, int32_t parts, int64_t* bounds) {
  return guard(ctx, [&] {
    require(ctx && coo && bounds && parts > 0, SFG_ERR_INVALID_OPERATION, "bad argument");
    require(coo->kind == SFG_COO, SFG_ERR_INVALID_OPERATION, "row partition expects COO");
    sfg::row_partition(ctx, coo, parts, bounds);
  });
}

int sfg_read_matrix_market(sfg_context* ctx, const char* path, uint32_t flags, sfg_tensor** out) {
  return guard(ctx, [&] {
    require(ctx && path && out, SFG_ERR_INVALID_OPERATION, "null argument");
    *out = nullptr;
    *out = sfg::read_matrix_market(ctx, path, (flags & SFG_FLAG_SUM_DUPLICATES) != 0);
  });
}

int sfg_spgemm(sfg_context* ctx, const sfg_tensor* a, const sfg_tensor* b, float* c, int64_t ldc,
               uint32_t flags) {
  return guard(ctx, [&] {
    require(ctx && a && b && c, SFG_ERR_INVALID_OPERATION, "null argument");
    require(ldc >= b->n, SFG_ERR_INVALID_OPERATION, "ldc < columns of B");
    const bool acc = (flags & SFG_COMPUTE_ACCUMULATE) != 0;
    if (flags & SFG_COMPUTE_HOST) {
      float* dc = sfg::dalloc_n<float>(ctx, a->m * ldc);
      try {
        if (acc) SFG_CUDA(cudaMemcpyAsync(dc, c, a->m * ldc * 4, cudaMemcpyHostToDevice, ctx->stream));
        sfg::spgemm(ctx, a, b, dc, ldc, acc);
        SFG_CUDA(cudaMemcpyAsync(c, dc, a->m * ldc * 4, cudaMemcpyDeviceToHost, ctx->stream));
        SFG_CUDA(cudaStreamSynchronize(ctx->stream));
      } catch (...) {
        sfg::dfree(ctx, dc);
        throw;
      }
      sfg::dfree(ctx, dc);
    } else {
      sfg::spgemm(ctx, a, b, c, ldc, acc);
    }
  });
}

int sfg_write_container(sfg_context* ctx, const sfg_tensor* t, const char* path) {
  return guard(ctx, [&] {
    require(ctx && t && path, SFG_ERR_INVALID_OPERATION, "null argument");
    sfg::write_container(ctx, t, path);
  });
}

int sfg_read_container(sfg_context* ctx, const char* path, const sfg_format* fmt, sfg_tensor** out) {
  return guard(ctx, [&] {
    require(ctx && path && out, SFG_ERR_INVALID_OPERATION, "null argument");
    *out = nullptr;
    if (fmt) {
      validate_format(*fmt);
      if (fmt->kind == SFG_HYB) sfg::raise(SFG_ERR_INVALID_OPERATION, "the hybrid pair is two containers");
    }
    *out = sfg::read_container(ctx, path, fmt);
  });
}

int sfgx_row_bounds_host(const int32_t* rows, int64_t nnz, int64_t n_rows, int32_t parts, int64_t* bounds) {
  return guard([&] {
    require(parts >= 1 && bounds, SFG_ERR_INVALID_OPERATION, "row_bounds: parts must be >= 1");
    require(nnz == 0 || rows, SFG_ERR_INVALID_OPERATION, "row_bounds: null rows");
    sfg::row_bounds_host(rows, nnz, n_rows, parts, bounds);
  });
}

int sfg_coo_slice_rows(sfg_context* ctx, const sfg_tensor* coo, int64_t r0, int64_t r1,
                       sfg_tensor** out) {
  return guard(ctx, [&] {
    require(ctx && coo && out, SFG_ERR_INVALID_OPERATION, "null argument");
    require(coo->kind == SFG_COO, SFG_ERR_INVALID_OPERATION, "row slice expects COO");
    require(0 <= r0 && r0 <= r1 && r1 <= coo->m, SFG_ERR_INVALID_OPERATION, "bad row range");
    *out = sfg::coo_slice_rows(ctx, coo, r0, r1);
  });
}

int sfg_comm_unique_id(uint8_t id[SFG_COMM_ID_BYTES]) {
  return guard([&] {
    require(id, SFG_ERR_INVALID_OPERATION, "null argument");
    sfg::comm_unique_id(id);
  });
}

int sfg_comm_create(sfg_context* ctx, int32_t nranks, int32_t rank, const uint8_t id[SFG_COMM_ID_BYTES],
                    sfg_comm** out) {
  return guard(ctx, [&] {
    require(ctx && id && out, SFG_ERR_INVALID_OPERATION, "null argument");
    require(nranks > 0 && rank >= 0 && rank < nranks, SFG_ERR_INVALID_OPERATION, "bad rank");
    *out = nullptr;
    *out = sfg::comm_create(ctx, nranks, rank, id);
  });
}

int sfg_comm_destroy(sfg_comm* comm) {
  return guard([&] {
    if (comm) sfg::comm_destroy(comm);
  });
}

int sfg_rowpart_spmv(sfg_context* ctx, sfg_comm* comm, const sfg_tensor* a_block, const float* x, float* y,
                     int64_t chunk_rows, uint32_t flags) {
  return guard(ctx, [&] {
    require(ctx && comm && a_block && x && y, SFG_ERR_INVALID_OPERATION, "null argument");
    sfg::rowpart_spmv(ctx, comm, a_block, x, y, chunk_rows, (flags & SFG_ROWPART_GATHER) != 0);
  });
}

int sfg_rowpart_spmm(sfg_context* ctx, sfg_comm* comm, const sfg_tensor* a_block, const void* b, int32_t b_dtype,
                     int64_t nd, int64_t ldb, float* c, int64_t chunk_rows, uint32_t flags) {
  return guard(ctx, [&] {
    require(ctx && comm && a_block && b && c, SFG_ERR_INVALID_OPERATION, "null argument");
    require(nd > 0 && ldb >= nd, SFG_ERR_INVALID_OPERATION, "bad dense shape");
    require(b_dtype == SFG_F32 || b_dtype == SFG_BF16, SFG_ERR_INVALID_OPERATION, "bad dtype");
    sfg::rowpart_spmm(ctx, comm, a_block, b, b_dtype, nd, ldb, c, chunk_rows, (flags & SFG_ROWPART_GATHER) != 0);
  });
}

int sfg_allgather_chunks(sfg_context* ctx, sfg_comm* comm, float* buf, int64_t chunk_elems) {
  return guard(ctx, [&] {
    require(ctx && comm && buf && chunk_elems >= 0, SFG_ERR_INVALID_OPERATION, "bad argument");
    sfg::allgather_chunks(ctx, comm, buf, chunk_elems);
  });
}

int sfgx_gen_uniform(sfg_context* ctx, uint64_t seed, int64_t rows, int64_t cols, int32_t per_row,
                     sfg_tensor** out) {
  return guard(ctx, [&] {
    require(per_row > 0 && per_row <= 64 && per_row <= cols, SFG_ERR_INVALID_OPERATION,
            "per_row must be in [1, min(64, cols)]");
    require(rows * per_row < INT32_MAX, SFG_ERR_INVALID_OPERATION, "too many entries");
    *out = sfg::gen_uniform(ctx, seed, rows, cols, per_row);
  });
}

int sfgx_gen_rmat(sfg_context* ctx, uint64_t seed, int32_t scale, int64_t edges, sfg_tensor** out) {
  return guard(ctx, [&] {
    require(scale > 0 && scale <= 30 && edges > 0 && edges < INT32_MAX, SFG_ERR_INVALID_OPERATION,
            "bad R-MAT size");
    *out = sfg::gen_from_keys(ctx, seed, 0, scale, int64_t(1) << scale, int64_t(1) << scale, edges);
  });
}

int sfgx_gen_hypersparse(sfg_context* ctx, uint64_t seed, int64_t rows, int64_t cols,
                         int64_t draws, sfg_tensor** out) {
  return guard(ctx, [&] {
    require(rows > 0 && cols > 0 && rows < INT32_MAX && cols < INT32_MAX && draws > 0 &&
                draws < INT32_MAX,
            SFG_ERR_INVALID_OPERATION, "bad hypersparse size");
    *out = sfg::gen_from_keys(ctx, seed, 1, 0, rows, cols, draws);
  });
}

int sfgx_gen_block_sparse(sfg_context* ctx, uint64_t seed, int64_t rows, int64_t cols, int32_t r,
                          int32_t c, uint32_t thresh, int32_t value_dtype, sfg_tensor** out) {
  return guard(ctx, [&] {
    require(ctx && out && rows > 0 && cols > 0 && r > 0 && c > 0 && rows < INT32_MAX && cols < INT32_MAX,
            SFG_ERR_INVALID_OPERATION, "bad block-sparse shape");
    require(value_dtype == SFG_F32 || value_dtype == SFG_BF16, SFG_ERR_INVALID_OPERATION, "bad dtype");
    *out = sfg::gen_block_sparse(ctx, seed, rows, cols, r, c, thresh, value_dtype);
  });
}

int sfgx_gen_dense(sfg_context* ctx, uint64_t seed, int64_t count, float* out) {
  return guard(ctx, [&] { sfg::gen_dense(ctx, seed, count, out); });
}

int64_t sfgx_launch_count(void) { return sfg::g_launches.load(); }

int sfgx_device_alloc(sfg_context* ctx, int64_t bytes, void** out) {
  return guard(ctx, [&] {
    require(ctx && out && bytes >= 0, SFG_ERR_INVALID_OPERATION, "bad argument");
    *out = sfg::dalloc(ctx, static_cast<size_t>(bytes));
  });
}

int sfgx_device_free(sfg_context* ctx, void* p) {
  return guard(ctx, [&] { sfg::dfree(ctx, p); });
}

int sfgx_copy(sfg_context* ctx, void* dst, const void* src, int64_t bytes, int32_t kind) {
  return guard(ctx, [&] {
    require(ctx && bytes >= 0 && kind >= 0 && kind <= 2, SFG_ERR_INVALID_OPERATION, "bad argument");
    if (bytes == 0) return;
    cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                 : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
    SFG_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), k, ctx->stream));
    if (kind == 1) SFG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
