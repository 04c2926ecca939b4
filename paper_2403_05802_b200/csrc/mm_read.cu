// mm_read.cu — Matrix Market ingest on the device.
//
// Reference: read_matrix_market (io.hpp:50-121) followed by from_coo
// (tensor.hpp:118) — how the reference CLI loads a COO operand. Semantics
// kept: banner/object/format/field/symmetry checks (UnsupportedHeader),
// '%' comment lines (only when '%' is the first character) and blank lines
// skipped, 1-based indices shifted to 0-based, symmetric inputs mirrored
// (diagonal not duplicated; the mirror entry follows its original),
// pattern entries = 1.0, the same Parse errors with the same line numbers
// ("bad entry line", "missing value", "coordinate out of range", "entry
// count N does not match declared D"), first failing line wins.
//
// Device plan: the header (banner + size line) is parsed on the host; the
// body bytes go to HBM once. (1) k_mm_lines: line starts by a single-pass
// look-back scan of newline counts over byte tiles. (2) k_mm_parse: a
// thread per line parses "r c [v]" — integers exactly, values with the
// exact Clinger fast path (<= 19 significant digits whose value is exactly
// representable, |decimal exponent| <= 22: one correctly rounded double
// multiply or divide). Anything else (hex, inf/nan, long mantissas, odd
// token endings) is marked for the host, which re-parses those lines with
// the reference's own istringstream rules. (3) k_mm_emit: look-back scan
// of per-line entry counts (0, 1, or 2 when mirrored) and the scatter into
// COO arrays in file order. Then the device from_coo (sort.cu).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <cctype>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kBlock = 256;
constexpr int kLineBytes = 16;                 // bytes per thread in the newline scan
constexpr int kLineTile = kBlock * kLineBytes;  // 4 KB of text per tile
constexpr int kEmitItems = 16;                 // lines per thread in the emit scan
constexpr int kEmitTile = kBlock * kEmitItems;

enum : uint8_t { kOk = 0, kBadEntry = 1, kMissingValue = 2, kOutOfRange = 3, kHard = 4 };

// (1) line starts: start[0] = 0, and position p + 1 for every '\n' at p
// that is not the last byte.
__global__ void __launch_bounds__(kBlock) k_mm_lines(const char* __restrict__ text, int64_t nbytes,
                                                      int64_t* __restrict__ start,
                                                      unsigned long long* __restrict__ status,
                                                      uint32_t epoch) {
  __shared__ uint32_t smem[34];
  __shared__ uint32_t slot;
  const int64_t b0 = (int64_t)blockIdx.x * kLineTile + (int64_t)threadIdx.x * kLineBytes;
  uint32_t mask = 0;
#pragma unroll
  for (int i = 0; i < kLineBytes; ++i) {
    int64_t p = b0 + i;
    if (p < nbytes - 1 && text[p] == '\n') mask |= 1u << i;  // a line starts at p + 1
  }
  const uint32_t cnt = __popc(mask);
  uint32_t total;
  const uint32_t excl = block_exclusive_scan<uint32_t, kBlock>(cnt, smem, &total);
  const uint32_t before = lookback_prefix(status, epoch, blockIdx.x, total, &slot);
  uint32_t k = before + excl + 1;  // line index of the next start (line 0 starts at 0)
  while (mask) {
    int i = __ffs(mask) - 1;
    mask &= mask - 1;
    start[k++] = b0 + i + 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) start[0] = 0;
}

// Newlines in text[0, n) (text 16-byte aligned): 16 bytes per thread per
// step.
__global__ void __launch_bounds__(kBlock) k_count_newlines(const char* __restrict__ text, int64_t n,
                                                            unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 16; b < n;
       b += (int64_t)gridDim.x * blockDim.x * 16) {
    if (b + 16 <= n) {
      const int4 v = ld_stream(reinterpret_cast<const int4*>(text + b));
      const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t x = w[i] ^ 0x0a0a0a0au;  // zero bytes where '\n'
        c += __popc(~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x | 0x7f7f7f7fu));
      }
    } else {
      for (int64_t p = b; p < n && p < b + 16; ++p) c += text[p] == '\n';
    }
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__device__ __forceinline__ bool is_ws(char ch) {
  return ch == ' ' || ch == '\t' || ch == '\r' || ch == '\v' || ch == '\f' || ch == '\n';
}

// Exactly representable powers of ten for the Clinger fast path.
__constant__ double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                  1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

// [p, e): parses "[+-]digits" followed by whitespace or the end. Returns
// false when the token is not of that simple shape (the host decides).
__device__ __forceinline__ bool parse_int(const char* __restrict__ t, int64_t& p, int64_t e, int64_t& out,
                                          bool& present) {
  while (p < e && is_ws(t[p])) ++p;
  present = p < e;
  if (!present) return true;
  bool neg = false;
  if (t[p] == '+' || t[p] == '-') {
    neg = t[p] == '-';
    ++p;
  }
  int64_t v = 0;
  int nd = 0;
  while (p < e && t[p] >= '0' && t[p] <= '9') {
    if (nd >= 18) return false;  // may overflow: host
    v = v * 10 + (t[p] - '0');
    ++p;
    ++nd;
  }
  if (nd == 0) return false;
  if (p < e && !is_ws(t[p])) return false;
  out = neg ? -v : v;
  return true;
}

// Decimal "[+-]d*[.d*][(e|E)[+-]d+]" with at least one mantissa digit,
// followed by whitespace or the end, when its value is exact under the
// Clinger fast path. Otherwise false (the host parses the line).
__device__ __forceinline__ bool parse_real(const char* __restrict__ t, int64_t& p, int64_t e, double& out,
                                           bool& present) {
  while (p < e && is_ws(t[p])) ++p;
  present = p < e;
  if (!present) return true;
  bool neg = false;
  if (t[p] == '+' || t[p] == '-') {
    neg = t[p] == '-';
    ++p;
  }
  uint64_t mant = 0;
  int sig = 0, digits = 0, dexp = 0;
  bool lead = true;
  while (p < e && t[p] >= '0' && t[p] <= '9') {
    ++digits;
    int d = t[p] - '0';
    if (lead && d == 0) {
      ++p;
      continue;
    }
    lead = false;
    if (sig < 19) {
      mant = mant * 10 + d;
      ++sig;
    } else {
      return false;
    }
    ++p;
  }
  if (p < e && t[p] == '.') {
    ++p;
    while (p < e && t[p] >= '0' && t[p] <= '9') {
      ++digits;
      int d = t[p] - '0';
      if (lead && d == 0) {
        --dexp;
        ++p;
        continue;
      }
      lead = false;
      if (sig < 19) {
        mant = mant * 10 + d;
        ++sig;
        --dexp;
      } else {
        return false;
      }
      ++p;
    }
  }
  if (digits == 0) return false;
  if (p < e && (t[p] == 'e' || t[p] == 'E')) {
    ++p;
    bool eneg = false;
    if (p < e && (t[p] == '+' || t[p] == '-')) {
      eneg = t[p] == '-';
      ++p;
    }
    int ev = 0, en = 0;
    while (p < e && t[p] >= '0' && t[p] <= '9') {
      if (ev < 100000) ev = ev * 10 + (t[p] - '0');
      ++p;
      ++en;
    }
    if (en == 0) return false;
    dexp += eneg ? -ev : ev;
  }
  if (p < e && !is_ws(t[p])) return false;
  double v;
  if (mant == 0) {
    v = 0.0;
  } else {
    if (mant > (1ull << 53) || dexp < -22 || dexp > 22) return false;
    v = (double)mant;
    v = dexp >= 0 ? v * kPow10[dexp] : v / kPow10[-dexp];
  }
  out = neg ? -v : v;
  return true;
}

// (2) a thread per line.
__global__ void __launch_bounds__(kBlock) k_mm_parse(const char* __restrict__ text, int64_t nbytes,
                                                      const int64_t* __restrict__ start, int64_t nlines,
                                                      int64_t rows, int64_t cols, int pattern, int symmetric,
                                                      int32_t* __restrict__ lr, int32_t* __restrict__ lc,
                                                      float* __restrict__ lv, uint8_t* __restrict__ lcnt,
                                                      uint8_t* __restrict__ lst, int64_t* __restrict__ hard,
                                                      unsigned long long* __restrict__ nhard) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nlines;
       l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = start[l];
    int64_t e = l + 1 < nlines ? start[l + 1] - 1 : nbytes;  // exclusive of '\n'
    if (e > s && text[e - 1] == '\n') --e;                    // a final '\n' (last line)
    uint8_t st = kOk, cnt = 0;
    int32_t r32 = 0, c32 = 0;
    float v32 = 1.f;
    bool blank = true;
    for (int64_t p = s; p < e; ++p)
      if (!(text[p] == ' ' || text[p] == '\t' || text[p] == '\r')) {
        blank = false;
        break;
      }
    if (e > s && text[s] == '%') {
      // comment
    } else if (blank) {
      // blank line
    } else {
      int64_t p = s, r = 0, c = 0;
      bool pr = false, pc = false, pv = true, ok = true;
      double v = 1.0;
      ok = parse_int(text, p, e, r, pr) && pr && parse_int(text, p, e, c, pc) && pc;
      if (ok && !pattern) ok = parse_real(text, p, e, v, pv) && pv;
      if (!ok) {
        st = kHard;  // malformed or not fast-path: the host applies the reference's rules
      } else if (r < 1 || r > rows || c < 1 || c > cols) {
        st = kOutOfRange;
      } else {
        cnt = (symmetric && r != c) ? 2 : 1;
        r32 = (int32_t)(r - 1);
        c32 = (int32_t)(c - 1);
        v32 = (float)v;
      }
    }
    lr[l] = r32;
    lc[l] = c32;
    lv[l] = v32;
    lcnt[l] = cnt;
    lst[l] = st;
    if (st == kHard) hard[atomicAdd(nhard, 1ull)] = l;
  }
}

// Host results for the lines the device left to it.
__global__ void k_mm_patch(const int64_t* __restrict__ line, const int32_t* __restrict__ r,
                           const int32_t* __restrict__ c, const float* __restrict__ v,
                           const uint8_t* __restrict__ cnt, const uint8_t* __restrict__ st, int64_t n,
                           int32_t* __restrict__ lr, int32_t* __restrict__ lc, float* __restrict__ lv,
                           uint8_t* __restrict__ lcnt, uint8_t* __restrict__ lst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t l = line[i];
    lr[l] = r[i];
    lc[l] = c[i];
    lv[l] = v[i];
    lcnt[l] = cnt[i];
    lst[l] = st[i];
  }
}

// First failing line and the number of entry lines.
__global__ void __launch_bounds__(kBlock) k_mm_check(const uint8_t* __restrict__ lst,
                                                      const uint8_t* __restrict__ lcnt, int64_t nlines,
                                                      unsigned long long* __restrict__ out) {
  unsigned long long first = ~0ull, seen = 0;
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nlines;
       l += (int64_t)gridDim.x * blockDim.x) {
    if (lst[l] != kOk && (unsigned long long)l < first) first = (unsigned long long)l;
    seen += lcnt[l] != 0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long f2 = __shfl_xor_sync(kFull, first, o);
    first = f2 < first ? f2 : first;
    seen += __shfl_xor_sync(kFull, seen, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (first != ~0ull) atomicMin(out, first);
    atomicAdd(out + 1, seen);
  }
}

// (3) entry positions (look-back scan of per-line counts) and the scatter,
// in file order: an entry, then its mirror.
__global__ void __launch_bounds__(kBlock) k_mm_emit(const int32_t* __restrict__ lr, const int32_t* __restrict__ lc,
                                                     const float* __restrict__ lv, const uint8_t* __restrict__ lcnt,
                                                     int64_t nlines, int32_t* __restrict__ row,
                                                     int32_t* __restrict__ col, float* __restrict__ val,
                                                     unsigned long long* __restrict__ status, uint32_t epoch) {
  __shared__ uint32_t smem[34];
  __shared__ uint32_t slot;
  const int64_t l0 = (int64_t)blockIdx.x * kEmitTile + (int64_t)threadIdx.x * kEmitItems;
  uint32_t n = 0;
#pragma unroll
  for (int i = 0; i < kEmitItems; ++i)
    if (l0 + i < nlines) n += lcnt[l0 + i];
  uint32_t total;
  const uint32_t excl = block_exclusive_scan<uint32_t, kBlock>(n, smem, &total);
  uint32_t pos = lookback_prefix(status, epoch, blockIdx.x, total, &slot) + excl;
  for (int i = 0; i < kEmitItems; ++i) {
    const int64_t l = l0 + i;
    if (l >= nlines) break;
    const int k = lcnt[l];
    if (k == 0) continue;
    const int32_t r = lr[l], c = lc[l];
    const float v = lv[l];
    row[pos] = r;
    col[pos] = c;
    val[pos] = v;
    if (k == 2) {
      row[pos + 1] = c;
      col[pos + 1] = r;
      val[pos + 1] = v;
    }
    pos += k;
  }
}

std::string lower(std::string s) {
  for (auto& ch : s) ch = (char)std::tolower((unsigned char)ch);
  return s;
}

[[noreturn]] void parse_fail(const std::string& path, int64_t line, const std::string& msg) {
  raise(SFG_ERR_PARSE, path + ":" + std::to_string(line) + ": " + msg);
}

// The reference's per-line rules (io.hpp:96-114), for the lines the device
// left to the host.
struct HostLine {
  int32_t r = 0, c = 0;
  float v = 1.f;
  uint8_t cnt = 0, st = kOk;
};

HostLine host_parse(const std::string& line, int64_t rows, int64_t cols, bool pattern, bool symmetric) {
  HostLine h;
  if (!line.empty() && line[0] == '%') return h;
  if (line.find_first_not_of(" \t\r") == std::string::npos) return h;
  std::istringstream es(line);
  int64_t r = 0, c = 0;
  double v = 1.0;
  if (!(es >> r >> c)) {
    h.st = kBadEntry;
    return h;
  }
  if (!pattern && !(es >> v)) {
    h.st = kMissingValue;
    return h;
  }
  if (r < 1 || r > rows || c < 1 || c > cols) {
    h.st = kOutOfRange;
    return h;
  }
  h.cnt = (symmetric && r != c) ? 2 : 1;
  h.r = (int32_t)(r - 1);
  h.c = (int32_t)(c - 1);
  h.v = (float)v;
  return h;
}

}  // namespace

// File -> the context's pinned staging (grow-only) by parallel preads; with
// `dev`, each chunk is also queued for a device copy as soon as it is read.
char* read_file_pinned(sfg_context* ctx, const char* path_c, int64_t* size_out, char** dev) {
  const std::string path(path_c);
  const int fd = ::open(path_c, O_RDONLY);
  if (fd < 0) raise(SFG_ERR_IO, "cannot open " + path);
  struct stat stt;
  if (::fstat(fd, &stt) != 0) {
    ::close(fd);
    raise(SFG_ERR_IO, "cannot open " + path);
  }
  const int64_t size = stt.st_size;
  if ((size_t)size + 1 > ctx->staging_bytes) {
    cudaStreamSynchronize(ctx->stream);  // earlier copies may still read it
    if (ctx->staging) cudaFreeHost(ctx->staging);
    ctx->staging = nullptr;
    ctx->staging_bytes = 0;
    const size_t want = (size_t)size + 1 + ((size_t)size >> 3);
    if (cudaMallocHost(&ctx->staging, want) != cudaSuccess) {
      cudaGetLastError();
      ::close(fd);
      raise(SFG_ERR_OOM, "pinned staging of " + std::to_string(want) + " bytes failed");
    }
    ctx->staging_bytes = want;
  } else {
    cudaStreamSynchronize(ctx->stream);  // the staging is about to be overwritten
  }
  char* host = ctx->staging;
  char* dcopy = (dev && size) ? static_cast<char*>(dalloc(ctx, size)) : nullptr;
  constexpr int64_t kChunk = 32 << 20;
  const int64_t nchunks = (size + kChunk - 1) / kChunk;
  const int nthreads = (int)std::min<int64_t>(nchunks, 8);
  std::atomic<int64_t> next{0};
  std::atomic<bool> bad{false};
  std::vector<std::thread> pool;
  for (int w = 0; w < nthreads; ++w)
    pool.emplace_back([&] {
      for (int64_t k = next++; k < nchunks; k = next++) {
        const int64_t off = k * kChunk, len = std::min(kChunk, size - off);
        int64_t done = 0;
        while (done < len) {
          ssize_t got = ::pread(fd, host + off + done, (size_t)(len - done), off + done);
          if (got <= 0) {
            bad = true;
            return;
          }
          done += got;
        }
        if (dcopy && cudaMemcpyAsync(dcopy + off, host + off, len, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
          bad = true;
      }
    });
  for (auto& th : pool) th.join();
  ::close(fd);
  if (bad) {
    cudaGetLastError();
    cudaStreamSynchronize(ctx->stream);
    dfree(ctx, dcopy);
    raise(SFG_ERR_IO, "cannot read " + path);
  }
  host[size] = 0;
  *size_out = size;
  if (dev) *dev = dcopy;
  return host;
}

sfg_tensor* read_matrix_market(sfg_context* ctx, const char* path_c, bool sum_duplicates) {
  static const bool trace = std::getenv("SFG_TRACE_MM") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(ctx->stream);
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[mm] %-12s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_start).count());
    t_start = now;
  };
  const std::string path(path_c);
  int64_t size = 0;
  char* dtext_all = nullptr;
  char* host = read_file_pinned(ctx, path_c, &size, &dtext_all);
  host[size] = 0;
  mark("read file");

  // ---- header on the host (io.hpp:59-90)
  int64_t pos = 0, lineno = 0;
  auto next_line = [&](std::string& out) {
    if (pos >= size) return false;
    int64_t e = pos;
    while (e < size && host[e] != '\n') ++e;
    out.assign(host + pos, host + e);
    pos = e < size ? e + 1 : size;
    return true;
  };
  std::string line;
  if (!next_line(line)) parse_fail(path, 1, "empty file");
  ++lineno;
  std::istringstream head(line);
  std::string banner, object, format, field, symmetry;
  head >> banner >> object >> format >> field >> symmetry;
  if (banner != "%%MatrixMarket") parse_fail(path, lineno, "missing MatrixMarket banner");
  object = lower(object);
  format = lower(format);
  field = lower(field);
  symmetry = lower(symmetry);
  if (object != "matrix") raise(SFG_ERR_UNSUPPORTED_HEADER, path + ": unsupported object: " + object);
  if (format != "coordinate") raise(SFG_ERR_UNSUPPORTED_HEADER, path + ": unsupported format: " + format);
  if (field != "real" && field != "integer" && field != "pattern")
    raise(SFG_ERR_UNSUPPORTED_HEADER, path + ": unsupported field: " + field);
  if (symmetry != "general" && symmetry != "symmetric")
    raise(SFG_ERR_UNSUPPORTED_HEADER, path + ": unsupported symmetry: " + symmetry);
  const bool pattern = field == "pattern";
  const bool symmetric = symmetry == "symmetric";
  int64_t rows = 0, cols = 0, declared = 0;
  for (;;) {
    if (!next_line(line)) parse_fail(path, lineno + 1, "missing size line");
    ++lineno;
    if (!line.empty() && line[0] == '%') continue;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::istringstream sz(line);
    if (!(sz >> rows >> cols >> declared)) parse_fail(path, lineno, "bad size line");
    break;
  }
  if (rows < 0 || cols < 0 || declared < 0) parse_fail(path, lineno, "negative size");
  const int64_t body_line0 = lineno + 1;  // file line number of body line 0

  // ---- body on the device (the file is already there: body = text + pos)
  const int64_t nbytes = size - pos;
  int64_t nlines = 0;
  int64_t* start = nullptr;
  const char* text = dtext_all + pos;
  if (nbytes > 0) {
    auto* cnt = static_cast<unsigned long long*>(scratch(ctx, 64));
    SFG_CUDA(cudaMemsetAsync(cnt, 0, 8, ctx->stream));
    // newlines in file[0, size - 1) (aligned loads over the whole file),
    // less the header's: each of its `lineno` lines ended in one
    SFG_LAUNCH(k_count_newlines, stream_grid(ctx, ceil_div(size, 16), kBlock, 1, 8), kBlock, 0, ctx->stream,
               dtext_all, size - 1, cnt);
    unsigned long long nl = 0;
    read_back(ctx, cnt, 8, &nl);
    nlines = (int64_t)nl - lineno + 1;  // a '\n' before the last byte starts a line
    mark("h2d + count");
    start = dalloc_n<int64_t>(ctx, nlines);
    const int tiles = (int)ceil_div(nbytes, kLineTile);
    SFG_LAUNCH(k_mm_lines, tiles, kBlock, 0, ctx->stream, text, nbytes, start, lookback_status(ctx, tiles),
               ctx->epoch++);
  }
  int32_t* lr = dalloc_n<int32_t>(ctx, nlines);
  int32_t* lc = dalloc_n<int32_t>(ctx, nlines);
  float* lv = dalloc_n<float>(ctx, nlines);
  uint8_t* lcnt = static_cast<uint8_t*>(dalloc(ctx, nlines + 1));
  uint8_t* lst = static_cast<uint8_t*>(dalloc(ctx, nlines + 1));
  int64_t* hard = dalloc_n<int64_t>(ctx, nlines);
  auto* counters = static_cast<unsigned long long*>(dalloc(ctx, 32));
  void* owned[] = {dtext_all, start, lr, lc, lv, lcnt, lst, hard, counters};
  auto cleanup = [&] {  // idempotent
    for (void*& p : owned) {
      dfree(ctx, p);
      p = nullptr;
    }
  };
  try {
    SFG_CUDA(cudaMemsetAsync(counters, 0, 32, ctx->stream));
    if (nlines)
      SFG_LAUNCH(k_mm_parse, stream_grid(ctx, nlines, kBlock, 1, 8), kBlock, 0, ctx->stream, text, nbytes, start,
                 nlines, rows, cols, pattern ? 1 : 0, symmetric ? 1 : 0, lr, lc, lv, lcnt, lst, hard, counters);
    unsigned long long nh = 0;
    read_back(ctx, counters, 8, &nh);
    mark("lines+parse");
    if (nh) {
      // lines the device declined: parse them here with the reference's rules
      std::vector<int64_t> hl(nh), st_off(nh), en_off(nh);
      SFG_CUDA(cudaMemcpyAsync(hl.data(), hard, nh * 8, cudaMemcpyDeviceToHost, ctx->stream));
      SFG_CUDA(cudaStreamSynchronize(ctx->stream));
      std::vector<int64_t> starts(nlines);
      SFG_CUDA(cudaMemcpyAsync(starts.data(), start, nlines * 8, cudaMemcpyDeviceToHost, ctx->stream));
      SFG_CUDA(cudaStreamSynchronize(ctx->stream));
      std::vector<int32_t> hr(nh), hc(nh);
      std::vector<float> hv(nh);
      std::vector<uint8_t> hcnt(nh), hst(nh);
      for (size_t i = 0; i < nh; ++i) {
        const int64_t l = hl[i];
        int64_t s = starts[l], e = l + 1 < nlines ? starts[l + 1] - 1 : nbytes;
        if (e > s && host[pos + e - 1] == '\n') --e;
        HostLine h = host_parse(std::string(host + pos + s, host + pos + e), rows, cols, pattern, symmetric);
        hr[i] = h.r;
        hc[i] = h.c;
        hv[i] = h.v;
        hcnt[i] = h.cnt;
        hst[i] = h.st;
      }
      int64_t* dl = dalloc_n<int64_t>(ctx, nh);
      int32_t* dr = dalloc_n<int32_t>(ctx, nh);
      int32_t* dc = dalloc_n<int32_t>(ctx, nh);
      float* dv = dalloc_n<float>(ctx, nh);
      uint8_t* dcnt = static_cast<uint8_t*>(dalloc(ctx, nh));
      uint8_t* dst = static_cast<uint8_t*>(dalloc(ctx, nh));
      SFG_CUDA(cudaMemcpyAsync(dl, hl.data(), nh * 8, cudaMemcpyHostToDevice, ctx->stream));
      SFG_CUDA(cudaMemcpyAsync(dr, hr.data(), nh * 4, cudaMemcpyHostToDevice, ctx->stream));
      SFG_CUDA(cudaMemcpyAsync(dc, hc.data(), nh * 4, cudaMemcpyHostToDevice, ctx->stream));
      SFG_CUDA(cudaMemcpyAsync(dv, hv.data(), nh * 4, cudaMemcpyHostToDevice, ctx->stream));
      SFG_CUDA(cudaMemcpyAsync(dcnt, hcnt.data(), nh, cudaMemcpyHostToDevice, ctx->stream));
      SFG_CUDA(cudaMemcpyAsync(dst, hst.data(), nh, cudaMemcpyHostToDevice, ctx->stream));
      SFG_LAUNCH(k_mm_patch, stream_grid(ctx, nh, kBlock, 1, 8), kBlock, 0, ctx->stream, dl, dr, dc, dv, dcnt, dst,
                 (int64_t)nh, lr, lc, lv, lcnt, lst);
      SFG_CUDA(cudaStreamSynchronize(ctx->stream));  // host vectors die at scope end
      for (void* p : {(void*)dl, (void*)dr, (void*)dc, (void*)dv, (void*)dcnt, (void*)dst}) dfree(ctx, p);
    }
    // first failing line, entry lines
    SFG_CUDA(cudaMemsetAsync(counters, 0xff, 8, ctx->stream));
    SFG_CUDA(cudaMemsetAsync(counters + 1, 0, 8, ctx->stream));
    if (nlines)
      SFG_LAUNCH(k_mm_check, stream_grid(ctx, nlines, kBlock, 4, 8), kBlock, 0, ctx->stream, lst, lcnt, nlines,
                 counters);
    unsigned long long chk[2];
    read_back(ctx, counters, 16, chk);
    if (chk[0] != ~0ull) {
      uint8_t st = 0;
      read_back(ctx, lst + chk[0], 1, &st);
      const int64_t ln = body_line0 + (int64_t)chk[0];
      parse_fail(path, ln, st == kBadEntry ? "bad entry line" : st == kMissingValue ? "missing value"
                                                                                      : "coordinate out of range");
    }
    const int64_t seen = (int64_t)chk[1];
    if (seen != declared)
      parse_fail(path, body_line0 + nlines - 1,
                 "entry count " + std::to_string(seen) + " does not match declared " + std::to_string(declared));
    if (rows >= INT32_MAX || cols >= INT32_MAX)
      raise(SFG_ERR_INVALID_OPERATION, "extent or nnz exceeds the int32 index range");
  } catch (...) {
    cleanup();
    throw;
  }
  // entries in file order, then the device from_coo
  int64_t total = 0;
  int32_t* row = nullptr;
  int32_t* col = nullptr;
  float* val = nullptr;
  sfg_tensor* t = nullptr;
  try {
    // mirrored entries: count them from the per-line counts (device scan)
    const int tiles = (int)std::max<int64_t>(1, ceil_div(nlines, kEmitTile));
    int64_t upper = symmetric ? 2 * declared : declared;
    row = dalloc_n<int32_t>(ctx, upper);
    col = dalloc_n<int32_t>(ctx, upper);
    val = dalloc_n<float>(ctx, upper);
    if (nlines)
      SFG_LAUNCH(k_mm_emit, tiles, kBlock, 0, ctx->stream, lr, lc, lv, lcnt, nlines, row, col, val,
                 lookback_status(ctx, tiles), ctx->epoch++);
    if (symmetric) {
      // total = declared + off-diagonal entries: from the emit scan's last
      // inclusive prefix (the look-back status of the last tile)
      unsigned long long w = 0;
      read_back(ctx, lookback_status(ctx, tiles) + (tiles - 1), 8, &w);
      total = (int64_t)(uint32_t)w;
    } else {
      total = declared;
    }
    if (total >= INT32_MAX) raise(SFG_ERR_INVALID_OPERATION, "extent or nnz exceeds the int32 index range");
    cleanup();
    mark("check+emit");
    t = sort_coo(ctx, rows, cols, total, row, col, val, sum_duplicates);
    mark("from_coo");
  } catch (...) {
    cleanup();
    dfree(ctx, row);
    dfree(ctx, col);
    dfree(ctx, val);
    throw;
  }
  dfree(ctx, row);
  dfree(ctx, col);
  dfree(ctx, val);
  return t;
}

}  // namespace sfg
