// sparseforge_b200/sparseforge.hpp — drop-in C++ host API for the B200 path.
//
// Mirrors the reference's proj/include/sparseforge API for the hot path
// (names, argument meaning, ErrorKind errors) so reference-style code such as
//
//   WorkingTensor t = from_coo(TensorShape{{m, n}}, coords, values);   // tensor.hpp:118
//   FormatEncoding enc = resolve_format("CSR");                          // formats.hpp:92
//   convert_structure(t, resolve_format("COO"), enc);                    // planner.hpp:261
//   MaterializedTensor mat = materialize(t, infer_storage(enc));         // storage.hpp:97
//   DenseTensor y = run_kernel(spmv_kernel(),                            // kernel.hpp:236
//       {KernelOperand::from_materialized(enc, mat), KernelOperand::from_dense(x)});
//
// compiles against this header (namespace sparseforge) and runs on the GPU
// through the C-ABI (include/sparseforge_b200.h, libsfg.so). Tensors live in
// device memory; host arrays (int64 idx/ptr, f64 values, like the reference)
// are produced by materialize(). Differences from the reference are listed in
// indices must fit int32, values are stored as fp32 (bf16
// optional for BCSR), kernels accumulate in fp32, and the device planner
// covers COO sources to COO/CSR/CSC/DCSR/ELL/BCSR(r,c) plus the hybrid pair.
#pragma once

#include <algorithm>
#include <array>
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../sparseforge_b200.h"

namespace sparseforge {

// ------------------------------------------------------------ errors.hpp
enum class ErrorKind {
  Parse,
  NonAffine,
  NonIntegral,
  UnsupportedSource,
  UnsupportedHeader,
  DuplicateCoordinate,
  Collision,
  InvalidOperation,
  Singular,
  Io,
};

class Error : public std::runtime_error {
 public:
  Error(ErrorKind kind, const std::string& message) : std::runtime_error(message), kind_(kind) {}
  ErrorKind kind() const { return kind_; }

 private:
  ErrorKind kind_;
};

// Device failures (no reference equivalent).
class DeviceError : public std::runtime_error {
 public:
  DeviceError(int status, const std::string& message)
      : std::runtime_error(message), status_(status) {}
  int status() const { return status_; }

 private:
  int status_;
};

[[noreturn]] inline void fail(ErrorKind kind, const std::string& message) { throw Error(kind, message); }

namespace b200 {
inline void check(int status) {
  if (status == SFG_OK) return;
  std::string msg = sfg_last_error();
  if (status >= 1 && status <= 10) throw Error(static_cast<ErrorKind>(status - 1), msg);
  throw DeviceError(status, msg);
}

// One context per process by default (device 0, default stream). Replace it
// with set_default_context() to run on another device or stream.
class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) { check(sfg_context_create(device, stream, &h_)); }
  ~Context() {
    if (h_) sfg_context_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  sfg_context* get() const { return h_; }

 private:
  sfg_context* h_ = nullptr;
};

inline std::shared_ptr<Context>& default_context_slot() {
  static std::shared_ptr<Context> ctx;
  return ctx;
}
inline Context& default_context() {
  auto& slot = default_context_slot();
  if (!slot) slot = std::make_shared<Context>(0, nullptr);
  return *slot;
}
inline void set_default_context(std::shared_ptr<Context> ctx) { default_context_slot() = std::move(ctx); }

struct TensorHandle {
  sfg_tensor* h = nullptr;
  explicit TensorHandle(sfg_tensor* t) : h(t) {}
  ~TensorHandle() {
    if (h) sfg_tensor_free(h);
  }
  TensorHandle(const TensorHandle&) = delete;
  TensorHandle& operator=(const TensorHandle&) = delete;
};
}  // namespace b200

// ------------------------------------------------------------ tensor.hpp
struct TensorShape {
  std::vector<std::int64_t> extents;
  size_t rank() const { return extents.size(); }
  std::int64_t volume() const {
    std::int64_t v = 1;
    for (auto e : extents) v *= e;
    return v;
  }
};

struct DenseTensor {
  TensorShape shape;
  std::vector<double> data;
  explicit DenseTensor(TensorShape s = {})
      : shape(std::move(s)), data(static_cast<size_t>(shape.volume()), 0.0) {}
  size_t offset(const std::vector<std::int64_t>& coords) const {
    size_t off = 0;
    for (size_t i = 0; i < shape.rank(); ++i) {
      if (coords[i] < 0 || coords[i] >= shape.extents[i])
        fail(ErrorKind::InvalidOperation, "dense coordinate out of range");
      off = off * static_cast<size_t>(shape.extents[i]) + static_cast<size_t>(coords[i]);
    }
    return off;
  }
  double at(const std::vector<std::int64_t>& c) const { return data[offset(c)]; }
  double& at(const std::vector<std::int64_t>& c) { return data[offset(c)]; }
};

// ---------------------------------------------------------- formats.hpp
struct FormatEncoding {
  sfg_format fmt{};
  std::string name;  // canonical registry name, e.g. "BCSR(4,4)"
};

namespace b200 {
inline std::string strip(const std::string& s) {
  std::string t;
  for (char c : s)
    if (!std::isspace(static_cast<unsigned char>(c))) t += c;
  return t;
}
inline std::string name_of(const sfg_format& f) {
  switch (f.kind) {
    case SFG_COO: return "COO";
    case SFG_CSR: return "CSR";
    case SFG_CSC: return "CSC";
    case SFG_DCSR: return "DCSR";
    case SFG_ELL: return "ELL";
    case SFG_BCSR: return "BCSR(" + std::to_string(f.block_r) + "," + std::to_string(f.block_c) + ")";
    case SFG_HYB: return "HYB(" + std::to_string(f.threshold) + ")";
    case SFG_DOK: return "DOK";
    case SFG_LIL: return "LIL";
    case SFG_BELL: return "BELL(" + std::to_string(f.block_r) + ")";
    case SFG_DIA: return "DIA";
    case SFG_BDIA: return "BDIA(" + std::to_string(f.block_r) + ")";
    case SFG_C2SR: return "C2SR(" + std::to_string(f.block_r) + ")";
    case SFG_CSB: return "CSB(" + std::to_string(f.block_r) + "," + std::to_string(f.block_c) + ")";
    case SFG_HBELL: return "HBELL(" + std::to_string(f.block_r) + "," + std::to_string(f.threshold) + ")";
    case SFG_DCSC: return "DCSC";
    case SFG_DIAV: return "DIA-variant";
    case SFG_CISR: return "CISR(" + std::to_string(f.block_r) + ")";
    case SFG_CISRP: return "CISR-plus(" + std::to_string(f.block_r) + ")";
  }
  return "?";
}
}  // namespace b200

// resolve_format (formats.hpp:92-125): registry names, plus the raw encoding
// texts of those names (formats.hpp:39-61), e.g. the coordinate encoding
// "map (d0, d1) -> (d0, d1); trim(0,1)".
inline FormatEncoding resolve_format(const std::string& text) {
  std::string t = b200::strip(text);
  if (t.rfind("map", 0) == 0) {
    static const std::pair<const char*, const char*> known[] = {
        {"map(d0,d1)->(d0,d1);trim(0,1)", "COO"},
        {"map(d0,d1)->(d0,d1)trim(0,1)", "COO"},
        {"map(d0,d1)->(d0,d1);merge(0),trim(1,1)", "CSR"},
        {"map(d0,d1)->(d1,d0);merge(0),trim(1,1)", "CSC"},
        {"map(d0,d1)->(d0,d1);merge(0),trim(0,1)", "DCSR"},
        {"map(d0,d1)->(d1,d0);merge(0),trim(0,1)", "DCSC"},
        {"map(d0,d1)->(d1-d0,d0);merge(0),trim(0,0)", "DIA"},
        {"map(d0,d1)->(d1-d0,d1);merge(0),trim(0,0)", "DIA-variant"},
        {"map(d0,d1)->(d0,d1);trim(0,1),pack(0,1)", "DOK"},
        {"map(d0,d1)->(d0,d1);merge(0),trim(1,1),pack(0,1)", "LIL"},
    };
    for (const auto& [enc, name] : known)
      if (t == enc) return resolve_format(name);
    if (t.find("indirect(d1),d0,d1") != std::string::npos && t.find("enum(value)") != std::string::npos)
      return resolve_format("ELL");
    long r = 0, c = 0, r2 = 0, c2 = 0;
    if (std::sscanf(t.c_str(), "map(d0,d1)->(d0/%ld,d1/%ld,d0%%%ld,d1%%%ld);merge(0),trim(1,1)", &r, &c,
                    &r2, &c2) == 4 &&
        r == r2 && c == c2)
      return resolve_format("BCSR(" + std::to_string(r) + "," + std::to_string(c) + ")");
    fail(ErrorKind::Parse, "encoding not covered by the B200 path: " + text);
  }
  FormatEncoding e;
  b200::check(sfg_format_resolve(text.c_str(), &e.fmt));
  e.name = b200::name_of(e.fmt);
  return e;
}

// ---------------------------------------------------------- storage.hpp
struct LevelStorage {
  bool size = false;
  bool ptr = false;
  bool idx = false;
  bool dense_vector = false;
};

struct StorageScheme {
  std::vector<LevelStorage> levels;
  FormatEncoding enc;
};

struct Interval {
  std::int64_t lo = 0;
  std::int64_t hi = -1;
  std::int64_t extent() const { return hi < lo ? 0 : hi - lo + 1; }
};

struct MaterializedLevel {
  LevelStorage storage;
  Interval bounds;
  size_t node_count = 0;
  std::vector<std::int64_t> idx;
  std::vector<std::int64_t> ptr;
};

// infer_storage (storage.hpp:35-51) for the covered formats.
inline StorageScheme infer_storage(const FormatEncoding& enc) {
  StorageScheme s;
  s.enc = enc;
  auto L = [](bool size, bool ptr, bool idx, bool dv) { return LevelStorage{size, ptr, idx, dv}; };
  switch (enc.fmt.kind) {
    case SFG_COO:
    case SFG_DOK: s.levels = {L(0, 0, 1, 0), L(0, 0, 1, 0)}; break;
    case SFG_CSR:
    case SFG_LIL:
    case SFG_CSC: s.levels = {L(1, 0, 0, 0), L(0, 1, 1, 0)}; break;
    case SFG_DCSR:
    case SFG_DCSC: s.levels = {L(0, 0, 1, 0), L(0, 1, 1, 0)}; break;
    case SFG_ELL: s.levels = {L(0, 0, 1, 0), L(1, 0, 0, 0), L(0, 0, 1, 0)}; break;
    case SFG_BCSR: s.levels = {L(1, 0, 0, 0), L(0, 1, 1, 0), L(1, 0, 0, 1), L(1, 0, 0, 1)}; break;
    case SFG_BELL:
      s.levels = {L(0, 0, 1, 0), L(1, 0, 0, 0), L(0, 0, 1, 0), L(1, 0, 0, 1), L(1, 0, 0, 1)};
      break;
    case SFG_DIA:
    case SFG_DIAV: s.levels = {L(0, 0, 1, 0), L(1, 0, 0, 1)}; break;
    case SFG_BDIA: s.levels = {L(1, 0, 0, 0), L(0, 1, 1, 0), L(1, 0, 0, 1)}; break;
    case SFG_C2SR: s.levels = {L(1, 0, 0, 0), L(1, 0, 0, 0), L(0, 1, 1, 0)}; break;
    case SFG_CISR:
    case SFG_CISRP: s.levels = {L(0, 0, 1, 0), L(0, 1, 1, 0), L(0, 1, 1, 0)}; break;
    case SFG_CSB: s.levels = {L(1, 0, 0, 0), L(1, 0, 0, 0), L(0, 1, 1, 0), L(0, 0, 1, 0)}; break;
    default: break;  // HYB: two parts, see DecomposeResult
  }
  return s;
}

inline std::string explain_storage(const StorageScheme& s) {
  char buf[512];
  b200::check(sfg_storage_explain(&s.enc.fmt, buf, sizeof buf));
  return buf;
}

// ----------------------------------------------------- WorkingTensor etc.
// The reference's expanded form is replaced by a device-resident handle: a
// canonical COO after from_coo, the target format after apply_plan.
struct WorkingTensor {
  TensorShape shape;
  FormatEncoding enc;  // current structure
  std::shared_ptr<b200::TensorHandle> dev;

  size_t level_count() const {
    switch (enc.fmt.kind) {
      case SFG_ELL: return 3;
      case SFG_BCSR: return 4;
      case SFG_BELL: return 5;
      case SFG_CSB: return 4;
      case SFG_BDIA:
      case SFG_C2SR:
      case SFG_CISR:
      case SFG_CISRP: return 3;
      default: return 2;
    }
  }
  size_t entry_count() const {
    sfg_tensor_view v;
    b200::check(sfg_tensor_view_get(b200::default_context().get(), dev->h, &v));
    return static_cast<size_t>(v.nvals);
  }
  // Host copy of the canonical COO columns and values (tensor.hpp:70-96).
  void download(std::vector<std::vector<std::int64_t>>& coords, std::vector<double>& values) const;
};

// ValueLayout (tensor.hpp:58-64): AoS over levels [aos_start, aos_end] after
// Pack (operators.hpp:424-430); DOK and LIL carry pack(0,1).
enum class ValueLayoutKind { SoA, AoS };
struct ValueLayout {
  ValueLayoutKind kind = ValueLayoutKind::SoA;
  size_t aos_start = 0;
  size_t aos_end = 0;
};

struct MaterializedTensor {
  TensorShape logical_shape;
  std::vector<MaterializedLevel> levels;
  std::vector<double> values;
  ValueLayout layout;
  std::vector<std::pair<size_t, size_t>> partitions;  // Partition value ranges (storage.hpp:90)
  FormatEncoding enc;
  std::shared_ptr<b200::TensorHandle> dev;  // the device arrays behind the host copy
};

namespace b200 {
template <class T>
std::vector<T> download_array(const void* dev, int64_t count) {
  std::vector<T> out(static_cast<size_t>(count));
  if (count > 0)
    check(sfgx_copy(default_context().get(), out.data(), dev, count * static_cast<int64_t>(sizeof(T)), 1));
  return out;
}
// count elements at dev[i * stride] (stride > 1: a field of packed records)
template <class T>
std::vector<T> download_strided(const void* dev, int64_t count, int64_t stride) {
  if (stride <= 1) return download_array<T>(dev, count);
  std::vector<T> rec = download_array<T>(dev, count > 0 ? (count - 1) * stride + 1 : 0);
  std::vector<T> out(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) out[static_cast<size_t>(i)] = rec[static_cast<size_t>(i * stride)];
  return out;
}
inline std::vector<std::int64_t> widen(const std::vector<std::int32_t>& v) {
  return std::vector<std::int64_t>(v.begin(), v.end());
}
inline std::vector<double> download_values(const sfg_tensor_view& v) {
  if (v.value_dtype == SFG_BF16) {
    auto raw = download_array<std::uint16_t>(v.values, v.nvals);
    std::vector<double> out(raw.size());
    for (size_t i = 0; i < raw.size(); ++i) {
      std::uint32_t bits = static_cast<std::uint32_t>(raw[i]) << 16;
      float f;
      std::memcpy(&f, &bits, 4);
      out[i] = f;
    }
    return out;
  }
  auto f = download_strided<float>(v.values, v.nvals, v.layout == 1 ? v.record_words : 1);
  return std::vector<double>(f.begin(), f.end());
}
}  // namespace b200

inline void WorkingTensor::download(std::vector<std::vector<std::int64_t>>& coords,
                                    std::vector<double>& values) const {
  if (enc.fmt.kind != SFG_COO) fail(ErrorKind::InvalidOperation, "download expects coordinate form");
  sfg_tensor_view v;
  b200::check(sfg_tensor_view_get(b200::default_context().get(), dev->h, &v));
  coords = {b200::widen(b200::download_array<std::int32_t>(v.level[0].idx, v.level[0].idx_len)),
            b200::widen(b200::download_array<std::int32_t>(v.level[1].idx, v.level[1].idx_len))};
  values = b200::download_values(v);
}

// from_coo (tensor.hpp:118-162): range check, stable sort, duplicates
// rejected (DuplicateCoordinate) or summed (f64, rounded once to fp32).
inline WorkingTensor from_coo(TensorShape shape, const std::vector<std::vector<std::int64_t>>& coords,
                              const std::vector<double>& values, bool sum_duplicates = false) {
  if (coords.size() != shape.rank() || shape.rank() != 2)
    fail(ErrorKind::InvalidOperation, "coordinate rank mismatch (the B200 path handles matrices)");
  const size_t nnz = values.size();
  if (coords[0].size() != nnz || coords[1].size() != nnz)
    fail(ErrorKind::InvalidOperation, "tensor columns out of sync");
  std::vector<std::int32_t> r(nnz), c(nnz);
  std::vector<float> v(nnz);
  for (size_t e = 0; e < nnz; ++e) {
    if (coords[0][e] < 0 || coords[0][e] >= shape.extents[0] || coords[1][e] < 0 ||
        coords[1][e] >= shape.extents[1])
      fail(ErrorKind::InvalidOperation, "coordinate out of range");
    r[e] = static_cast<std::int32_t>(coords[0][e]);
    c[e] = static_cast<std::int32_t>(coords[1][e]);
    v[e] = static_cast<float>(values[e]);
  }
  sfg_tensor* h = nullptr;
  std::uint32_t flags = SFG_FLAG_HOST | (sum_duplicates ? std::uint32_t(SFG_FLAG_SUM_DUPLICATES) : 0u);
  b200::check(sfg_from_coo(b200::default_context().get(), shape.extents[0], shape.extents[1],
                           static_cast<int64_t>(nnz), r.data(), c.data(), v.data(), flags, &h));
  WorkingTensor t;
  t.shape = std::move(shape);
  t.enc = resolve_format("COO");
  t.dev = std::make_shared<b200::TensorHandle>(h);
  return t;
}

// -------------------------------------------------------------- io.hpp
// read_matrix_market (io.hpp:50-121). The file is parsed on the device;
// CooData holds the entries in canonical (row, col) order — from_coo of it
// gives the same tensor as from_coo of the reference's file-order CooData.
struct CooData {
  TensorShape shape;
  std::vector<std::vector<std::int64_t>> coords;
  std::vector<double> values;
};

// The device path end to end: file -> canonical COO WorkingTensor (what the
// reference's CLI builds with read_matrix_market + from_coo).
inline WorkingTensor load_matrix_market(const std::string& path, bool sum_duplicates = false) {
  sfg_tensor* h = nullptr;
  b200::check(sfg_read_matrix_market(b200::default_context().get(), path.c_str(),
                                     sum_duplicates ? std::uint32_t(SFG_FLAG_SUM_DUPLICATES) : 0u, &h));
  sfg_tensor_view v;
  b200::check(sfg_tensor_view_get(b200::default_context().get(), h, &v));
  WorkingTensor t;
  t.shape = TensorShape{{v.rows, v.cols}};
  t.enc = resolve_format("COO");
  t.dev = std::make_shared<b200::TensorHandle>(h);
  return t;
}

inline CooData read_matrix_market(const std::string& path) {
  WorkingTensor t = load_matrix_market(path);  // duplicates: DuplicateCoordinate, as from_coo would
  CooData d;
  d.shape = t.shape;
  t.download(d.coords, d.values);
  return d;
}

// Host-side text utilities of io.hpp, same formats and messages: Matrix
// Market output (io.hpp:123-134, values as %.17g), FROSTT .tns input
// (151-184), one value per line vectors (186-202).
namespace b200 {
inline std::string format_value(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}
inline void write_text(const std::string& path, const std::string& text) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) fail(ErrorKind::Io, "cannot write " + path);
  const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
  if (std::fclose(f) != 0 || !ok) fail(ErrorKind::Io, "write failed: " + path);
}
}  // namespace b200

inline void write_matrix_market(const std::string& path, const CooData& d) {
  if (d.shape.rank() != 2) fail(ErrorKind::InvalidOperation, "matrix market output is rank-2");
  std::string out = "%%MatrixMarket matrix coordinate real general\n";
  out += std::to_string(d.shape.extents[0]) + " " + std::to_string(d.shape.extents[1]) + " " +
         std::to_string(d.values.size()) + "\n";
  for (size_t e = 0; e < d.values.size(); ++e)
    out += std::to_string(d.coords[0][e] + 1) + " " + std::to_string(d.coords[1][e] + 1) + " " +
           b200::format_value(d.values[e]) + "\n";
  b200::write_text(path, out);
}

inline CooData read_tns(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(ErrorKind::Io, "cannot open " + path);
  auto bad = [&](size_t line, const std::string& msg) {
    fail(ErrorKind::Parse, path + ":" + std::to_string(line) + ": " + msg);
  };
  CooData out;
  std::string text;
  size_t line = 0, rank = 0;
  while (std::getline(in, text)) {
    ++line;
    if (!text.empty() && (text[0] == '#' || text[0] == '%')) continue;
    if (text.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::istringstream fields(text);
    std::vector<double> nums;
    for (double x; fields >> x;) nums.push_back(x);
    if (nums.size() < 2) bad(line, "need coordinates and a value");
    if (rank == 0) {
      rank = nums.size() - 1;
      out.coords.resize(rank);
      out.shape.extents.assign(rank, 0);
    } else if (nums.size() - 1 != rank) {
      bad(line, "inconsistent rank");
    }
    for (size_t k = 0; k < rank; ++k) {
      const auto c = static_cast<std::int64_t>(nums[k]);
      if (c < 1) bad(line, "coordinates are 1-based");
      out.coords[k].push_back(c - 1);
      out.shape.extents[k] = std::max(out.shape.extents[k], c);
    }
    out.values.push_back(nums.back());
  }
  if (rank == 0) bad(line ? line : 1, "no entries");
  return out;
}

inline std::vector<double> read_vector_text(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(ErrorKind::Io, "cannot open " + path);
  std::vector<double> out;
  for (double v; in >> v;) out.push_back(v);
  return out;
}

inline void write_vector_text(const std::string& path, const std::vector<double>& v) {
  std::string out;
  for (double x : v) out += b200::format_value(x) + "\n";
  b200::write_text(path, out);
}

// to_coo_data (io.hpp:136-149): the coordinates of a tensor whose map is
// the identity (COO, and CSR / DCSR / DOK / LIL brought back to COO on the
// device), in canonical order.
inline CooData to_coo_data(const WorkingTensor& t) {
  const int k = t.enc.fmt.kind;
  if (k != SFG_COO && k != SFG_CSR && k != SFG_DCSR && k != SFG_DOK && k != SFG_LIL)
    fail(ErrorKind::InvalidOperation, "tensor is not in coordinate form");
  CooData d;
  d.shape = t.shape;
  if (k == SFG_COO) {
    t.download(d.coords, d.values);
    return d;
  }
  sfg_format coo{};
  b200::check(sfg_format_resolve("COO", &coo));
  sfg_tensor* h = nullptr;
  b200::check(sfg_convert(b200::default_context().get(), t.dev->h, &coo, &h));
  WorkingTensor c;
  c.shape = t.shape;
  c.enc = resolve_format("COO");
  c.dev = std::make_shared<b200::TensorHandle>(h);
  c.download(d.coords, d.values);
  return d;
}

// from_dense (tensor.hpp:164-179): the nonzero cells in row-major order.
inline WorkingTensor from_dense(const DenseTensor& d) {
  if (d.shape.rank() != 2) fail(ErrorKind::InvalidOperation, "coordinate rank mismatch (the B200 path handles matrices)");
  std::vector<std::vector<std::int64_t>> coords(2);
  std::vector<double> values;
  const std::int64_t n = d.shape.extents[1];
  for (size_t off = 0; off < d.data.size(); ++off)
    if (d.data[off] != 0.0) {
      coords[0].push_back(static_cast<std::int64_t>(off) / n);
      coords[1].push_back(static_cast<std::int64_t>(off) % n);
      values.push_back(d.data[off]);
    }
  return from_coo(d.shape, coords, values);
}

// to_dense (tensor.hpp:184-201) for identity-mapped tensors: the nonzero
// values back in their cells (zero values, padding, are dropped).
inline DenseTensor to_dense(const WorkingTensor& t) {
  const CooData c = to_coo_data(t);
  DenseTensor out(t.shape);
  for (size_t e = 0; e < c.values.size(); ++e)
    if (c.values[e] != 0.0) out.at({c.coords[0][e], c.coords[1][e]}) = c.values[e];
  return out;
}

// equal_dense (tensor.hpp:203-211)
inline bool equal_dense(const DenseTensor& a, const DenseTensor& b, double tol = 0.0) {
  if (a.shape.extents != b.shape.extents) return false;
  for (size_t i = 0; i < a.data.size(); ++i) {
    const double diff = a.data[i] > b.data[i] ? a.data[i] - b.data[i] : b.data[i] - a.data[i];
    if (diff > tol) return false;
  }
  return true;
}

// write_container / read_container (io.hpp:240, 283): the USPT file of a
// materialized tensor, written from / read into device memory.
struct MaterializedTensor;
inline void write_container(const std::string& path, const MaterializedTensor& m);
inline MaterializedTensor read_container(const std::string& path);

// --------------------------------------------------------- planner.hpp
struct ConversionOp {
  std::string text;  // print_op form, e.g. "Fill(0)"
};
inline std::string print_op(const ConversionOp& op) { return op.text; }

struct ConversionPlan {
  std::vector<ConversionOp> ops;
  FormatEncoding src, dst;
};

inline std::vector<std::string> plan_lines(const ConversionPlan& plan) {
  std::vector<std::string> out;
  for (const auto& op : plan.ops) out.push_back(op.text);
  return out;
}

// plan_conversion (planner.hpp:95-252) for COO sources.
inline ConversionPlan plan_conversion(const FormatEncoding& src, const FormatEncoding& dst) {
  ConversionPlan p;
  p.src = src;
  p.dst = dst;
  // the op list as the reference prints it; from a compressed source the
  // device executes it by dematerializing and regrowing in one call
  // (convert_src.cu). Sources with indirect levels or a value layout raise
  // UnsupportedSource here, as in the reference (planner.hpp:96-99).
  if (src.fmt.kind == SFG_HYB) return p;  // the hybrid pair: two tensors, no single plan
  char buf[1024];
  b200::check(sfg_plan_text(&src.fmt, &dst.fmt, buf, sizeof buf));
  std::string s(buf);
  size_t pos = 0;
  while (pos < s.size()) {
    size_t nl = s.find('\n', pos);
    if (nl == std::string::npos) nl = s.size();
    if (nl > pos) p.ops.push_back({s.substr(pos, nl - pos)});
    pos = nl + 1;
  }
  return p;
}

// apply_plan (planner.hpp:254-257): executes the whole plan on the device.
inline void apply_plan(WorkingTensor& t, const ConversionPlan& plan) {
  if (t.enc.fmt.kind != plan.src.fmt.kind)
    fail(ErrorKind::InvalidOperation, "tensor structure does not match the plan source");
  if (plan.dst.fmt.kind == SFG_COO && plan.src.fmt.kind == SFG_COO) return;  // empty plan
  sfg_tensor* out = nullptr;
  b200::check(sfg_convert(b200::default_context().get(), t.dev->h, &plan.dst.fmt, &out));
  t.dev = std::make_shared<b200::TensorHandle>(out);
  t.enc = plan.dst;
  sfg_tensor_view v;  // a BCSR source regrows over its whole block grid
  b200::check(sfg_tensor_view_get(b200::default_context().get(), out, &v));
  t.shape = TensorShape{{v.rows, v.cols}};
}

inline void convert_structure(WorkingTensor& t, const FormatEncoding& src, const FormatEncoding& dst) {
  apply_plan(t, plan_conversion(src, dst));
}

// materialize (storage.hpp:97-234): the device already holds the compact
// arrays; this returns their host copy (int64 / f64) with the device handle.
inline MaterializedTensor materialize(const WorkingTensor& t, const StorageScheme& scheme) {
  if (scheme.enc.fmt.kind != t.enc.fmt.kind)
    fail(ErrorKind::InvalidOperation, "storage scheme rank mismatch");
  sfg_tensor_view v;
  b200::check(sfg_tensor_view_get(b200::default_context().get(), t.dev->h, &v));
  MaterializedTensor m;
  m.logical_shape = t.shape;
  m.enc = t.enc;
  m.dev = t.dev;
  for (int l = 0; l < v.nlevels; ++l) {
    const sfg_level_view& lv = v.level[l];
    MaterializedLevel ml;
    ml.storage = {(lv.storage & SFG_LEVEL_SIZE) != 0, (lv.storage & SFG_LEVEL_PTR) != 0,
                  (lv.storage & SFG_LEVEL_IDX) != 0, (lv.storage & SFG_LEVEL_DENSE_VECTOR) != 0};
    ml.bounds = {lv.lo, lv.hi};
    ml.node_count = static_cast<size_t>(lv.node_count);
    const bool packed = v.layout == 1 && l >= v.aos_start && l <= v.aos_end;
    ml.idx = b200::widen(b200::download_strided<std::int32_t>(lv.idx, lv.idx_len, packed ? v.record_words : 1));
    ml.ptr = b200::widen(b200::download_array<std::int32_t>(lv.ptr, lv.ptr_len));
    m.levels.push_back(std::move(ml));
  }
  m.values = b200::download_values(v);
  if (v.layout == 1)
    m.layout = {ValueLayoutKind::AoS, static_cast<size_t>(v.aos_start), static_cast<size_t>(v.aos_end)};
  for (int64_t q = 0; q < v.npartitions; ++q)
    m.partitions.push_back({static_cast<size_t>(v.partitions[2 * q]), static_cast<size_t>(v.partitions[2 * q + 1])});
  return m;
}

// dematerialize (storage.hpp:284-343): the working form behind a
// materialized tensor — on the B200 path, the device arrays it was
// downloaded from (or read into, read_container).
inline WorkingTensor dematerialize(const MaterializedTensor& m, const FormatEncoding& enc) {
  if (!m.dev) fail(ErrorKind::InvalidOperation, "materialized tensor without device arrays");
  if (m.enc.fmt.kind != enc.fmt.kind || m.levels.size() != infer_storage(enc).levels.size())
    fail(ErrorKind::InvalidOperation, "container rank does not match the encoding");
  WorkingTensor t;
  t.shape = m.logical_shape;
  t.enc = enc;
  t.dev = m.dev;
  return t;
}

inline void write_container(const std::string& path, const MaterializedTensor& m) {
  if (!m.dev) fail(ErrorKind::InvalidOperation, "the tensor has no device form");
  b200::check(sfg_write_container(b200::default_context().get(), m.dev->h, path.c_str()));
}

// The container does not name its format: the level kinds do (CSR is taken
// for the CSR / CSC look-alikes; pass the encoding to read a CSC).
inline MaterializedTensor read_container(const std::string& path, const FormatEncoding& enc) {
  sfg_tensor* h = nullptr;
  b200::check(sfg_read_container(b200::default_context().get(), path.c_str(), &enc.fmt, &h));
  WorkingTensor t;
  t.enc = enc;
  t.dev = std::make_shared<b200::TensorHandle>(h);
  sfg_tensor_view v;
  b200::check(sfg_tensor_view_get(b200::default_context().get(), h, &v));
  t.shape = TensorShape{{v.rows, v.cols}};
  return materialize(t, infer_storage(enc));
}

inline MaterializedTensor read_container(const std::string& path) {
  sfg_tensor* h = nullptr;
  b200::check(sfg_read_container(b200::default_context().get(), path.c_str(), nullptr, &h));
  sfg_tensor_view v;
  b200::check(sfg_tensor_view_get(b200::default_context().get(), h, &v));
  sfg_format f{};
  f.kind = v.kind;
  f.value_dtype = v.value_dtype;
  FormatEncoding enc;
  enc.fmt = f;
  WorkingTensor t;
  t.enc = enc;
  t.dev = std::make_shared<b200::TensorHandle>(h);
  t.shape = TensorShape{{v.rows, v.cols}};
  return materialize(t, infer_storage(enc));
}

// ------------------------------------------------------- decompose.hpp
// The device decompose covers the row-count rule
//   sum(value) groupBy (d0, d1) -> (d0) with value ne 0 -> 1 | otherwise -> 0
// (the count query of formats.hpp:20-23, used by ELL and the hybrid).
struct DecomposeRule {
  std::string query =
      "sum(value) groupBy (d0, d1) -> (d0) with value ne 0 -> 1 | otherwise -> 0";
  std::int64_t min_sum = 1;
};

using GroupKey = std::vector<std::int64_t>;

struct DecomposeResult {
  WorkingTensor selected;
  WorkingTensor remainder;
  std::map<GroupKey, std::int64_t> totals;
};

inline DecomposeResult decompose(const WorkingTensor& t, const DecomposeRule& rule) {
  if (b200::strip(rule.query) != b200::strip(DecomposeRule{}.query))
    fail(ErrorKind::InvalidOperation, "the device decompose covers the row-count rule only");
  if (t.enc.fmt.kind != SFG_COO) fail(ErrorKind::InvalidOperation, "decompose expects coordinate-form input");
  auto& ctx = b200::default_context();
  void* dtot = nullptr;
  b200::check(sfgx_device_alloc(ctx.get(), t.shape.extents[0] * 4, &dtot));
  sfg_tensor *s = nullptr, *r = nullptr;
  int st = sfg_decompose_rows(ctx.get(), t.dev->h, rule.min_sum, &s, &r, static_cast<int32_t*>(dtot));
  std::vector<std::int32_t> tot;
  if (st == SFG_OK) tot = b200::download_array<std::int32_t>(dtot, t.shape.extents[0]);
  sfgx_device_free(ctx.get(), dtot);
  b200::check(st);
  DecomposeResult out;
  out.selected = {t.shape, t.enc, std::make_shared<b200::TensorHandle>(s)};
  out.remainder = {t.shape, t.enc, std::make_shared<b200::TensorHandle>(r)};
  for (size_t i = 0; i < tot.size(); ++i) out.totals[{static_cast<std::int64_t>(i)}] = tot[i];
  return out;
}

// ---------------------------------------------------------- kernel.hpp
struct KernelSpec {
  std::string name;
};
inline KernelSpec spmv_kernel() { return {"spmv"}; }
inline KernelSpec spmm_kernel() { return {"spmm"}; }
inline KernelSpec spgemm_kernel() { return {"spgemm"}; }
inline KernelSpec builtin_kernel(const std::string& name) {
  if (name == "spmv" || name == "spmm" || name == "spgemm") return {name};
  fail(ErrorKind::InvalidOperation, "unknown kernel: " + name);
}

struct KernelOperand {
  bool sparse = false;
  FormatEncoding enc;
  MaterializedTensor mat;
  DenseTensor dense;

  static KernelOperand from_dense(DenseTensor d) {
    KernelOperand o;
    o.dense = std::move(d);
    return o;
  }
  static KernelOperand from_materialized(FormatEncoding e, MaterializedTensor m) {
    KernelOperand o;
    o.sparse = true;
    o.enc = std::move(e);
    o.mat = std::move(m);
    return o;
  }
  const TensorShape& shape() const { return sparse ? mat.logical_shape : dense.shape; }
};

struct KernelOptions {
  bool optimize = true;
  bool bounds_guards = true;
  int threads = 1;  // accepted for source compatibility; the GPU ignores it
};

// run_kernel (kernel.hpp:236) for one sparse operand followed by one dense
// operand: y = A x (spmv) or C = A B (spmm), fp32 on the device, returned as
// an f64 DenseTensor like the reference.
inline DenseTensor run_kernel(const KernelSpec& spec, const std::vector<KernelOperand>& inputs,
                              const KernelOptions& opt = {}) {
  (void)opt;
  if (inputs.size() != 2) fail(ErrorKind::InvalidOperation, "operand count does not match the kernel");
  const KernelOperand& a = inputs[0];
  const KernelOperand& d = inputs[1];
  auto& ctx = b200::default_context();
  if (a.sparse && d.sparse) {  // two sparse operands (kernel.hpp:424-567): dense C
    if (spec.name != "spgemm" && spec.name != "spmm")
      fail(ErrorKind::InvalidOperation, "two sparse operands run the spgemm kernel");
    if (!a.mat.dev || !d.mat.dev) fail(ErrorKind::InvalidOperation, "materialized tensor has no device arrays");
    const std::int64_t m = a.mat.logical_shape.extents[0], n2 = d.mat.logical_shape.extents[1];
    if (a.mat.logical_shape.extents[1] != d.mat.logical_shape.extents[0])
      fail(ErrorKind::InvalidOperation, "operand shapes disagree on a shared iterator");
    std::vector<float> c(static_cast<size_t>(m * n2));
    b200::check(sfg_spgemm(ctx.get(), a.mat.dev->h, d.mat.dev->h, c.data(), n2, SFG_COMPUTE_HOST));
    DenseTensor out(TensorShape{{m, n2}});
    std::copy(c.begin(), c.end(), out.data.begin());
    return out;
  }
  if (!a.sparse || d.sparse)
    fail(ErrorKind::InvalidOperation, "the B200 path runs one sparse operand times one dense operand");
  if (!a.mat.dev) fail(ErrorKind::InvalidOperation, "materialized tensor has no device arrays");
  const std::int64_t m = a.mat.logical_shape.extents[0], n = a.mat.logical_shape.extents[1];
  if (spec.name == "spmv") {
    if (d.dense.shape.rank() != 1 || d.dense.shape.extents[0] != n)
      fail(ErrorKind::InvalidOperation, "operand shapes disagree on a shared iterator");
    std::vector<float> x(d.dense.data.begin(), d.dense.data.end()), y(static_cast<size_t>(m));
    b200::check(sfg_spmv(ctx.get(), a.mat.dev->h, x.data(), y.data(), SFG_COMPUTE_HOST));
    DenseTensor out(TensorShape{{m}});
    std::copy(y.begin(), y.end(), out.data.begin());
    return out;
  }
  if (spec.name == "spmm") {
    if (d.dense.shape.rank() != 2 || d.dense.shape.extents[0] != n)
      fail(ErrorKind::InvalidOperation, "operand shapes disagree on a shared iterator");
    const std::int64_t nd = d.dense.shape.extents[1];
    std::vector<float> b(d.dense.data.begin(), d.dense.data.end()), c(static_cast<size_t>(m * nd));
    b200::check(sfg_spmm(ctx.get(), a.mat.dev->h, b.data(), SFG_F32, nd, nd, c.data(), nd, SFG_COMPUTE_HOST));
    DenseTensor out(TensorShape{{m, nd}});
    std::copy(c.begin(), c.end(), out.data.begin());
    return out;
  }
  fail(ErrorKind::InvalidOperation, "the B200 path runs spmv, spmm and spgemm");
}

// ------------------------------------------------ row-partitioned multi-GPU
// No reference equivalent (its only parallelism is run_kernel's host threads,
// kernel.hpp:365-384): one process per GPU, rank r holding the row block
// [bounds[r], bounds[r+1]) of A. Communicator: rank 0 calls
// comm_unique_id() and shares the bytes; every rank constructs a Comm.
namespace b200 {

inline std::array<std::uint8_t, SFG_COMM_ID_BYTES> comm_unique_id() {
  std::array<std::uint8_t, SFG_COMM_ID_BYTES> id{};
  check(sfg_comm_unique_id(id.data()));
  return id;
}

class Comm {
 public:
  Comm(int nranks, int rank, const std::array<std::uint8_t, SFG_COMM_ID_BYTES>& id) : nranks_(nranks), rank_(rank) {
    check(sfg_comm_create(default_context().get(), nranks, rank, id.data(), &h_));
  }
  ~Comm() {
    if (h_) sfg_comm_destroy(h_);
  }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  sfg_comm* get() const { return h_; }
  int nranks() const { return nranks_; }
  int rank() const { return rank_; }

 private:
  sfg_comm* h_ = nullptr;
  int nranks_, rank_;
};

}  // namespace b200

// run_kernel over a row-partitioned operand: `inputs[0]` is this rank's row
// block (chunk_rows >= the largest block), `inputs[1]` the replicated dense
// operand. Returns the whole product on every rank: P chunks of chunk_rows
// rows, chunk r holding block r (rows past a block are padding).
inline DenseTensor run_kernel_rowpart(const KernelSpec& spec, const std::vector<KernelOperand>& inputs,
                                      b200::Comm& comm, std::int64_t chunk_rows) {
  if (inputs.size() != 2 || !inputs[0].sparse || inputs[1].sparse || !inputs[0].mat.dev)
    fail(ErrorKind::InvalidOperation, "row-partitioned run_kernel takes a sparse block and a dense operand");
  const KernelOperand& a = inputs[0];
  const KernelOperand& d = inputs[1];
  auto& ctx = b200::default_context();
  const std::int64_t n = a.mat.logical_shape.extents[1];
  if (d.dense.shape.extents[0] != n) fail(ErrorKind::InvalidOperation, "operand shapes disagree on a shared iterator");
  const std::int64_t nd = spec.name == "spmv" ? 1 : d.dense.shape.extents[1];
  if (spec.name != "spmv" && (spec.name != "spmm" || d.dense.shape.rank() != 2))
    fail(ErrorKind::InvalidOperation, "row-partitioned run_kernel runs spmv or spmm");
  const std::int64_t total = comm.nranks() * chunk_rows * nd;
  std::vector<float> host(d.dense.data.begin(), d.dense.data.end());
  void *db = nullptr, *dc = nullptr;
  b200::check(sfgx_device_alloc(ctx.get(), n * nd * 4, &db));
  b200::check(sfgx_device_alloc(ctx.get(), total * 4, &dc));
  std::vector<float> out_f(static_cast<size_t>(total));
  int st = sfgx_copy(ctx.get(), db, host.data(), n * nd * 4, 0);
  if (st == SFG_OK)
    st = spec.name == "spmv"
             ? sfg_rowpart_spmv(ctx.get(), comm.get(), a.mat.dev->h, static_cast<const float*>(db),
                                static_cast<float*>(dc), chunk_rows, SFG_ROWPART_GATHER)
             : sfg_rowpart_spmm(ctx.get(), comm.get(), a.mat.dev->h, db, SFG_F32, nd, nd, static_cast<float*>(dc),
                                chunk_rows, SFG_ROWPART_GATHER);
  if (st == SFG_OK) st = sfgx_copy(ctx.get(), out_f.data(), dc, total * 4, 1);
  sfgx_device_free(ctx.get(), db);
  sfgx_device_free(ctx.get(), dc);
  b200::check(st);
  DenseTensor out(nd == 1 && spec.name == "spmv" ? TensorShape{{comm.nranks() * chunk_rows}}
                                                 : TensorShape{{comm.nranks() * chunk_rows, nd}});
  std::copy(out_f.begin(), out_f.end(), out.data.begin());
  return out;
}

}  // namespace sparseforge
