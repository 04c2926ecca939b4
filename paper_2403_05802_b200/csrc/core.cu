// core.cu — context, allocation, tensor lifetime and error plumbing.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.cuh"

namespace sfg {

std::atomic<int64_t> g_launches{0};

bool debug_launches() {
  static const bool on = [] {
    const char* v = std::getenv("SFG_DEBUG");
    return v && *v && *v != '0';
  }();
  return on;
}

void trace_launch(const char* name, cudaStream_t stream) {
  std::fprintf(stderr, "[sfg] launch %s (stream %p)\n", name, (void*)stream);
  std::fflush(stderr);
}

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

void raise(int code, const std::string& msg) { throw Failure{code, msg}; }

void raise_cuda(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "%s: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
  cudaGetLastError();  // clear sticky-free errors so the next call can proceed
  raise(e == cudaErrorMemoryAllocation ? SFG_ERR_OOM : SFG_ERR_CUDA, buf);
}

static bool trace_alloc() {
  static const bool on = [] {
    const char* v = std::getenv("SFG_TRACE_ALLOC");
    return v && *v && *v != '0';
  }();
  return on;
}

// Size classes: powers of two up to 1 MB, then multiples of 2 MB. A cached
// block serves a request of at least 7/8 of its size, so repeated
// conversions of one matrix reuse their blocks exactly.
static size_t size_class(size_t bytes) {
  if (bytes <= (1u << 20)) {
    size_t c = 512;
    while (c < bytes) c <<= 1;
    return c;
  }
  constexpr size_t kGran = 2u << 20;
  return (bytes + kGran - 1) / kGran * kGran;
}

static void* pool_alloc(sfg_context* ctx, size_t bytes) {
  void* p = nullptr;
  auto t0 = std::chrono::steady_clock::now();
  cudaError_t e = cudaMallocAsync(&p, bytes, ctx->stream);
  if (e != cudaSuccess) {
    // out of memory: give the cached blocks back and try once more
    cudaGetLastError();
    release_cached(ctx);
    cudaStreamSynchronize(ctx->stream);
    e = cudaMallocAsync(&p, bytes, ctx->stream);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    raise(SFG_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed: " +
                           cudaGetErrorString(e));
  }
  if (trace_alloc()) {
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[sfg] pool alloc %zu bytes: %.2f ms\n", bytes, ms);
  }
  return p;
}

void* dalloc(sfg_context* ctx, size_t bytes) {
  size_t cls = size_class(bytes ? bytes : 1);
  auto it = ctx->free_blocks.lower_bound(cls);
  if (it != ctx->free_blocks.end() && it->first - it->first / 8 <= cls) {
    void* p = it->second;
    ctx->cached_bytes -= it->first;
    ctx->free_blocks.erase(it);
    return p;
  }
  void* p = pool_alloc(ctx, cls);
  ctx->block_size[p] = cls;
  return p;
}

void dfree(sfg_context* ctx, void* p) {
  if (!p) return;
  auto it = ctx->block_size.find(p);
  if (it == ctx->block_size.end()) {
    cudaFreeAsync(p, ctx->stream);
    return;
  }
  ctx->free_blocks.emplace(it->second, p);
  ctx->cached_bytes += it->second;
}

void release_cached(sfg_context* ctx) {
  for (auto& kv : ctx->free_blocks) {
    ctx->block_size.erase(kv.second);
    cudaFreeAsync(kv.second, ctx->stream);
  }
  ctx->free_blocks.clear();
  ctx->cached_bytes = 0;
}

void* scratch(sfg_context* ctx, size_t bytes) {
  if (bytes > ctx->scratch_bytes) {
    if (ctx->scratch) dfree(ctx, ctx->scratch);
    size_t want = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 4;
    ctx->scratch = dalloc(ctx, want);
    ctx->scratch_bytes = want;
  }
  return ctx->scratch;
}

unsigned long long* lookback_status(sfg_context* ctx, size_t words) {
  if (words > ctx->status_words) {
    if (ctx->status) dfree(ctx, ctx->status);
    size_t want = words < 4096 ? 4096 : words + words / 4;
    ctx->status = dalloc(ctx, want * 8);
    SFG_CUDA(cudaMemsetAsync(ctx->status, 0, want * 8, ctx->stream));
    ctx->status_words = want;
  }
  return static_cast<unsigned long long*>(ctx->status);
}

void read_back(sfg_context* ctx, const void* dev, size_t bytes, void* host) {
  if (bytes > 4096) raise(SFG_ERR_INVALID_OPERATION, "read_back too large");
  SFG_CUDA(cudaMemcpyAsync(ctx->pinned, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  SFG_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(host, ctx->pinned, bytes);
}

// second KB of the pinned scratch, so a plain read_back in between is safe
void read_back_start(sfg_context* ctx, const void* dev, size_t bytes) {
  if (bytes > 1024) raise(SFG_ERR_INVALID_OPERATION, "read_back too large");
  if (!ctx->sizes_ev) SFG_CUDA(cudaEventCreateWithFlags(&ctx->sizes_ev, cudaEventDisableTiming));
  SFG_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->pinned) + 2048, dev, bytes, cudaMemcpyDeviceToHost,
                           ctx->stream));
  SFG_CUDA(cudaEventRecord(ctx->sizes_ev, ctx->stream));
}

void read_back_wait(sfg_context* ctx, size_t bytes, void* host) {
  SFG_CUDA(cudaEventSynchronize(ctx->sizes_ev));
  std::memcpy(host, reinterpret_cast<char*>(ctx->pinned) + 2048, bytes);
}

constexpr int kSizeSlots = 1024;

int size_slot_start(sfg_context* ctx, const int32_t* dev) {
  if (!ctx->size_slots) {
    SFG_CUDA(cudaMallocHost(&ctx->size_slots, kSizeSlots * sizeof(int32_t)));
    ctx->size_events.assign(kSizeSlots, nullptr);
    for (int i = kSizeSlots - 1; i >= 0; --i) ctx->free_size_slots.push_back(i);
  }
  if (ctx->free_size_slots.empty()) return -1;
  const int slot = ctx->free_size_slots.back();
  if (!ctx->size_events[slot])
    SFG_CUDA(cudaEventCreateWithFlags(&ctx->size_events[slot], cudaEventDisableTiming));
  SFG_CUDA(cudaMemcpyAsync(ctx->size_slots + slot, dev, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  SFG_CUDA(cudaEventRecord(ctx->size_events[slot], ctx->stream));
  ctx->free_size_slots.pop_back();
  return slot;
}

int32_t size_slot_finish(sfg_context* ctx, int slot) {
  const cudaError_t e = cudaEventSynchronize(ctx->size_events[slot]);
  ctx->free_size_slots.push_back(slot);  // returned even when the wait failed
  if (e != cudaSuccess) raise_cuda(e, "cudaEventSynchronize(size slot)", __FILE__, __LINE__);
  return ctx->size_slots[slot];
}

int64_t tensor_nnr(const sfg_tensor* t) {
  if (t->nnr_slot >= 0) {
    auto* mt = const_cast<sfg_tensor*>(t);
    const int slot = mt->nnr_slot;
    mt->nnr_slot = -1;
    mt->nnr = size_slot_finish(mt->ctx, slot);
  }
  return t->nnr;
}

sfg_tensor* new_tensor(sfg_context* ctx, int kind, int64_t m, int64_t n) {
  auto* t = new sfg_tensor;
  t->ctx = ctx;
  t->kind = kind;
  t->m = m;
  t->n = n;
  return t;
}

void free_tensor_arrays(sfg_tensor* t) {
  sfg_context* ctx = t->ctx;
  // a pending read-back must land before its slot is reused; on the free
  // path a failed wait (a sticky CUDA error) must not leak the arrays or
  // the slot, so it is waited for without raising
  if (t->nnr_slot >= 0) {
    if (cudaEventSynchronize(ctx->size_events[t->nnr_slot]) != cudaSuccess) cudaGetLastError();
    ctx->free_size_slots.push_back(t->nnr_slot);
    t->nnr_slot = -1;
  }
  dfree(ctx, t->row);
  dfree(ctx, t->ptr);
  dfree(ctx, t->idx);
  dfree(ctx, t->slots);
  dfree(ctx, t->ptr1);
  t->ptr1 = nullptr;
  dfree(ctx, t->val);
  dfree(ctx, t->tc_plan);
  dfree(ctx, t->tc_base);
  dfree(ctx, t->tc_desc);
  t->tc_plan = nullptr;
  t->tc_base = nullptr;
  t->tc_desc = nullptr;
  t->row = t->ptr = t->idx = t->slots = nullptr;
  t->val = nullptr;
}

}  // namespace sfg
