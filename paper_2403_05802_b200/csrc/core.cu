// core.cu — context, allocation, tensor lifetime and error plumbing.
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

void* dalloc(sfg_context* ctx, size_t bytes) {
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 1, ctx->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    raise(SFG_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed: " +
                           cudaGetErrorString(e));
  }
  return p;
}

void dfree(sfg_context* ctx, void* p) {
  if (p) cudaFreeAsync(p, ctx->stream);
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
  dfree(ctx, t->row);
  dfree(ctx, t->ptr);
  dfree(ctx, t->idx);
  dfree(ctx, t->slots);
  dfree(ctx, t->val);
  dfree(ctx, t->tc_plan);
  t->tc_plan = nullptr;
  t->row = t->ptr = t->idx = t->slots = nullptr;
  t->val = nullptr;
}

}  // namespace sfg
