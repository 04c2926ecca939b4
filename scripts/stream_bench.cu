// stream_bench.cu — microbenchmark: how fast can a kernel stream-read a
// 261 MB int32 array (the R-MAT s22 row array) on this part, with the load
// shapes the conversion kernels use. Sets the realistic ceiling for
// k_row_ptr-like passes. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ int4 ldnc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// grid-stride, U int4 per thread per iteration, all loads before use
template <int U>
__global__ void k_read(const int4* __restrict__ a, int64_t n4, int* out) {
  int acc = 0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n4; i += stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * blockDim.x < n4 ? ldnc(a + i + u * blockDim.x) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

// copy (read + write), U int4 per thread
template <int U>
__global__ void k_copy(const int4* __restrict__ a, int4* __restrict__ b, int64_t n4) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x * U;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n4; i += stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * blockDim.x < n4) v[u] = ldnc(a + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * blockDim.x < n4) b[i + u * blockDim.x] = v[u];
  }
}

// write-only
__global__ void k_fill(int4* __restrict__ b, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = make_int4(1, 2, 3, 4);
}

int main() {
  const int64_t n = 65247337 + 3;  // R-MAT s22 nnz, rounded to int4
  const int64_t n4 = n / 4;
  int4 *a, *b;
  int* out;
  char* flush;
  cudaMalloc(&a, n4 * 16);
  cudaMalloc(&b, n4 * 16);
  cudaMalloc(&out, 4);
  cudaMalloc(&flush, 256 << 20);
  cudaMemset(a, 1, n4 * 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](const char* name, double bytes, auto launch) {
    float best = 1e9;
    for (int rep = 0; rep < 6; ++rep) {
      cudaMemsetAsync(flush, rep, 256 << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("%-34s %8.1f us  %7.0f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
  };
  for (int per : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, sizeof nm, "read U=1 grid=%dxSM", per);
    time(nm, n4 * 16.0, [&] { k_read<1><<<sms * per, 256>>>(a, n4, out); });
    snprintf(nm, sizeof nm, "read U=4 grid=%dxSM", per);
    time(nm, n4 * 16.0, [&] { k_read<4><<<sms * per, 256>>>(a, n4, out); });
  }
  time("read U=4 grid=full", n4 * 16.0, [&] { k_read<4><<<(int)((n4 + 1023) / 1024), 256>>>(a, n4, out); });
  time("copy U=4 grid=8xSM", n4 * 32.0, [&] { k_copy<4><<<sms * 8, 256>>>(a, b, n4); });
  time("copy U=2 grid=full", n4 * 32.0, [&] { k_copy<2><<<(int)((n4 + 511) / 512), 256>>>(a, b, n4); });
  time("fill grid=8xSM", n4 * 16.0, [&] { k_fill<<<sms * 8, 256>>>(b, n4); });
  time("cudaMemcpy d2d", n4 * 32.0, [&] { cudaMemcpyAsync(b, a, n4 * 16, cudaMemcpyDeviceToDevice); });
  return 0;
}
