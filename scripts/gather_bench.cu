// gather_bench.cu — microbenchmark: random 4-byte gathers from an L2-resident
// vector (the x / B-row access of SpMV), under different load flavours.
// Establishes the L1TEX gather ceiling that bounds CSR SpMV on uniform
// random columns. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ float ld(const float* p) {
  float r;
  if (MODE == 0) r = __ldg(p);
  else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  else if (MODE == 2) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(r) : "l"(p));
  else if (MODE == 3) asm volatile("ld.global.L1::evict_last.f32 %0, [%1];" : "=f"(r) : "l"(p));
  else r = *p;
  return r;
}

template <int MODE, int UNROLL>
__global__ void k_gather(const int* __restrict__ idx, const float* __restrict__ x, float* out,
                         int64_t n) {
  float acc = 0.f;
  int64_t stride = (int64_t)gridDim.x * blockDim.x * UNROLL;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x) * UNROLL + threadIdx.x; i < n; i += stride) {
    int c[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) c[u] = i + u * blockDim.x < n ? __ldg(idx + i + u * blockDim.x) : 0;
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += ld<MODE>(x + c[u]);
  }
  if (acc == 123.456f) out[0] = acc;
}

__global__ void k_init(int* idx, int64_t n, int range, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    idx[i] = (int)((z >> 33) % range);
  }
}

template <int MODE>
float run(const int* idx, const float* x, float* out, int64_t n, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_gather<MODE, 4><<<grid, 256>>>(idx, x, out, n);
  cudaEventRecord(a);
  for (int it = 0; it < 10; ++it) k_gather<MODE, 4><<<grid, 256>>>(idx, x, out, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 10;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n = 1 << 24;
  int* idx;
  float *x, *out;
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&x, (64 << 20) * 4);
  cudaMalloc(&out, 4);
  cudaMemset(x, 0, (64 << 20) * 4);
  for (int range : {1 << 10, 1 << 16, 1 << 20, 1 << 22, 1 << 24}) {
    k_init<<<1024, 256>>>(idx, n, range, 42);
    cudaDeviceSynchronize();
    int grid = sms * 8;
    float t0 = run<0>(idx, x, out, n, grid), t1 = run<1>(idx, x, out, n, grid);
    float t2 = run<2>(idx, x, out, n, grid), t3 = run<3>(idx, x, out, n, grid);
    float t4 = run<4>(idx, x, out, n, grid);
    std::printf("range %8d (%6.1f MB x): ldg %.1f us  nc.noalloc %.1f us  cg %.1f us  evict_last %.1f us  plain %.1f us"
                "  => %.2f Ggather/s best\n",
                range, range * 4.0 / 1e6, t0 * 1e3, t1 * 1e3, t2 * 1e3, t3 * 1e3, t4 * 1e3,
                n / 1e9 / (std::min(std::min(t0, t1), std::min(t2, std::min(t3, t4))) * 1e-3));
  }
  return 0;
}
