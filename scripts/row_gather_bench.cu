// row_gather_bench.cu — microbenchmark: random gathers of whole 128-byte rows
// of a dense operand far larger than L2 (the B-row access of the config-5
// CSR SpMM, nd = 32 fp32). Each 8-lane group loads one row with float4s;
// K rows in flight per group. Uniform random row ids over `rows` rows:
// almost every gather misses L2, so this is the DRAM random-row ceiling
// (rows/s and GB/s) that bounds a gather-bound SpMM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o row_gather_bench row_gather_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_init(int* idx, int64_t n, int64_t range, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    idx[i] = (int)((z >> 33) % range);
  }
}

template <int K>
__global__ void __launch_bounds__(256) k_rows(const int* __restrict__ idx, const float* __restrict__ b, int64_t n,
                                              float* out) {
  const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
  float acc = 0.f;
  const int64_t warps = (int64_t)gridDim.x * 8;
  for (int64_t base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * 4 * K; base < n;
       base += warps * 4 * K) {
    int r[K];
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const int64_t e = base + u * 4 + grp;
      r[u] = e < n ? __ldg(idx + e) : 0;
    }
    float4 v[K];
#pragma unroll
    for (int u = 0; u < K; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(b + (int64_t)r[u] * 32) + sub);
#pragma unroll
    for (int u = 0; u < K; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

template <int K>
void run(const int* idx, const float* b, int64_t n, float* out, int sms, int ctas_per_sm, const char* what) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_rows<K><<<sms * ctas_per_sm, 256>>>(idx, b, n, out);
  cudaEventRecord(e0);
  for (int i = 0; i < 3; ++i) k_rows<K><<<sms * ctas_per_sm, 256>>>(idx, b, n, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 3;
  printf("%-28s K=%2d ctas/SM=%d: %.3f ms, %.2f G rows/s, %.0f GB/s of 128-B rows\n", what, K, ctas_per_sm, ms,
         n / ms / 1e6, n * 128.0 / ms / 1e6);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t rows = 1ll << 26;  // 8.6 GB of 128-byte rows (config 5's B)
  const int64_t n = 1ll << 28;     // gathers per launch
  float* b;
  int* idx;
  float* out;
  cudaMalloc(&b, rows * 128);
  cudaMalloc(&idx, n * 4);
  cudaMalloc(&out, 64);
  cudaMemset(b, 0, rows * 128);
  for (int64_t range : {rows, (int64_t)1 << 20, (int64_t)1 << 18}) {
    k_init<<<sms * 8, 256>>>(idx, n, range, 7);
    char what[64];
    snprintf(what, sizeof what, "uniform over %lld rows", (long long)range);
    run<4>(idx, b, n, out, sms, 8, what);
    run<8>(idx, b, n, out, sms, 8, what);
    run<8>(idx, b, n, out, sms, 4, what);
    run<16>(idx, b, n, out, sms, 4, what);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(err));
  return err != cudaSuccess;
}
