// coo_exp.cu — experiment: what bounds COO SpMV on the config-2 COO part?
// Variants of the same entry stream + x gather, timed on the real data
// (driven by scripts/coo_exp.py through ctypes).
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ int ldsi(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float ldsf(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ldsi4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ldsf4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// V0/V1: lane-strided, R entries per lane per iteration; kRow: also stream row
template <int R, bool kRow>
__global__ void k_strided(const int* __restrict__ row, const int* __restrict__ col, const float* __restrict__ val,
                          const float* __restrict__ x, float* out, int64_t nnz) {
  const int lane = threadIdx.x & 31;
  const int64_t span = 32 * R;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  float acc = 0.f;
  int racc = 0;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * span < nnz; w += warps) {
    int c[R], r[R];
    float v[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      int64_t e = w * span + 32 * i + lane;
      bool ok = e < nnz;
      c[i] = ok ? ldsi(col + e) : 0;
      v[i] = ok ? ldsf(val + e) : 0.f;
      if (kRow) r[i] = ok ? ldsi(row + e) : 0;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      acc += v[i] * __ldg(x + c[i]);
      if (kRow) racc ^= r[i];
    }
  }
  if (acc == 1.2345f || racc == 0x7654321) out[0] = acc + racc;
}

// V2: blocked int4 per lane (4 consecutive entries), R4 vectors per lane
template <int R4, bool kRow>
__global__ void k_vec(const int* __restrict__ row, const int* __restrict__ col, const float* __restrict__ val,
                      const float* __restrict__ x, float* out, int64_t nnz) {
  const int lane = threadIdx.x & 31;
  const int64_t span = 128 * R4;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  float acc = 0.f;
  int racc = 0;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; (w + 1) * span <= nnz; w += warps) {
    int4 c[R4], r[R4];
    float4 v[R4];
#pragma unroll
    for (int i = 0; i < R4; ++i) {
      int64_t e = w * span + 128 * i + 4 * lane;
      c[i] = ldsi4(reinterpret_cast<const int4*>(col + e));
      v[i] = ldsf4(reinterpret_cast<const float4*>(val + e));
      if (kRow) r[i] = ldsi4(reinterpret_cast<const int4*>(row + e));
    }
#pragma unroll
    for (int i = 0; i < R4; ++i) {
      acc += v[i].x * __ldg(x + c[i].x) + v[i].y * __ldg(x + c[i].y) + v[i].z * __ldg(x + c[i].z) +
             v[i].w * __ldg(x + c[i].w);
      if (kRow) racc ^= r[i].x ^ r[i].y ^ r[i].z ^ r[i].w;
    }
  }
  if (acc == 1.2345f || racc == 0x7654321) out[0] = acc + racc;
}

// V3: gathers only (col stream + x gather, no val)
template <int R>
__global__ void k_gather_only(const int* __restrict__ col, const float* __restrict__ x, float* out, int64_t nnz) {
  const int lane = threadIdx.x & 31;
  const int64_t span = 32 * R;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  float acc = 0.f;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * span < nnz; w += warps) {
    int c[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      int64_t e = w * span + 32 * i + lane;
      c[i] = e < nnz ? ldsi(col + e) : 0;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) acc += __ldg(x + c[i]);
  }
  if (acc == 1.2345f) out[0] = acc;
}

extern "C" float coo_exp_run(int variant, int blocks_per_sm, const int* row, const int* col, const float* val,
                             const float* x, float* out, int64_t nnz, int reps) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * blocks_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int rep = 0; rep < reps + 1; ++rep) {
    cudaEventRecord(a);
    switch (variant) {
      case 0: k_strided<16, true><<<grid, 256>>>(row, col, val, x, out, nnz); break;
      case 1: k_strided<16, false><<<grid, 256>>>(row, col, val, x, out, nnz); break;
      case 2: k_strided<8, true><<<grid, 256>>>(row, col, val, x, out, nnz); break;
      case 3: k_vec<2, true><<<grid, 256>>>(row, col, val, x, out, nnz); break;
      case 4: k_vec<2, false><<<grid, 256>>>(row, col, val, x, out, nnz); break;
      case 5: k_gather_only<16><<<grid, 256>>>(col, x, out, nnz); break;
      case 6: k_vec<4, true><<<grid, 256>>>(row, col, val, x, out, nnz); break;
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  return best;
}
