// mma_bench.cu — microbenchmark: cycles per tcgen05.mma.kind::f16
// (M = 128, K = 16, bf16 from shared memory, fp32 accumulate in TMEM) as a
// function of N, issued back-to-back by one thread (or by several warps into
// disjoint accumulators). Decides how small the per-block MMAs of the BCSR
// SpMM may be. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

template <int N, int WARPS>
__global__ void __launch_bounds__(32 * WARPS, 1) k_mma(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[WARPS];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int w = 0; w < WARPS; ++w)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[w])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  // A: 128 x 16 MN-major SW128 (4 KB); B: N x 16 K-major SW32
  const uint64_t adesc = sdesc(su32(sm), 2048, 1024, 2);
  const uint64_t bdesc = sdesc(su32(sm + 4096), 16, 256, 6);
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(N >> 3) << 17) |
                         ((uint32_t)(128 >> 4) << 24);
  // each warp owns its accumulator columns
  const uint32_t dcol = tmem + (uint32_t)(warp * (512 / WARPS));
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile(
        "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dcol),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(i > 0 ? 1 : 0)
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(&bar[warp]))
      : "memory");
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
          su32(&bar[warp]))
      : "memory");
  long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) out[warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Per-stage overhead: each "stage" = [proxy fence] + MPS MMAs + commit to a
// barrier (as the SpMM's MMA warp does), back-to-back, one warp.
template <int MPS, bool kProxyFence, bool kCommit>
__global__ void __launch_bounds__(32, 1) k_stage(int stages, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint64_t adesc = sdesc(su32(sm), 2048, 1024, 2);
  const uint64_t bdesc = sdesc(su32(sm + 4096), 16, 256, 6);
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(16 >> 3) << 17) |
                         ((uint32_t)(128 >> 4) << 24);
  long long t0 = clock64();
  for (int s = 0; s < stages; ++s) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (kProxyFence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int k = 0; k < MPS; ++k)
      asm volatile(
          "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 16 * ((s * MPS + k) & 31)),
          "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1)
          : "memory");
    if (kCommit)
      asm volatile(
          "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(&bar))
          : "memory");
  }
  long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int MPS, bool kProxyFence, bool kCommit>
void run_stage(long long* d) {
  const int stages = 4096;
  cudaFuncSetAttribute(k_stage<MPS, kProxyFence, kCommit>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  k_stage<MPS, kProxyFence, kCommit><<<148, 32, 64 << 10>>>(stages, d);
  k_stage<MPS, kProxyFence, kCommit><<<148, 32, 64 << 10>>>(stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("stage: %d MMAs, proxy fence %d, commit %d: %7.1f cycles per stage (issue side)  %s\n", MPS, (int)kProxyFence,
         (int)kCommit, (double)h / stages, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int N, int WARPS>
void run(long long* d) {
  const int iters = 4096;
  cudaFuncSetAttribute(k_mma<N, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  k_mma<N, WARPS><<<148, 32 * WARPS, 64 << 10>>>(iters, d);
  k_mma<N, WARPS><<<148, 32 * WARPS, 64 << 10>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[8] = {0};
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int w = 0; w < WARPS; ++w) mx = h[w] > mx ? h[w] : mx;
  double cyc = (double)mx / (iters * WARPS);
  printf("N=%3d warps=%d: %7.1f cycles per MMA (SM-wide), %6.1f TFLOP/s/chip at 1.965 GHz  %s\n", N, WARPS, cyc,
         2.0 * 128 * N * 16 / cyc * 1.965e9 * 148 / 1e12, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<16, 1>(d);
  run<32, 1>(d);
  run<64, 1>(d);
  run<128, 1>(d);
  run<256, 1>(d);
  run<16, 2>(d);
  run<16, 4>(d);
  run<64, 2>(d);
  run_stage<3, false, false>(d);
  run_stage<3, false, true>(d);
  run_stage<3, true, true>(d);
  run_stage<1, false, true>(d);
  run_stage<1, true, true>(d);
  return 0;
}
