// mma_tmem_bench.cu — microbenchmark for the config-4 "next" idea
// (DESIGN.md §7): tcgen05.mma.kind::f16 M=128/N=16/K=16 with the A operand
// (the dense 128 x 16 bf16 tile) read from TMEM instead of shared memory,
// and the cost of staging that tile with tcgen05.cp (smem -> TMEM,
// .128x256b). Timing only (operand contents are irrelevant).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 mma_tmem_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

// mode 0: A from smem (MN-major SW128), 1: A from TMEM, 2: A from TMEM with
// one tcgen05.cp of a fresh 128x256b tile every `per_cp` MMAs, 3: cp only
template <int MODE>
__global__ void __launch_bounds__(32, 1) k_bench(int iters, int per_cp, long long* out) {
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
  const uint64_t adesc = sdesc(su32(sm), 2048, 1024, 2);             // SW128 MN-major (mode 0)
  const uint64_t bdesc = sdesc(su32(sm + 8192), 16, 256, 6);         // SW32 K-major value block
  const uint64_t cdesc = sdesc(su32(sm + 16384), 16, 256, 6);        // SW32 K-major 128 x 16 tile (cp source)
  const uint32_t a_mn = 1u << 15;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (MODE == 0 ? a_mn : 0u) | ((uint32_t)(16 >> 3) << 17) |
                         ((uint32_t)(128 >> 4) << 24);
  const uint32_t a_tmem = tmem + 448;  // 8 columns per tile, 8 slots
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t d = tmem + 16 * (i % 28);
    if (MODE >= 2 && i % per_cp == 0)
      asm volatile(
          "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n}\n" ::"r"(a_tmem + 8 * ((i / per_cp) & 7)),
          "l"(cdesc)
          : "memory");
    if (MODE == 3) continue;
    if (MODE == 0)
      asm volatile(
          "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
          "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1)
          : "memory");
    else
      asm volatile(
          "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
          "r"(a_tmem + 8 * ((i / (per_cp > 0 ? per_cp : 1)) & 7)), "l"(bdesc), "r"(idesc), "r"(1)
          : "memory");
  }
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(&bar))
      : "memory");
  asm volatile(
      "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar))
      : "memory");
  long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncwarp();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int MODE>
void run(long long* d, int per_cp, const char* what) {
  const int iters = 8192;
  cudaFuncSetAttribute(k_bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 << 10);
  k_bench<MODE><<<148, 32, 64 << 10>>>(iters, per_cp, d);
  k_bench<MODE><<<148, 32, 64 << 10>>>(iters, per_cp, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-48s per_cp=%d: %7.2f cycles per iteration  %s\n", what, per_cp, (double)h / iters,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<0>(d, 1, "MMA M128 N16 K16, A from smem");
  run<1>(d, 1, "MMA M128 N16 K16, A from TMEM");
  run<3>(d, 1, "tcgen05.cp 128x256b only");
  for (int k : {1, 2, 3, 4, 8}) run<2>(d, k, "A from TMEM + one tcgen05.cp every per_cp MMAs");
  return 0;
}
