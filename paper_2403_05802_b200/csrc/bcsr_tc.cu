// bcsr_tc.cu — BCSR(16,16) SpMM on the 5th-generation tensor cores.
//
// Reference: run_kernel(spmm_kernel(), {A_bcsr, B}) (kernel.hpp:236-384):
// C[d0][d2] += A[d0][d1] * B[d1][d2] over every stored slot of every dense
// block (storage.hpp:238-280 walk), slots past M/N guarded out.
//
// Formulation: per stored block k of block row br (block column bc),
//   C^T[nd x 16] += B_k^T[nd x 16] . A_k^T[16 x 16]
// i.e. one tcgen05.mma.kind::f16 with M = nd = 128 (the dense width),
// N = 16 (rows of the block row), K = 16 (columns of the block), bf16
// operands, fp32 accumulator in TMEM (128 lanes x 16 columns per block row).
//   A operand = the B tile rows [bc*16, bc*16+16) x all 128 columns,
//               MN-major, loaded by TMA with 128-byte swizzle (two 64-column
//               boxes);
//   B operand = the 16x16 value block, K-major, TMA with 32-byte swizzle.
// Warp roles (192 threads): warps 0-3 epilogue (TMEM -> registers -> C, one
// warp per 32-lane TMEM quarter), warp 4 TMA producer, warp 5 MMA issuer.
// An 8-stage smem ring (full/empty mbarriers) feeds the MMA; two TMEM
// accumulators let the epilogue of one block row overlap the MMAs of the
// next. Persistent CTAs stride over block rows.
//
// Applies to: BCSR with r = c = 16, bf16 values, bf16 B with nd = 128.
// Everything else uses the CUDA-core kernel in spmm.cu.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "async.cuh"
#include "devutil.cuh"
#include "internal.cuh"

namespace sfg {

namespace {

constexpr int kStages = 8;
constexpr int kND = 128;              // dense width handled by one MMA (M)
constexpr int kBlk = 16;              // block rows (N) and columns (K)
constexpr int kTileBytes = kBlk * kND * 2;          // 4096: B tile (two 2 KB boxes)
constexpr int kABytes = kBlk * kBlk * 2;            // 512: value block
constexpr int kStageBytes = 5120;                   // 1024-aligned stage stride
constexpr int kThreads = 192;
constexpr int kAccCols = 32;                        // 2 accumulators x 16 columns

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor (sm_100): start >> 4 [0,14), LBO >> 4
// [16,30), SBO >> 4 [32,46), version 1 [46,48), layout type [61,64).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

// Instruction descriptor: F32 accumulate, BF16 x BF16, A MN-major, B K-major,
// N = 16, M = 128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(kBlk >> 3) << 17) |
                            ((uint32_t)(kND >> 4) << 24);

struct Shared {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t acc_full[2];
  uint64_t acc_empty[2];
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(kThreads, 1)
    k_bcsr_tc(const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_a,
              const int32_t* __restrict__ ptr, const int32_t* __restrict__ bcol, int32_t nbr, int32_t m,
              float* __restrict__ c, int64_t ldc, int accumulate) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Shared* sh = reinterpret_cast<Shared*>(stages + kStages * kStageBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&sh->full[s], 1);
      mbar_init(&sh->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&sh->acc_full[a], 1);
      mbar_init(&sh->acc_empty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh->tmem_base)),
                 "r"(kAccCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh->tmem_base;

  if (warp == 4) {
    // ---------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int32_t br = blockIdx.x; br < nbr; br += gridDim.x) {
        int32_t s = __ldg(ptr + br), e = __ldg(ptr + br + 1);
        for (int32_t k = s; k < e; ++k) {
          mbar_wait(&sh->empty[stage], phase ^ 1);
          uint8_t* st = stages + stage * kStageBytes;
          mbar_expect_tx(&sh->full[stage], kTileBytes + kABytes);
          int brow = __ldg(bcol + k) * kBlk;
          tma_2d(st, &tmap_b, &sh->full[stage], 0, brow);
          tma_2d(st + 2048, &tmap_b, &sh->full[stage], 64, brow);
          tma_2d(st + kTileBytes, &tmap_a, &sh->full[stage], 0, k * kBlk);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 5) {
    // ---------------------------------------------------- MMA issuer
    int stage = 0, it = 0;
    uint32_t phase = 0;
    for (int32_t br = blockIdx.x; br < nbr; br += gridDim.x) {
      int32_t s = __ldg(ptr + br), e = __ldg(ptr + br + 1);
      if (s == e) continue;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&sh->acc_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      for (int32_t k = s; k < e; ++k) {
        mbar_wait(&sh->full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          uint32_t base = smem_u32(stages + stage * kStageBytes);
          uint64_t adesc = smem_desc(base, 2048, 1024, 2);          // SW128, MN-major
          uint64_t bdesc = smem_desc(base + kTileBytes, 16, 256, 6);  // SW32, K-major
          tc_mma(tmem + acc * kBlk, adesc, bdesc, kIdesc, k > s ? 1u : 0u);
          tc_commit(&sh->empty[stage]);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) tc_commit(&sh->acc_full[acc]);
      __syncwarp();
      ++it;
    }
  } else {
    // ---------------------------------------------------- epilogue
    int it = 0;
    const int col = warp * 32 + lane;  // dense column = TMEM lane
    for (int32_t br = blockIdx.x; br < nbr; br += gridDim.x) {
      int32_t s = __ldg(ptr + br), e = __ldg(ptr + br + 1);
      const int64_t r0 = (int64_t)br * kBlk;
      if (s == e) {
        if (!accumulate)
          for (int i = 0; i < kBlk; ++i)
            if (r0 + i < m) c[(r0 + i) * ldc + col] = 0.f;
        continue;
      }
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      mbar_wait(&sh->acc_full[acc], acc_phase);
      tc_fence_after();
      float v[16];
      tc_ld16(tmem + ((uint32_t)(warp * 32) << 16) + acc * kBlk, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh->acc_empty[acc]);
#pragma unroll
      for (int i = 0; i < kBlk; ++i) {
        if (r0 + i < m) {
          float* p = c + (r0 + i) * ldc + col;
          *p = accumulate ? *p + v[i] : v[i];
        }
      }
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kAccCols));
  }
}

// ------------------------------------------------------------------------
// Grouped variant: a CTA owns kGroup consecutive block rows, all resident in
// TMEM at once (kGroup x 16 fp32 columns = 512). The producer warp merges
// the group's block-column lists (lane j holds block row j's cursor; warp
// min + ballot per step), so each B tile is loaded ONCE per group and
// multiplied into every block row that holds that block column. Per stage:
// one B tile (4 KB, SW128) + up to kMaxA value blocks (512 B each, SW32,
// packed in block-row order); a block column held by more than kMaxA of the
// group's block rows spills into further stages that reload the tile. The
// stage's block-row mask travels in shared memory. The ring is deep (26
// stages, ~8 KB each): the kernel is bound by bytes in flight per SM, since
// every stage round-trips through L2/HBM. At the end of the group the
// epilogue drains all accumulators.
constexpr int kGroup = 32;
constexpr int kMaxA = 8;
constexpr int kGStages = 26;
constexpr int kGStageBytes = kTileBytes + kMaxA * kABytes;  // 8 KB

struct GShared {
  uint64_t full[kGStages];
  uint64_t empty[kGStages];
  uint64_t acc_full;
  uint64_t acc_empty;
  uint32_t mask[kGStages];
  uint32_t started;
  uint32_t tmem_base;
};

__device__ __forceinline__ void mbar_arrive_plain(uint64_t* bar) { mbar_arrive(bar); }

__global__ void __launch_bounds__(kThreads, 1)
    k_bcsr_tc_group(const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_a,
                    const int32_t* __restrict__ ptr, const int32_t* __restrict__ bcol, int32_t nbr,
                    int32_t m, float* __restrict__ c, int64_t ldc, int accumulate,
                    const uint32_t* __restrict__ plan, int32_t nbc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  GShared* sh = reinterpret_cast<GShared*>(stages + kGStages * kGStageBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t ngroups = (nbr + kGroup - 1) / kGroup;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&sh->full[s], 1);
      mbar_init(&sh->empty[s], 1);
    }
    mbar_init(&sh->acc_full, 1);
    mbar_init(&sh->acc_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh->tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh->tmem_base;

  // One pipeline step: the B tile of block column `bc` and the value blocks
  // of the block rows in `mask` (split into stages of <= kMaxA blocks).
  // Lanes whose bit is set issue their own value-block load and advance.
  auto issue = [&](uint32_t mask, uint32_t bc, int32_t& cur, int& stage, uint32_t& phase) {
    uint32_t rest = mask;
    do {
      uint32_t chunk = rest;
      if (__popc(rest) > kMaxA) {  // rare: more than kMaxA block rows share bc
        chunk = 0;
        uint32_t t = rest;
#pragma unroll
        for (int k = 0; k < kMaxA; ++k) {
          uint32_t low = t & (0u - t);
          chunk |= low;
          t ^= low;
        }
      }
      rest ^= chunk;
      if (lane == 0) {
        mbar_wait(&sh->empty[stage], phase ^ 1);
        sh->mask[stage] = chunk;
        uint8_t* st = stages + stage * kGStageBytes;
        mbar_expect_tx(&sh->full[stage], kTileBytes + __popc(chunk) * kABytes);
        tma_2d(st, &tmap_b, &sh->full[stage], 0, (int)bc * kBlk);
        tma_2d(st + 2048, &tmap_b, &sh->full[stage], 64, (int)bc * kBlk);
      }
      __syncwarp();
      if (chunk >> lane & 1u) {
        uint8_t* st = stages + stage * kGStageBytes;
        int slot = __popc(chunk & ((1u << lane) - 1u));
        tma_2d(st + kTileBytes + slot * kABytes, &tmap_a, &sh->full[stage], 0, cur * kBlk);
      }
      if (++stage == kGStages) {
        stage = 0;
        phase ^= 1;
      }
    } while (rest);
    if (mask >> lane & 1u) ++cur;
  };
  auto end_group = [&](int& stage, uint32_t& phase) {
    if (lane == 0) {
      mbar_wait(&sh->empty[stage], phase ^ 1);
      sh->mask[stage] = 0;
      mbar_arrive_plain(&sh->full[stage]);  // end-of-group marker
    }
    __syncwarp();
    if (++stage == kGStages) {
      stage = 0;
      phase ^= 1;
    }
  };

  if (warp == 4 && plan != nullptr) {
    // ------------------------------------ producer: stream the mask plan
    // plan[g * nbc + bc] = bit j set iff block row g*32+j holds block
    // column bc. Lane l reads the masks of 32 consecutive block columns
    // (one coalesced load, the next batch prefetched); the nonzero ones are
    // issued in order.
    int stage = 0;
    uint32_t phase = 0;
    for (int32_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
      const int32_t br = g * kGroup + lane;
      int32_t cur = br < nbr ? __ldg(ptr + br) : 0;
      const uint32_t* pg = plan + (int64_t)g * nbc;
      uint32_t nxt = lane < nbc ? __ldg(pg + lane) : 0u;
      for (int32_t bc0 = 0; bc0 < nbc; bc0 += 32) {
        uint32_t mine = nxt;
        nxt = bc0 + 32 + lane < nbc ? __ldg(pg + bc0 + 32 + lane) : 0u;
        uint32_t nz = __ballot_sync(kFull, mine != 0);
        while (nz) {
          int src = __ffs(nz) - 1;
          nz &= nz - 1;
          uint32_t mask = __shfl_sync(kFull, mine, src);
          issue(mask, (uint32_t)(bc0 + src), cur, stage, phase);
        }
      }
      end_group(stage, phase);
    }
  } else if (warp == 4) {
    // ------------------------------------------- producer: k-way merge
    int stage = 0;
    uint32_t phase = 0;
    for (int32_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
      const int32_t br = g * kGroup + lane;
      int32_t cur = 0, end = 0;
      if (br < nbr) {
        cur = __ldg(ptr + br);
        end = __ldg(ptr + br + 1);
      }
      // Block-column window in registers, double-buffered: wa holds the
      // next 8 block columns of this lane's block row, wb the 8 after, whose
      // loads were issued 8 advances earlier — the merge never waits on a
      // dependent global load.
      uint32_t wa[8], wb[8];
      int wi = 0;
      int32_t next = cur + 16;  // first block index not yet requested
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        wa[k] = cur + k < end ? (uint32_t)__ldg(bcol + cur + k) : 0xffffffffu;
        wb[k] = cur + 8 + k < end ? (uint32_t)__ldg(bcol + cur + 8 + k) : 0xffffffffu;
      }
      uint32_t bc = wa[0];
      while (true) {
        uint32_t mn = __reduce_min_sync(kFull, bc);
        uint32_t mask = __ballot_sync(kFull, bc == mn && mn != 0xffffffffu);
        if (!mask) {
          end_group(stage, phase);
          break;
        }
        issue(mask, mn, cur, stage, phase);
        if (mask >> lane & 1u) {
          if (++wi == 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              wa[k] = wb[k];
              wb[k] = next + k < end ? (uint32_t)__ldg(bcol + next + k) : 0xffffffffu;
            }
            next += 8;
            wi = 0;
          }
          bc = wa[0];
#pragma unroll
          for (int k = 1; k < 8; ++k)
            if (k == wi) bc = wa[k];
        }
        if (!mask) break;
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------- MMA issuer
    int stage = 0, it = 0;
    uint32_t phase = 0;
    for (int32_t g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
      mbar_wait(&sh->acc_empty, (it & 1) ^ 1);
      tc_fence_after();
      uint32_t started = 0;
      while (true) {
        mbar_wait(&sh->full[stage], phase);
        tc_fence_after();
        uint32_t mask = sh->mask[stage];
        if (lane == 0) {
          if (mask) {
            uint32_t base = smem_u32(stages + stage * kGStageBytes);
            uint64_t adesc = smem_desc(base, 2048, 1024, 2);
            uint32_t mm = mask;
            for (int slot = 0; mm; ++slot) {
              int j = __ffs(mm) - 1;
              mm &= mm - 1;
              uint64_t bdesc = smem_desc(base + kTileBytes + slot * kABytes, 16, 256, 6);
              tc_mma(tmem + j * kBlk, adesc, bdesc, kIdesc, (started >> j) & 1u);
            }
            tc_commit(&sh->empty[stage]);
          } else {
            tc_commit(&sh->acc_full);
            mbar_arrive(&sh->empty[stage]);
          }
        }
        started |= mask;
        __syncwarp();
        if (++stage == kGStages) {
          stage = 0;
          phase ^= 1;
        }
        if (!mask) break;
      }
    }
  } else {
    // ------------------------------------------- epilogue
    int it = 0;
    const int col = warp * 32 + lane;
    for (int32_t g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
      mbar_wait(&sh->acc_full, it & 1);
      tc_fence_after();
      for (int j = 0; j < kGroup; ++j) {
        const int64_t r0 = ((int64_t)g * kGroup + j) * kBlk;
        if (r0 >= m) break;
        const int32_t br = g * kGroup + j;
        float v[16];
        if (__ldg(ptr + br) < __ldg(ptr + br + 1)) {  // accumulator j was written
          tc_ld16(tmem + ((uint32_t)(warp * 32) << 16) + j * kBlk, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < kBlk; ++i) {
          if (r0 + i < m) {
            float* p = c + (r0 + i) * ldc + col;
            *p = accumulate ? *p + v[i] : v[i];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh->acc_empty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// SpMM plan: plan[g * nbc + bc] |= 1 << (br % 32) for every stored block
// (br, bc), g = br / 32. A warp per block row, one lane per block.
__global__ void __launch_bounds__(256) k_bcsr_plan(const int32_t* __restrict__ ptr,
                                                    const int32_t* __restrict__ bcol, int32_t nbr,
                                                    int32_t nbc, uint32_t* __restrict__ plan) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t br = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; br < nbr; br += warps) {
    uint32_t* pg = plan + (br / kGroup) * (int64_t)nbc;
    const uint32_t bit = 1u << (br % kGroup);
    for (int32_t k = __ldg(ptr + br) + lane; k < __ldg(ptr + br + 1); k += 32) atomicOr(pg + __ldg(bcol + k), bit);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace

bool spmm_bcsr_tc(sfg_context* ctx, const sfg_tensor* a, const void* b, int b_dtype, int64_t nd,
                  int64_t ldb, float* c, int64_t ldc, bool accumulate) {
  if (a->kind != SFG_BCSR || a->dtype != SFG_BF16 || b_dtype != SFG_BF16 || nd != kND) return false;
  if (a->br != kBlk || a->bc != kBlk || a->rb != kBlk || a->cb != kBlk) return false;
  if ((ldb * 2) % 16 != 0 || (reinterpret_cast<uintptr_t>(b) & 15) || a->nnz == 0) return false;
  if (a->nbr > INT32_MAX || a->nnz * kBlk > INT32_MAX) return false;
  auto encode = get_encode();
  if (!encode) return false;
  CUtensorMap tb, ta;
  {
    cuuint64_t dims[2] = {(cuuint64_t)nd, (cuuint64_t)a->n};
    cuuint64_t strides[1] = {(cuuint64_t)ldb * 2};
    cuuint32_t box[2] = {64, kBlk};
    cuuint32_t es[2] = {1, 1};
    if (encode(&tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(b), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      raise(SFG_ERR_CUDA, "cuTensorMapEncodeTiled(B) failed");
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)kBlk, (cuuint64_t)(a->nnz * kBlk)};
    cuuint64_t strides[1] = {(cuuint64_t)kBlk * 2};
    cuuint32_t box[2] = {kBlk, kBlk};
    cuuint32_t es[2] = {1, 1};
    if (encode(&ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a->val, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      raise(SFG_ERR_CUDA, "cuTensorMapEncodeTiled(A) failed");
  }
  const size_t smem = 1024 + kStages * kStageBytes + sizeof(Shared) + 64;
  const size_t gsmem = 1024 + kGStages * kGStageBytes + sizeof(GShared) + 64;
  static bool attr = false;
  if (!attr) {
    SFG_CUDA(cudaFuncSetAttribute(k_bcsr_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SFG_CUDA(cudaFuncSetAttribute(k_bcsr_tc_group, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem));
    attr = true;
  }
  static const bool per_row = [] {
    const char* v = std::getenv("SFG_BCSR_TC_PER_ROW");  // A/B switch: one block row per accumulator
    return v && *v == '1';
  }();
  if (per_row) {
    int grid = (int)std::min<int64_t>(a->nbr, (int64_t)ctx->sms);
    SFG_LAUNCH(k_bcsr_tc, grid, kThreads, smem, ctx->stream, tb, ta, a->ptr, a->idx, (int32_t)a->nbr,
               (int32_t)a->m, c, ldc, accumulate ? 1 : 0);
  } else {
    // The mask plan (per 32-block-row group, per block column) is built once
    // per matrix and cached on the tensor; it is used when the group masks
    // are dense enough that streaming them beats the in-kernel merge.
    const int64_t ngroups = ceil_div(a->nbr, kGroup);
    const int64_t words = ngroups * a->nbc;
    sfg_tensor* mut = const_cast<sfg_tensor*>(a);  // plan is a cache, not tensor state
    if (!mut->tc_plan && a->nnz * 4 >= words && words <= (int64_t(1) << 30)) {
      mut->tc_plan = dalloc_n<uint32_t>(ctx, words);
      SFG_CUDA(cudaMemsetAsync(mut->tc_plan, 0, words * 4, ctx->stream));
      SFG_LAUNCH(k_bcsr_plan, stream_grid(ctx, a->nbr * 32, 256, 1, 8), 256, 0, ctx->stream, a->ptr, a->idx,
                 (int32_t)a->nbr, (int32_t)a->nbc, mut->tc_plan);
    }
    int grid = (int)std::min<int64_t>(ngroups, (int64_t)ctx->sms);
    SFG_LAUNCH(k_bcsr_tc_group, grid, kThreads, gsmem, ctx->stream, tb, ta, a->ptr, a->idx, (int32_t)a->nbr,
               (int32_t)a->m, c, ldc, accumulate ? 1 : 0, mut->tc_plan, (int32_t)a->nbc);
  }
  return true;
}

}  // namespace sfg
