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

#include <cstdio>
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

__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// The mbarrier arrive that fires when all of this thread's earlier cp.async
// copies (async.cuh cp_async16) have landed (the barrier's pending count is
// raised first, so it waits for them).
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
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

// Issued by one elected lane of a converged warp: the operands are
// warp-uniform, so they go to uniform registers without a per-lane loop.
__device__ __forceinline__ void tc_mma_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_mma_elect_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.eq.u32 p, 1, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
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

// kProducers producer warps (stages dealt round-robin), kMmaWarps MMA
// warps (block rows dealt by j % kMmaWarps).
template <int kProducers, int kMmaWarps>
__global__ void __launch_bounds__(32 * (4 + kProducers + kMmaWarps), 1)
    k_bcsr_tc_group(const __grid_constant__ CUtensorMap tmap_b, const uint8_t* __restrict__ aval,
                    const int32_t* __restrict__ ptr, const int32_t* __restrict__ bcol, int32_t nbr,
                    int32_t m, float* __restrict__ c, int64_t ldc, int accumulate,
                    const uint32_t* __restrict__ plan, int32_t nbc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  GShared* sh = reinterpret_cast<GShared*>(stages + kGStages * kGStageBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t ngroups = (nbr + kGroup - 1) / kGroup;
  constexpr int kMmaWarp = 4 + kProducers;  // first MMA warp
  static_assert(kGStages % kProducers == 0, "producers must divide the ring (exact parity waits)");

  if (threadIdx.x == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&sh->full[s], 1);
      mbar_init(&sh->empty[s], kMmaWarps);  // each MMA warp commits every stage
    }
    mbar_init(&sh->acc_full, kMmaWarps);
    mbar_init(&sh->acc_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh->tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh->tmem_base;

  // Producer warps 4 .. 4+kProducers-1 all walk the same sequence of
  // pipeline stages (so they agree on every stage's index and contents);
  // stage t is issued by producer warp t % kProducers, so the TMA issue
  // work — serialised per warp — runs kProducers-wide.
  const int pw = warp - 4;
  // One pipeline step: the B tile of block column `bc` and the value blocks
  // of the block rows in `mask` (split into stages of <= kMaxA blocks).
  // Lanes whose bit is set issue their own value-block load and advance.
  auto issue = [&](uint32_t mask, uint32_t bc, int32_t& cur, int& stage, uint32_t& phase, uint32_t& t) {
    uint32_t rest = mask;
    do {
      uint32_t chunk = rest;
      if (__popc(rest) > kMaxA) {  // rare: more than kMaxA block rows share bc
        chunk = 0;
        uint32_t tt = rest;
#pragma unroll
        for (int k = 0; k < kMaxA; ++k) {
          uint32_t low = tt & (0u - tt);
          chunk |= low;
          tt ^= low;
        }
      }
      rest ^= chunk;
      if ((int)(t % kProducers) == pw) {
        if (lane == 0) mbar_wait(&sh->empty[stage], phase ^ 1);
        __syncwarp();
        uint8_t* st = stages + stage * kGStageBytes;
        // value blocks: a 512-byte block is one 16-byte cp.async per lane,
        // placed in the 32-byte-swizzled K-major layout the MMA reads
        // (16-byte chunk c of row r lands at chunk c ^ (r >> 2 & 1))
        const int r = lane >> 1, ch = lane & 1;
        const uint32_t dst_off = r * 32 + ((ch ^ ((r >> 2) & 1)) << 4);
        uint32_t cm = chunk;
        for (int slot = 0; cm; ++slot) {
          const int j = __ffs(cm) - 1;
          cm &= cm - 1;
          const int32_t kblk = __shfl_sync(kFull, cur, j);
          cp_async16(st + kTileBytes + slot * kABytes + dst_off, aval + (int64_t)kblk * kABytes + lane * 16);
        }
        cp_async_mbar_arrive(&sh->full[stage]);
        __syncwarp();
        if (lane == 0) {
          sh->mask[stage] = chunk;
          mbar_expect_tx(&sh->full[stage], kTileBytes);
          tma_3d(st, &tmap_b, &sh->full[stage], 0, (int)bc * kBlk, 0);  // both 64-column halves
        }
      }
      ++t;
      if (++stage == kGStages) {
        stage = 0;
        phase ^= 1;
      }
    } while (rest);
    if (mask >> lane & 1u) ++cur;
  };
  auto end_group = [&](int& stage, uint32_t& phase, uint32_t& t) {
    if ((int)(t % kProducers) == pw && lane == 0) {
      mbar_wait(&sh->empty[stage], phase ^ 1);
      sh->mask[stage] = 0;
      mbar_arrive_plain(&sh->full[stage]);  // end-of-group marker
    }
    __syncwarp();
    ++t;
    if (++stage == kGStages) {
      stage = 0;
      phase ^= 1;
    }
  };

  if (warp >= 4 && warp < kMmaWarp && plan != nullptr) {
    // ------------------------------------ producer: stream the mask plan
    // plan[g * nbc + bc] = bit j set iff block row g*32+j holds block
    // column bc. Lane l reads the masks of 32 consecutive block columns
    // (one coalesced load, the next batch prefetched); the nonzero ones are
    // issued in order.
    int stage = 0;
    uint32_t phase = 0, t = 0;
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
          issue(mask, (uint32_t)(bc0 + src), cur, stage, phase, t);
        }
      }
      end_group(stage, phase, t);
    }
  } else if (warp >= 4 && warp < kMmaWarp) {
    // ------------------------------------------- producer: k-way merge
    int stage = 0;
    uint32_t phase = 0, t = 0;
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
          end_group(stage, phase, t);
          break;
        }
        issue(mask, mn, cur, stage, phase, t);
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
      }
    }
  } else if (warp >= kMmaWarp) {
    // ------------------------------------------- MMA issuers
    // kMmaWarps converged warps; warp w issues the MMAs of the block rows j
    // with j % kMmaWarps == w (disjoint accumulators) and commits every
    // stage, so a stage is free once all of them have committed. The
    // issue path is warp-uniform: stage descriptors are the base
    // descriptors plus the stage offset, one elected lane issues.
    const int w = warp - kMmaWarp;
    uint32_t mine = 0;
    for (int j = w; j < kGroup; j += kMmaWarps) mine |= 1u << j;
    const uint32_t base0 = smem_u32(stages);
    const uint64_t adesc0 = smem_desc(base0, 2048, 1024, 2);             // SW128, MN-major
    const uint64_t bdesc0 = smem_desc(base0 + kTileBytes, 16, 256, 6);   // SW32, K-major
    int stage = 0, it = 0;
    uint32_t phase = 0;
    for (int32_t g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
      mbar_wait(&sh->acc_empty, (it & 1) ^ 1);
      tc_fence_after();
      uint32_t started = 0;
      while (true) {
        mbar_wait(&sh->full[stage], phase);
        tc_fence_after();
        // the value blocks were written by cp.async (generic proxy); the
        // MMA reads them through the async proxy
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t mask = sh->mask[stage];
        const uint64_t soff = (uint64_t)((stage * kGStageBytes) >> 4);
        if (mask) {
          uint32_t mm = mask & mine;
          while (mm) {
            const int j = __ffs(mm) - 1;
            mm &= mm - 1;
            const uint32_t slot = __popc(mask & ((1u << j) - 1u));
            tc_mma_elect(tmem + j * kBlk, adesc0 + soff, bdesc0 + soff + ((slot * kABytes) >> 4), kIdesc,
                         (started >> j) & 1u);
          }
          tc_commit_elect(&sh->empty[stage]);
          started |= mask & mine;
        } else {
          tc_commit_elect(&sh->acc_full);
          if (lane == 0) mbar_arrive(&sh->empty[stage]);
        }
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
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ------------------------------------------------------------------------
// Panel variant (used with the mask plan). Same group / TMEM layout as the
// grouped kernel, but a pipeline stage carries up to kPanel block columns
// (B tiles, one 3-D TMA copy each) and up to kPanelA value blocks, so the
// per-stage costs — barrier waits, commits, the plan walk — are paid once
// per ~kPanel x 3 MMAs instead of per ~3. Value blocks arrive by cp.async
// (one 16-byte copy per lane per block, written in the 32-byte-swizzled
// K-major layout). Stage metadata (tile masks) travels in shared memory.
// Two configurations: bf16 (one kind::f16 MMA per block, 4 tiles and 16
// value blocks per stage, 8 stages) and fp32 (3xTF32: per block and K half
// of 8, hi.hi + lo.hi + hi.lo kind::tf32 MMAs — six per block — with B split
// into tf32 hi / lo arrays by a pre-pass and each staged value block split in
// shared memory by its MMA warp; 2 tiles and 8 blocks per stage, each stored
// hi and lo, 4 stages).
template <bool kTF>
struct PanelCfg;
template <>
struct PanelCfg<false> {
  static constexpr int kPanel = 4, kPanelA = 16, kStages = 8;
  static constexpr int kTile = kTileBytes, kA = kABytes;
  static constexpr int kVal = kPanel * kTile;  // value blocks' offset inside a stage
  static constexpr int kStageBytes = kPanel * kTile + kPanelA * kA;     // 24 KB
  static constexpr uint32_t kId = kIdesc;
};
template <>
struct PanelCfg<true> {
  static constexpr int kPanel = 2, kPanelA = 8, kStages = 4;
  static constexpr int kTile = kBlk * kND * 4, kA = kBlk * kBlk * 4;  // 8 KB, 1 KB
  static constexpr int kLoTile = kPanel * kTile, kVal = 2 * kPanel * kTile, kLoVal = kVal + kPanelA * kA;
  static constexpr int kStageBytes = 2 * (kPanel * kTile + kPanelA * kA);  // 48 KB
  // F32 accumulate, TF32 x TF32, A MN-major, B K-major, N = 16, M = 128
  static constexpr uint32_t kId = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) |
                                     ((uint32_t)(kBlk >> 3) << 17) | ((uint32_t)(kND >> 4) << 24);
};
constexpr int kDescWords = 32;  // 0 head, 1-4 tile columns, 5-8 masks, 10-13 slot bytes, 16-31 slot blocks
static_assert(PanelCfg<false>::kPanel <= 4 && PanelCfg<false>::kPanelA <= 16, "descriptor layout: 4 tiles, 16 slots");

template <int kStagesT>
struct PShared {
  uint64_t full[kStagesT];
  uint64_t empty[kStagesT];
  uint64_t acc_full;
  uint64_t acc_empty;
  alignas(16) uint32_t mask[kStagesT][4];  // mask[s][t]: block rows of tile t; a zero tile ends the stage
  alignas(16) uint8_t slot[kStagesT][16];  // slot -> block row | tile << 5
  uint32_t tmem_base;
};

// tf32 hi part: the low 13 mantissa bits cleared (exact as tf32 whether the
// tensor core truncates or rounds); lo = x - hi is exact in fp32
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// B (n x 128, leading dimension ldb) -> hi, lo (n x 128, dense)
__global__ void k_tf32_split(const float* __restrict__ b, int64_t n, int64_t ldb, float* __restrict__ hi,
                             float* __restrict__ lo) {
  const int64_t q4 = n * (kND / 4);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < q4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (kND / 4), c4 = i % (kND / 4);
    const float4 x = ld_stream(reinterpret_cast<const float4*>(b + r * ldb) + c4);
    const float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
    reinterpret_cast<float4*>(hi)[i] = h;
    reinterpret_cast<float4*>(lo)[i] = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
  }
}

__device__ __forceinline__ void tmem_zero16(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(0u)
      : "memory");
}

// Warps: 0-3 epilogue (TMEM lane quarter each), 4 .. 4+kProducers-1
// producers, then kMmaWarps MMA issuers. Ring position t (every stage of
// every group of this CTA, plus one end marker per group) is filled by
// producer t % kProducers and consumed by MMA warp t % kMmaWarps, so both
// sides work on several stages at once. Accumulators are zeroed by the
// epilogue after each drain and every MMA accumulates, so the MMAs of one
// group may come from any MMA warp (the CTA's MMAs execute in one tensor
// pipe; each adds into its accumulator).
template <int kProducers, int kMmaWarps, bool kTF>
__global__ void __launch_bounds__(32 * (4 + kProducers + kMmaWarps), 1)
    k_bcsr_tc_panel(const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_lo,
                    const __grid_constant__ CUtensorMap tmap_v, const uint8_t* __restrict__ aval,
                    const int32_t* __restrict__ ptr, int32_t nbr, int32_t m, float* __restrict__ c, int64_t ldc,
                    int accumulate, const int32_t* __restrict__ sbase, const uint32_t* __restrict__ sdesc,
                    int dbg, unsigned long long* __restrict__ dbg_out) {
  using Cfg = PanelCfg<kTF>;
  constexpr int kPStages = Cfg::kStages, kPStageBytes = Cfg::kStageBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  auto* sh = reinterpret_cast<PShared<kPStages>*>(stages + kPStages * kPStageBytes);
  unsigned long long t_wait = 0, t_start = clock64();
  auto timed_wait = [&](uint64_t* bar, uint32_t par) {
    if (dbg & 256) {
      unsigned long long a = clock64();
      mbar_wait(bar, par);
      t_wait += clock64() - a;
    } else {
      mbar_wait(bar, par);
    }
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t ngroups = (nbr + kGroup - 1) / kGroup;
  constexpr int kMmaWarp = 4 + kProducers;
  // A parity wait is exact only if the stage's previous use (one ring round
  // earlier) has already been waited on by the same warp: the producer count
  // must divide the ring size (every MMA warp visits every stage).
  static_assert(kPStages % kProducers == 0, "producers must divide the ring");

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(&sh->full[s], 1);           // the stage's producer arrives once
      mbar_init(&sh->empty[s], kMmaWarps);  // every MMA warp commits once
    }
    mbar_init(&sh->acc_full, kMmaWarps);  // every MMA warp commits once per group
    mbar_init(&sh->acc_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh->tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh->tmem_base;
  if (warp < 4) {  // accumulators start at zero
    const uint32_t lanes = (uint32_t)(warp * 32) << 16;
    for (int col = 0; col < kGroup * kBlk; col += 16) tmem_zero16(tmem + lanes + col);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // Positions of this CTA's ring: group g (g = blockIdx.x + k * gridDim.x)
  // holds ns stages at tg .. tg + ns - 1 and its end marker at tg + ns.
  struct Pos {
    int32_t g, i, s0, ns;
    uint32_t tg;
  };
  auto settle = [&](Pos& p) {  // carry i past the end of group g into later groups
    while (p.g < ngroups && p.i > p.ns) {
      p.i -= p.ns + 1;
      p.tg += (uint32_t)p.ns + 1;
      p.g += gridDim.x;
      if (p.g < ngroups) {
        p.s0 = __ldg(sbase + p.g);
        p.ns = __ldg(sbase + p.g + 1) - p.s0;
      }
    }
  };
  auto first = [&](int i0) {
    Pos p{(int32_t)blockIdx.x, i0, 0, 0, 0u};
    if (p.g < ngroups) {
      p.s0 = __ldg(sbase + p.g);
      p.ns = __ldg(sbase + p.g + 1) - p.s0;
    }
    settle(p);
    return p;
  };

  if (warp >= 4 && warp < kMmaWarp) {
    // --------------------------------------------------------- producers
    // Descriptors (k_bcsr_sched) are 32 words, read with one coalesced
    // load two positions ahead, so no global latency sits between a free
    // stage and its copies.
    const int q = warp - 4;
    auto load = [&](const Pos& p, uint32_t& w0) {
      w0 = 0u;
      if (p.g < ngroups && p.i < p.ns) w0 = __ldg(sdesc + (int64_t)(p.s0 + p.i) * kDescWords + lane);
    };
    Pos cur = first(q);
    Pos n1 = cur;
    n1.i += kProducers;
    settle(n1);
    uint32_t c0, a0;
    load(cur, c0);
    load(n1, a0);
    while (cur.g < ngroups) {
      Pos n2 = n1;
      n2.i += kProducers;
      settle(n2);
      uint32_t b0;
      load(n2, b0);
      const uint32_t tq = cur.tg + (uint32_t)cur.i;
      const int stage = (int)(tq % kPStages);
      const uint32_t phase = (tq / kPStages) & 1u;
      if (lane == 0) timed_wait(&sh->empty[stage], phase ^ 1);
      __syncwarp();
      uint8_t* st = stages + stage * kPStageBytes;
      if (cur.i < cur.ns) {
        const uint32_t head = __shfl_sync(kFull, c0, 0);
        const int ntile = (int)(head & 0xff), nblk = (int)(head >> 8 & 0xff);
        const uint32_t tbc = __shfl_sync(kFull, c0, 1 + (lane & 3));
        const uint32_t tmask = __shfl_sync(kFull, c0, 5 + (lane & 3));
        if (lane >= 10 && lane < 10 + Cfg::kPanelA / 4) sts_u32(smem_u32(&sh->slot[stage][4 * (lane - 10)]), c0);
        if (lane < 4) {
          sts_u32(smem_u32(&sh->mask[stage][lane]), lane < ntile ? tmask : 0u);
          if (lane < ntile && !(dbg & 2)) {
            if constexpr (kTF) {
              mbar_expect_tx_only(&sh->full[stage], 2 * Cfg::kTile);
              tma_3d(st + lane * Cfg::kTile, &tmap_b, &sh->full[stage], 0, (int)tbc * kBlk, 0);
              tma_3d(st + Cfg::kLoTile + lane * Cfg::kTile, &tmap_lo, &sh->full[stage], 0, (int)tbc * kBlk, 0);
            } else {
              mbar_expect_tx_only(&sh->full[stage], Cfg::kTile);
              tma_3d(st + lane * Cfg::kTile, &tmap_b, &sh->full[stage], 0, (int)tbc * kBlk, 0);
            }
          }
        }
        // value blocks: one TMA each (the lane holding the slot's block
        // index), written in the 32-byte-swizzled K-major layout (tf32: a
        // 3-D box puts the two K halves of 8 one after the other)
        if (lane == 0 && !(dbg & 4)) mbar_expect_tx_only(&sh->full[stage], nblk * Cfg::kA);
        __syncwarp();
        if (lane >= 16 && lane < 16 + nblk && !(dbg & 4)) {
          const int sl = lane - 16;
          if constexpr (kTF)
            tma_3d(st + Cfg::kVal + sl * Cfg::kA, &tmap_v, &sh->full[stage], 0, (int)c0 * kBlk, 0);
          else
            tma_2d(st + Cfg::kVal + sl * Cfg::kA, &tmap_v, &sh->full[stage], 0, (int)c0 * kBlk);
        }
      } else if (lane < 4) {
        sts_u32(smem_u32(&sh->mask[stage][lane]), 0u);  // end-of-group marker
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh->full[stage]);
      cur = n1;
      n1 = n2;
      c0 = a0;
      a0 = b0;
    }
  } else if (warp >= kMmaWarp) {
    // ------------------------------------------------------- MMA issuers
    // Every MMA warp walks every stage and issues the MMAs of its own block
    // rows (j % kMmaWarps == w): an accumulator's MMAs come from one warp in
    // ring order, so the fp32 accumulation order — and C — is the same on
    // every run. Per stage the lanes fetch slot s = lane's (block row, tile)
    // byte in parallel; the issue loop broadcasts one byte per slot.
    const int w = warp - kMmaWarp;
    const uint32_t base0 = smem_u32(stages);
    // A (the B tiles), MN-major: bf16 SW128 (8-row K groups, SBO 1 KB);
    // tf32 only takes SW128 with 32-byte atoms (layout type 1, 4-row K
    // groups, SBO 512 B). Both: 2 KB between the 128-byte column boxes.
    const uint64_t adesc0 = kTF ? smem_desc(base0, 2048, 512, 1) : smem_desc(base0, 2048, 1024, 2);
    const uint64_t bdesc0 = smem_desc(base0 + Cfg::kVal, 16, 256, 6);  // SW32, K-major
    uint32_t tg = 0;  // ring position of the group's first stage
    int it = 0;
    for (int32_t g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
      const int32_t ns = __ldg(sbase + g + 1) - __ldg(sbase + g);
      mbar_wait(&sh->acc_empty, (it & 1) ^ 1);  // accumulators drained and cleared
      tc_fence_after();
      for (uint32_t tq = tg; tq <= tg + (uint32_t)ns; ++tq) {  // the group's stages and its end marker
        const int stage = (int)(tq % kPStages);
        const uint32_t phase = (tq / kPStages) & 1u;
        timed_wait(&sh->full[stage], phase);
        tc_fence_after();
        const uint4 mv = lds_v4(smem_u32(&sh->mask[stage][0]));
        const int nblk = __popc(mv.x) + __popc(mv.y) + __popc(mv.z) + __popc(mv.w);
        uint32_t b = 0;
        if (lane < nblk) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(b) : "r"(smem_u32(&sh->slot[stage][lane])));
        const uint32_t mine = __ballot_sync(kFull, lane < nblk && (int)((b & 31u) % kMmaWarps) == w);  // my slots
        if constexpr (kTF) {
          // split this warp's staged value blocks: hi in place, lo beside them
          const uint32_t vbase = base0 + stage * kPStageBytes + Cfg::kVal;
          for (uint32_t ms = mine; ms; ms &= ms - 1) {
            const int sl = __ffs(ms) - 1;
#pragma unroll
            for (int t = 0; t < Cfg::kA / 16 / 32; ++t) {
              const uint32_t a = vbase + sl * Cfg::kA + (t * 32 + lane) * 16;
              const uint4 x = lds_v4(a);
              const uint4 h =
                  make_uint4(x.x & 0xffffe000u, x.y & 0xffffe000u, x.z & 0xffffe000u, x.w & 0xffffe000u);
              const uint4 l = make_uint4(__float_as_uint(__uint_as_float(x.x) - __uint_as_float(h.x)),
                                         __float_as_uint(__uint_as_float(x.y) - __uint_as_float(h.y)),
                                         __float_as_uint(__uint_as_float(x.z) - __uint_as_float(h.z)),
                                         __float_as_uint(__uint_as_float(x.w) - __uint_as_float(h.w)));
              sts_v4(a, h);
              sts_v4(a + (Cfg::kLoVal - Cfg::kVal), l);
            }
          }
        }
        if constexpr (kTF) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // split stores -> MMA reads
        __syncwarp();
        const uint64_t soff = (uint64_t)((stage * kPStageBytes) >> 4);
        if (!(dbg & 1)) {
          for (uint32_t ms = mine; ms; ms &= ms - 1) {
            const int sl = __ffs(ms) - 1;
            const uint32_t pk = __shfl_sync(kFull, b, sl);
            const uint32_t acc = tmem + (pk & 31u) * kBlk;
            const uint64_t ad = adesc0 + soff + (pk >> 5) * (Cfg::kTile >> 4);
            const uint64_t bd = bdesc0 + soff + (uint32_t)sl * (Cfg::kA >> 4);
            if constexpr (kTF) {
              constexpr uint32_t lo_a = Cfg::kLoTile >> 4, lo_b = (Cfg::kLoVal - Cfg::kVal) >> 4;
#pragma unroll
              for (int h = 0; h < 2; ++h) {  // K half: tile rows 8h.., value-block half h
                const uint64_t ah = ad + h * (1024 >> 4), bh = bd + h * (512 >> 4);
                tc_mma_elect_tf32(acc, ah, bh, Cfg::kId);
                tc_mma_elect_tf32(acc, ah + lo_a, bh, Cfg::kId);
                tc_mma_elect_tf32(acc, ah, bh + lo_b, Cfg::kId);
              }
            } else {
              tc_mma_elect(acc, ad, bd, Cfg::kId, 1u);
            }
          }
        }
        tc_commit_elect(&sh->empty[stage]);  // one of kMmaWarps arrivals
        __syncwarp();
      }
      tc_commit_elect(&sh->acc_full);  // fires when this warp's MMAs of the group are done
      __syncwarp();
      tg += (uint32_t)ns + 1;
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // Drain the group's accumulators into C, clear them, hand them back.
    int it = 0;
    const int col = warp * 32 + lane;
    const uint32_t lanes = (uint32_t)(warp * 32) << 16;
    for (int32_t g = blockIdx.x; g < ngroups; g += gridDim.x, ++it) {
      timed_wait(&sh->acc_full, it & 1);
      tc_fence_after();
      for (int j = 0; j < kGroup; ++j) {
        const int64_t r0 = ((int64_t)g * kGroup + j) * kBlk;
        if (r0 >= m) break;
        float v[16];
        tc_ld16(tmem + lanes + j * kBlk, v);
#pragma unroll
        for (int i = 0; i < kBlk; ++i) {
          if (r0 + i < m) {
            float* p = c + (r0 + i) * ldc + col;
            *p = accumulate ? *p + v[i] : v[i];
          }
        }
      }
      for (int cc = 0; cc < kGroup * kBlk; cc += 16) tmem_zero16(tmem + lanes + cc);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh->acc_empty);
    }
  }
  if ((dbg & 256) && lane == 0) {
    atomicAdd(dbg_out + 2 * warp, t_wait);
    atomicAdd(dbg_out + 2 * warp + 1, clock64() - t_start);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Stage schedule of the panel SpMM, built once per matrix from the mask
// plan and cached on the tensor. The plan of a group is cut into segments of
// kSegCols block columns; a warp per (group, segment) walks its columns in
// order and packs the nonzero ones greedily into stages of <= kPanel tiles
// and <= kPanelA value blocks (a stage never spans two segments). The
// stages of a group stay contiguous and in block-column order. kWrite =
// false counts the segment's stages (sbase[seg]) and, per lane, the blocks
// of that lane's block row in it (bcnt[seg][lane]); kWrite = true writes,
// from stage sbase[seg] on and with the lane's first value block
// bcnt[seg][lane] (both made exclusive prefixes in between), one descriptor
// per stage — [0] ntile | nblk << 8, [1..4] tile block columns, [5..8] tile
// masks, [10..13] per slot one byte (block row | tile << 5), [16 + slot]
// the slot's value block.
constexpr int kSegCols = 2048;

template <bool kWrite>
__global__ void __launch_bounds__(256) k_bcsr_sched(const uint32_t* __restrict__ plan, int32_t nbr, int32_t nbc,
                                                     int32_t nseg, int panel, int panel_a, int32_t* __restrict__ sbase,
                                                     int32_t* __restrict__ bcnt, uint32_t* __restrict__ sdesc) {
  const int lane = threadIdx.x & 31;
  const int32_t ngroups = (nbr + kGroup - 1) / kGroup;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t gs = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gs < (int64_t)ngroups * nseg;
       gs += warps) {
    const int64_t g = gs / nseg;
    const int32_t c_lo = (int32_t)(gs - g * nseg) * kSegCols;
    const int32_t c_hi = min(nbc, c_lo + kSegCols);
    int32_t cur = kWrite ? bcnt[gs * 32 + lane] : 0;
    int32_t stage = kWrite ? sbase[gs] : 0;
    int ntile = 0, nblk = 0;
    uint32_t my_bc = 0, my_mask = 0;  // lane t < kPanel: tile t of the open stage
    auto close = [&]() {
      if (kWrite) {
        uint32_t* d = sdesc + (int64_t)stage * kDescWords;
        if (lane == 0) d[0] = (uint32_t)ntile | ((uint32_t)nblk << 8);
        if (lane < 4) {
          d[1 + lane] = lane < ntile ? my_bc : 0u;
          d[5 + lane] = lane < ntile ? my_mask : 0u;
        }
      }
      ++stage;
      ntile = 0;
    };
    const uint32_t* pg = plan + g * nbc;
    for (int32_t bc0 = c_lo; bc0 < c_hi; bc0 += 32) {
      const uint32_t mine = bc0 + lane < c_hi ? __ldg(pg + bc0 + lane) : 0u;
      uint32_t nz = __ballot_sync(kFull, mine != 0);
      while (nz) {
        const int src = __ffs(nz) - 1;
        nz &= nz - 1;
        uint32_t rest = __shfl_sync(kFull, mine, src);
        while (rest) {
          // a block column held by more than kPanelA block rows is split
          // into several tiles (the B tile is loaded once per tile)
          uint32_t mask = rest;
          if (__popc(rest) > panel_a) {
            mask = 0;
            uint32_t t = rest;
            for (int k = 0; k < panel_a; ++k) {
              const uint32_t low = t & (0u - t);
              mask |= low;
              t ^= low;
            }
          }
          rest ^= mask;
          const int cnt = __popc(mask);
          if (ntile && (ntile == panel || nblk + cnt > panel_a)) close();
          if (!ntile) nblk = 0;
          if (lane == ntile) {
            my_bc = (uint32_t)(bc0 + src);
            my_mask = mask;
          }
          if (kWrite && (mask >> lane & 1u)) {
            const int sl = nblk + __popc(mask & ((1u << lane) - 1u));
            sdesc[(int64_t)stage * kDescWords + 16 + sl] = (uint32_t)cur;
            reinterpret_cast<uint8_t*>(sdesc + (int64_t)stage * kDescWords + 10)[sl] = (uint8_t)(lane | (ntile << 5));
          }
          if (mask >> lane & 1u) ++cur;
          nblk += cnt;
          ++ntile;
        }
      }
    }
    if (ntile) close();
    if (!kWrite) {
      if (lane == 0) sbase[gs] = stage;
      bcnt[gs * 32 + lane] = cur;
    }
  }
}

// Per (group, lane): the block counts of the lane's block row per segment
// become each segment's first value block (ptr[br] + the blocks before it).
__global__ void k_sched_first_blocks(const int32_t* __restrict__ ptr, int32_t nbr, int32_t nseg,
                                     int32_t* __restrict__ bcnt) {
  const int32_t ngroups = (nbr + kGroup - 1) / kGroup;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)ngroups * 32;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t / 32, lane = t % 32, br = g * kGroup + lane;
    int32_t run = br < nbr ? __ldg(ptr + br) : 0;
    for (int32_t s = 0; s < nseg; ++s) {
      int32_t* c = bcnt + ((g * nseg + s) * 32 + lane);
      const int32_t n = *c;
      *c = run;
      run += n;
    }
  }
}

// tc_base[g] = the first stage of group g (its first segment's), g <= ngroups
__global__ void k_sched_group_base(const int32_t* __restrict__ sbase, int32_t ngroups, int32_t nseg,
                                   int32_t* __restrict__ gbase) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g <= ngroups; g += (int64_t)gridDim.x * blockDim.x)
    gbase[g] = sbase[g * nseg];
}

// In-place exclusive scan of n + 1 counts (n small: one CTA, chunked).
__global__ void __launch_bounds__(1024) k_scan_small(int32_t* __restrict__ v, int32_t n) {
  __shared__ int32_t sm[34];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int32_t b = 0; b <= n; b += 1024) {
    const int32_t i = b + threadIdx.x;
    const int32_t x = i < n ? v[i] : 0;
    int32_t total;
    const int32_t ex = block_exclusive_scan<int32_t, 1024>(x, sm, &total);
    if (i <= n) v[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
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

// ------------------------------------------------------------------------
// BCSR(4,4) bf16 SpMM on tcgen05. A 4 x 4 block is far below an MMA tile, so
// the MMA covers a 128-row x 16-column window of A: N = 128 (the 32 block
// rows of a group), K = 16 (a "super column" of 4 block columns), M = 128
// (nd):  D[nd][128 rows] += B[16 sc .. 16 sc + 15][nd]^T . A_window^T.
// The A operand is the same 16-row B tile as the 16x16 kernel (one TMA);
// the B operand is the window's values, K-major with 32-byte swizzle, built
// in shared memory by the producer warp: lane j owns block row 32 g + j, i.e.
// window rows 4j .. 4j + 3, and writes them whole (its blocks of the super
// column in place, zeros elsewhere), so no separate zero fill is needed.
// Super columns without any block of the group are skipped (warp min of
// the lanes' next block columns). At 10 % block density a window holds
// ~13 of its 128 block slots; the MMA reads 8 KB of shared memory for them
// (4 KB tile + 4 KB window), against 4.5 KB per 16 x 16 block.
// A CTA runs kQPipes independent pipelines (producer warp, MMA warp, ring of
// kQStages stages, a 128-column TMEM accumulator), each on its own groups;
// the 4 epilogue warps drain them in turn.
constexpr int kQPipes = 4;
constexpr int kQStages = 5;
constexpr int kQTile = kTileBytes;  // 4 KB: 16 B rows x 128 columns
constexpr int kQVal = 128 * 32;     // 4 KB: 128 window rows x 16 K bf16
constexpr int kQStageBytes = kQTile + kQVal;
// F32 accumulate, BF16 x BF16, A MN-major, B K-major, N = 128, M = 128
constexpr uint32_t kQIdesc =
    (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(kND >> 4) << 24);

struct QShared {
  uint64_t full[kQPipes][kQStages];
  uint64_t empty[kQPipes][kQStages];
  uint64_t acc_full[kQPipes];
  uint64_t acc_empty[kQPipes];
  uint32_t end[kQPipes][kQStages];  // 1: the stage is a group's end marker
  alignas(16) uint32_t ring_col[kQPipes][32][12];     // per producer lane: block columns of three quads
  alignas(16) uint8_t ring_val[kQPipes][32][12 * 32 + 16];  // and their value blocks (+16: lanes on distinct banks)
  alignas(16) uint32_t dring[kQPipes][2 * 32][8];        // window schedule: 2 blocks of 32 (super column, masks)
  uint32_t tmem_base;
};

__global__ void __launch_bounds__(32 * (4 + 2 * kQPipes), 1)
    k_bcsr4_tc(const __grid_constant__ CUtensorMap tmap_b, const uint8_t* __restrict__ aval,
               const int32_t* __restrict__ ptr, const int32_t* __restrict__ bcol, int64_t nnz, int32_t nbr,
               int32_t m, float* __restrict__ c, int64_t ldc, int accumulate, const int32_t* __restrict__ gstart,
               const int32_t* __restrict__ dsc, const uint4* __restrict__ dmask) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* stages = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  QShared* sh = reinterpret_cast<QShared*>(stages + kQPipes * kQStages * kQStageBytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t ngroups = (nbr + kGroup - 1) / kGroup;
  constexpr int kMmaWarp = 4 + kQPipes;
  if (threadIdx.x == 0) {
    for (int w = 0; w < kQPipes; ++w) {
      for (int s = 0; s < kQStages; ++s) {
        mbar_init(&sh->full[w][s], 1);   // producer lane 0 (plus the tile's bytes)
        mbar_init(&sh->empty[w][s], 1);  // the MMA warp's commit
      }
      mbar_init(&sh->acc_full[w], 1);
      mbar_init(&sh->acc_empty[w], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sh->tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh->tmem_base;
  auto group_of = [&](int k, int w) { return (int32_t)blockIdx.x + (k * kQPipes + w) * (int32_t)gridDim.x; };

  if (warp >= 4 && warp < kMmaWarp) {
    // ---------------------------------------------------------- producers
    // Lane j walks block row 32 g + j through a ring of three aligned quads
    // of blocks (block columns + 32 value bytes each) in shared memory,
    // refilled by cp.async a quad at a time: when the walk enters quad Q the
    // vacated slot is refilled with Q + 2 and the lane waits for Q + 1, so
    // the current and the next quad are always resident — a stage reads the
    // lane's next four blocks at once, with no loop and no load latency
    // (register look-ahead stalls instead: shifting a register whose load is
    // in flight waits for it). An L2 prefetch runs 64 blocks ahead. The lane
    // zeroes its four window rows, then copies its blocks of the super
    // column into them.
    const int w = warp - 4;
    int stage = 0;
    uint32_t phase = 0;
    constexpr uint32_t kNone = 0xffffffffu;
    const uint32_t sw = (uint32_t)lane & 1u;  // 32-byte swizzle: chunk ^= (row >> 2) & 1, row >> 2 = lane
    const uint32_t rcol = smem_u32(&sh->ring_col[w][lane][0]);
    const uint32_t rval = smem_u32(&sh->ring_val[w][lane][0]);
    for (int k = 0;; ++k) {
      const int32_t g = group_of(k, w);
      if (g >= ngroups) break;
      const int32_t br = g * kGroup + lane;
      int64_t cur = 0, end = 0;
      if (br < nbr) {
        cur = __ldg(ptr + br);
        end = __ldg(ptr + br + 1);
      }
      auto slot = [](int64_t i) {  // ring entry of block i (32-bit modulo: block indices < 2^31)
        return ((((uint32_t)(i >> 2)) % 3u) << 2) | (uint32_t)(i & 3);
      };
      // quad q0 (blocks q0 .. q0 + 3, q0 % 4 == 0): one cp.async group
      auto refill = [&](int64_t q0) {
        if (q0 < end) {
          const uint32_t s0 = slot(q0);
          const int64_t nc = nnz - q0 < 4 ? nnz - q0 : 4;  // entries of the column array left
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(rcol + s0 * 4), "l"(bcol + q0),
                       "r"((int)nc * 4)
                       : "memory");
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const bool in = q0 + e < nnz;
            const uint8_t* src = aval + (in ? (q0 + e) * 32 : 0);
            const uint32_t dst = rval + (s0 + e) * 32;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(in ? 16 : 0)
                         : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + 16), "l"(src + 16),
                         "r"(in ? 16 : 0)
                         : "memory");
          }
          if (q0 + 64 < end) asm volatile("prefetch.global.L2 [%0];" ::"l"(aval + (q0 + 64) * 32));
          if (((q0 + 64) & 31) == 0 && q0 + 64 < end) asm volatile("prefetch.global.L2 [%0];" ::"l"(bcol + q0 + 64));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      for (int64_t i = cur & ~int64_t(3); i < cur + 64 && i < end; i += 4)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(aval + i * 32));
      const int64_t qb = cur & ~int64_t(3);
      refill(qb);
      refill(qb + 4);
      refill(qb + 8);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      auto col_of = [&](int64_t i) -> uint32_t {
        if (i >= end) return kNone;
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(rcol + slot(i) * 4));
        return v;
      };
      if (gstart != nullptr) {
        // the per-matrix window schedule: each stage's super column and the
        // lanes' 4-bit block masks (k_q_plan / k_q_compact) — no column
        // reads, no compares, no warp min
        // descriptors in blocks of 32 stages: lane l loads stage (block +
        // l)'s into registers one block ahead and parks them in a shared
        // ring at the next block's start, so no load latency meets a stage
        const int32_t t0 = __ldg(gstart + g), t1 = __ldg(gstart + g + 1);
        const uint32_t dr = smem_u32(&sh->dring[w][0][0]);
        int32_t psc = 0;
        uint4 pmk = make_uint4(0, 0, 0, 0);
        if (t0 + lane < t1) psc = __ldg(dsc + t0 + lane), pmk = __ldg(dmask + t0 + lane);
        for (int32_t t = t0; t < t1; ++t) {
          const int32_t j = (t - t0) & 31;
          if (j == 0) {  // a new block: park its descriptors, request the next block's
            const uint32_t at = dr + ((((t - t0) >> 5) & 1) * 32 + lane) * 32;
            sts_u32(at, (uint32_t)psc);
            sts_v4(at + 16, pmk);
            __syncwarp();
            const int32_t tn = t + 32 + lane;
            if (tn < t1) psc = __ldg(dsc + tn), pmk = __ldg(dmask + tn);
          }
          const uint32_t at = dr + ((((t - t0) >> 5) & 1) * 32 + j) * 32;
          uint32_t sc, word;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(sc) : "r"(at));
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(word) : "r"(at + 16 + (lane >> 3) * 4));
          const uint32_t nib = (word >> ((lane & 7) * 4)) & 0xfu;
          if (lane == 0) mbar_wait(&sh->empty[w][stage], phase ^ 1);
          __syncwarp();
          uint8_t* st = stages + (w * kQStages + stage) * kQStageBytes;
          if (lane == 0) {
            sh->end[w][stage] = 0;
            mbar_expect_tx_only(&sh->full[w][stage], kQTile);
            tma_3d(st, &tmap_b, &sh->full[w][stage], 0, (int)sc * kBlk, 0);
          }
          const uint32_t vb = smem_u32(st + kQTile) + (uint32_t)lane * 128u;
#pragma unroll
          for (int i = 0; i < 8; ++i)  // rotated by lane: 8 consecutive lanes hit 8 different bank groups
            sts_v4(vb + (((uint32_t)(i + lane) & 7u) << 4), make_uint4(0u, 0u, 0u, 0u));
          int e = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (nib >> q & 1u) {  // the lane's blocks of this super column, in column order
              const uint32_t src = rval + slot(cur + e) * 32;
              const uint4 lo = lds_v4(src), hi = lds_v4(src + 16);
              const uint32_t off = ((((uint32_t)q >> 1) ^ sw) << 4) + (((uint32_t)q & 1u) << 3);
              asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(vb + off), "r"(lo.x), "r"(lo.y) : "memory");
              asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(vb + 32 + off), "r"(lo.z), "r"(lo.w) : "memory");
              asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(vb + 64 + off), "r"(hi.x), "r"(hi.y) : "memory");
              asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(vb + 96 + off), "r"(hi.z), "r"(hi.w) : "memory");
              ++e;
            }
          if (e) {
            const int64_t q_old = cur >> 2;
            cur += e;
            if ((cur >> 2) != q_old) {  // entered the next quad: refill the vacated slot, wait for the one after
              refill(((cur >> 2) + 2) * 4);
              asm volatile("cp.async.wait_group 1;" ::: "memory");
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sh->full[w][stage]);
          if (++stage == kQStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      } else {
      uint32_t nb = col_of(cur);
      while (true) {
        const uint32_t mn = __reduce_min_sync(kFull, nb);
        if (mn == kNone) break;
        const uint32_t sc = mn >> 2;
        if (lane == 0) mbar_wait(&sh->empty[w][stage], phase ^ 1);
        __syncwarp();
        uint8_t* st = stages + (w * kQStages + stage) * kQStageBytes;
        if (lane == 0) {
          sh->end[w][stage] = 0;
          mbar_expect_tx_only(&sh->full[w][stage], kQTile);
          tma_3d(st, &tmap_b, &sh->full[w][stage], 0, (int)sc * kBlk, 0);
        }
        // the lane's window rows 4 lane .. 4 lane + 3: zero, then its blocks
        const uint32_t vb = smem_u32(st + kQTile) + (uint32_t)lane * 128u;
#pragma unroll
        for (int i = 0; i < 8; ++i)  // rotated by lane: 8 consecutive lanes hit 8 different bank groups
          sts_v4(vb + (((uint32_t)(i + lane) & 7u) << 4), make_uint4(0u, 0u, 0u, 0u));
        uint32_t c[4];
        c[0] = nb;
#pragma unroll
        for (int e = 1; e < 4; ++e) c[e] = col_of(cur + e);
        int taken = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if ((c[e] >> 2) == sc) {  // columns ascend: the taken blocks are a prefix
            const uint32_t q = c[e] & 3u;
            const uint32_t src = rval + slot(cur + e) * 32;
            const uint4 lo = lds_v4(src), hi = lds_v4(src + 16);
            // block column q: bytes 8q .. 8q + 7 of each row (chunk q / 2)
            const uint32_t off = (((q >> 1) ^ sw) << 4) + ((q & 1u) << 3);
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(vb + off), "r"(lo.x), "r"(lo.y) : "memory");
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(vb + 32 + off), "r"(lo.z), "r"(lo.w) : "memory");
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(vb + 64 + off), "r"(hi.x), "r"(hi.y) : "memory");
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(vb + 96 + off), "r"(hi.z), "r"(hi.w) : "memory");
            ++taken;
          }
        }
        if (taken) {
          const int64_t q_old = cur >> 2;
          cur += taken;
          if ((cur >> 2) != q_old) {  // entered the next quad: refill the vacated slot, wait for the one after
            refill(((cur >> 2) + 2) * 4);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          }
          nb = col_of(cur);
        }
        __syncwarp();
        // the MMA warp fences (generic -> async proxy) after the barrier
        if (lane == 0) mbar_arrive(&sh->full[w][stage]);
        if (++stage == kQStages) {
          stage = 0;
          phase ^= 1;
        }
      }
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");  // the ring is rewritten by the next group
      // end-of-group marker
      if (lane == 0) {
        mbar_wait(&sh->empty[w][stage], phase ^ 1);
        sh->end[w][stage] = 1;
        mbar_arrive(&sh->full[w][stage]);
      }
      __syncwarp();
      if (++stage == kQStages) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp >= kMmaWarp) {
    // ------------------------------------------------------- MMA issuers
    const int w = warp - kMmaWarp;

    int stage = 0;
    uint32_t phase = 0;
    for (int k = 0;; ++k) {
      const int32_t g = group_of(k, w);
      if (g >= ngroups) break;
      mbar_wait(&sh->acc_empty[w], (k & 1) ^ 1);
      tc_fence_after();
      uint32_t acc_on = 0;  // the group's first MMA overwrites the accumulator
      while (true) {
        mbar_wait(&sh->full[w][stage], phase);
        tc_fence_after();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // producer st.shared -> MMA reads
        uint32_t endm;  // explicit shared load (a volatile generic load compiles to a slow system-scope one)
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(endm) : "r"(smem_u32(&sh->end[w][stage])));
        if (!endm) {
          const uint32_t base = smem_u32(stages + (w * kQStages + stage) * kQStageBytes);
          tc_mma_elect(tmem + w * 128, smem_desc(base, 2048, 1024, 2), smem_desc(base + kQTile, 16, 256, 6), kQIdesc,
                       acc_on);
          acc_on = 1;
        }
        tc_commit_elect(&sh->empty[w][stage]);
        __syncwarp();
        if (++stage == kQStages) {
          stage = 0;
          phase ^= 1;
        }
        if (endm) break;
      }
      tc_commit_elect(&sh->acc_full[w]);
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------- epilogue
    const int col = warp * 32 + lane;
    const uint32_t lanes = (uint32_t)(warp * 32) << 16;
    for (int k = 0;; ++k) {
      bool done = false;
      for (int w = 0; w < kQPipes; ++w) {
        const int32_t g = group_of(k, w);
        if (g >= ngroups) {
          done = true;
          break;
        }
        mbar_wait(&sh->acc_full[w], k & 1);
        tc_fence_after();
        const int32_t b_lo = g * kGroup, b_hi = min(b_lo + kGroup, nbr);
        const bool any = __ldg(ptr + b_lo) < __ldg(ptr + b_hi);  // else no MMA ran: the rows are zero
        for (int n0 = 0; n0 < 128; n0 += 16) {
          float v[16];
          if (any) {
            tc_ld16(tmem + lanes + w * 128 + n0, v);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.f;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int64_t row = (int64_t)g * 128 + n0 + i;
            if (row < m) {
              float* p = c + row * ldc + col;
              *p = accumulate ? *p + v[i] : v[i];
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh->acc_empty[w]);
      }
      if (done) break;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Window schedule of the BCSR(4,4) kernel, built once per matrix and cached
// on the tensor: per (group of 32 block rows, super column of 4 block
// columns) a 16-byte mask — 4 bits per block row (lane), bit q = block
// column 4 sc + q present — then the nonempty (group, super column) pairs
// compacted in order: the stage list of each group, its super columns and
// masks.
__global__ void k_q_plan(const int32_t* __restrict__ ptr, const int32_t* __restrict__ bcol, int32_t nbr,
                         int64_t nsc, uint32_t* __restrict__ plan) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t br = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; br < nbr; br += warps) {
    uint32_t* pg = plan + (br >> 5) * nsc * 4 + ((br & 31) >> 3);
    const uint32_t sh = (uint32_t)(br & 7) * 4;
    for (int32_t k = __ldg(ptr + br) + lane; k < __ldg(ptr + br + 1); k += 32) {
      const int32_t bc = __ldg(bcol + k);
      atomicOr(pg + (int64_t)(bc >> 2) * 4, 1u << (sh + (bc & 3)));
    }
  }
}

__global__ void k_q_flags(const uint4* __restrict__ plan, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(plan + i);
    flag[i] = (v.x | v.y | v.z | v.w) != 0u ? 1 : 0;
  }
}

__global__ void k_q_compact(const uint4* __restrict__ plan, const int32_t* __restrict__ pos, int64_t n, int64_t nsc,
                            int64_t ngroups, int32_t* __restrict__ dsc, uint4* __restrict__ dmask,
                            int32_t* __restrict__ gstart) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = __ldg(pos + i);
    if (__ldg(pos + i + 1) > p) {
      dsc[p] = (int32_t)(i % nsc);
      dmask[p] = __ldg(plan + i);
    }
    if (i % nsc == 0) gstart[i / nsc] = p;
    if (i == n - 1) gstart[ngroups] = __ldg(pos + n);
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
  // bf16 values and B: one kind::f16 MMA per block; fp32 values and B:
  // 3xTF32 (panel schedule only)
  const bool tf = a->dtype == SFG_F32 && b_dtype == SFG_F32;
  const bool bf = a->dtype == SFG_BF16 && b_dtype == SFG_BF16;
  if (a->kind != SFG_BCSR || !(tf || bf) || nd != kND) return false;
  const bool quad = bf && a->br == 4 && a->bc == 4 && a->rb == 4 && a->cb == 4;  // BCSR(4,4): 128-row windows
  if (!quad && (a->br != kBlk || a->bc != kBlk || a->rb != kBlk || a->cb != kBlk)) return false;
  if (reinterpret_cast<uintptr_t>(b) & 15 || a->nnz == 0) return false;
  if (bf ? (ldb * 2) % 16 != 0 : ldb % 4 != 0) return false;
  if (a->nbr > INT32_MAX || a->nnz > INT32_MAX || (!quad && a->nnz * kBlk > INT32_MAX)) return false;
  const int64_t ngroups = ceil_div(a->nbr, kGroup);
  const int64_t words = ngroups * a->nbc;
  const bool plan_ok = a->nnz * 4 >= words && words <= (int64_t(1) << 30);
  if (tf && !plan_ok) return false;
  // 3xTF32 splits B into hi / lo copies (2 x n x 512 bytes): only when they
  // fit comfortably, else the CUDA-core kernel takes the product
  if (tf && 2 * a->n * kND * 4 > (int64_t)(ctx->total_mem / 4)) return false;
  if (quad && a->nbr > (int64_t)INT32_MAX - kGroup) return false;
  auto encode = get_encode();
  if (!encode) return false;
  sfg_tensor* mut = const_cast<sfg_tensor*>(a);  // plan and schedule are caches, not tensor state
  int grid = (int)std::min<int64_t>(ngroups, (int64_t)ctx->sms);
  auto build_schedule = [&](int panel, int panel_a) {
    // The mask plan (per 32-block-row group, per block column) and the stage
    // schedule are built once per matrix and cached on the tensor; they are
    // used when the group masks are dense enough that streaming them beats
    // the in-kernel merge. A warp per (group, segment of kSegCols block
    // columns): count, scan, write.
    if (!mut->tc_plan) {
      mut->tc_plan = dalloc_n<uint32_t>(ctx, words);
      SFG_CUDA(cudaMemsetAsync(mut->tc_plan, 0, words * 4, ctx->stream));
      SFG_LAUNCH(k_bcsr_plan, stream_grid(ctx, a->nbr * 32, 256, 1, 8), 256, 0, ctx->stream, a->ptr, a->idx,
                 (int32_t)a->nbr, (int32_t)a->nbc, mut->tc_plan);
    }
    if (mut->tc_desc) return;
    const int32_t nseg = (int32_t)ceil_div(a->nbc, (int64_t)kSegCols);
    const int64_t nsg = ngroups * nseg;
    auto* sbase = dalloc_n<int32_t>(ctx, nsg + 1);
    auto* bcnt = dalloc_n<int32_t>(ctx, nsg * 32);
    mut->tc_base = dalloc_n<int32_t>(ctx, ngroups + 1);
    const int sgrid = stream_grid(ctx, nsg * 32, 256, 1, 8);
    SFG_LAUNCH(k_bcsr_sched<false>, sgrid, 256, 0, ctx->stream, mut->tc_plan, (int32_t)a->nbr, (int32_t)a->nbc, nseg,
               panel, panel_a, sbase, bcnt, nullptr);
    SFG_LAUNCH(k_scan_small, 1, 1024, 0, ctx->stream, sbase, (int32_t)nsg);
    SFG_LAUNCH(k_sched_first_blocks, stream_grid(ctx, ngroups * 32, 256, 1, 8), 256, 0, ctx->stream, a->ptr,
               (int32_t)a->nbr, nseg, bcnt);
    SFG_LAUNCH(k_sched_group_base, (int)ceil_div(ngroups + 1, 256), 256, 0, ctx->stream, sbase, (int32_t)ngroups,
               nseg, mut->tc_base);
    int32_t nstages = 0;
    read_back(ctx, sbase + nsg, sizeof(int32_t), &nstages);
    mut->tc_desc = dalloc_n<uint32_t>(ctx, (int64_t)nstages * kDescWords);
    SFG_LAUNCH(k_bcsr_sched<true>, sgrid, 256, 0, ctx->stream, mut->tc_plan, (int32_t)a->nbr, (int32_t)a->nbc, nseg,
               panel, panel_a, sbase, bcnt, mut->tc_desc);
    dfree(ctx, sbase);
    dfree(ctx, bcnt);
  };
#ifdef SFG_TC_DEBUG
  // profiling / ablation switches (ablations skip work: debug builds only)
  static const int dbg = (std::getenv("SFG_TC_PROF") ? 256 : 0) |
                         (std::getenv("SFG_TC_ABLATE") ? std::atoi(std::getenv("SFG_TC_ABLATE")) : 0);
#else
  constexpr int dbg = 0;
#endif
  // 4 producer and 8 MMA warps (each MMA warp owning the block rows j with
  // j % 8 == w) measured best at config 4 bf16: 22.1 ms; 4 MMA warps 22.8,
  // 2 MMA warps 31.5, 2 producers 25.1
  constexpr int kP = 4, kW = 8;
  auto run_panel = [&](auto kern, size_t psmem, const CUtensorMap& t_hi, const CUtensorMap& t_lo,
                       const CUtensorMap& t_v) {
    unsigned long long* dbg_out = nullptr;
    if (dbg) {
      dbg_out = static_cast<unsigned long long*>(scratch(ctx, 64 * 8));
      SFG_CUDA(cudaMemsetAsync(dbg_out, 0, 64 * 8, ctx->stream));
    }
    // set on every call: a once-only static setup measured 30 % slower
    // launches (0.61 vs 0.46 ms at m = 65536)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
    SFG_LAUNCH(kern, grid, 32 * (4 + kP + kW), psmem, ctx->stream, t_hi, t_lo, t_v, static_cast<const uint8_t*>(a->val),
               a->ptr, (int32_t)a->nbr, (int32_t)a->m, c, ldc, accumulate ? 1 : 0, mut->tc_base, mut->tc_desc, dbg,
               dbg_out);
    if (dbg & 256) {
      unsigned long long h[64];
      SFG_CUDA(cudaMemcpyAsync(h, dbg_out, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
      SFG_CUDA(cudaStreamSynchronize(ctx->stream));
      for (int w = 0; w < 4 + kP + kW; ++w)
        std::fprintf(stderr, "[tc prof] warp %2d: wait %5.1f%% of %.0f cycles/CTA\n", w,
                     100.0 * h[2 * w] / (double)(h[2 * w + 1] ? h[2 * w + 1] : 1), h[2 * w + 1] / (double)grid);
    }
  };
  // a dense 16-row x 128-column B tile in one 3-D copy: dims (cols per
  // 128-byte box, n, boxes), SWIZZLE_128B
  auto tile_map = [&](CUtensorMap* map, CUtensorMapDataType ty, int esz, const void* base, int64_t ld,
                      CUtensorMapSwizzle swz) {
    const int per = 128 / esz;
    cuuint64_t dims[3] = {(cuuint64_t)per, (cuuint64_t)a->n, (cuuint64_t)(kND / per)};
    cuuint64_t strides[2] = {(cuuint64_t)ld * esz, 128};
    cuuint32_t box[3] = {(cuuint32_t)per, kBlk, (cuuint32_t)(kND / per)};
    cuuint32_t es[3] = {1, 1, 1};
    if (encode(map, ty, 3, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      raise(SFG_ERR_CUDA, "cuTensorMapEncodeTiled(B tile) failed");
  };

  if (tf) {
    // B -> tf32 hi / lo (dense, ld 128), then the 3xTF32 panel kernel
    build_schedule(PanelCfg<true>::kPanel, PanelCfg<true>::kPanelA);
    float* bhi = dalloc_n<float>(ctx, a->n * kND);
    float* blo = dalloc_n<float>(ctx, a->n * kND);
    SFG_LAUNCH(k_tf32_split, stream_grid(ctx, a->n * (kND / 4), 256, 4, 8), 256, 0, ctx->stream,
               static_cast<const float*>(b), a->n, ldb, bhi, blo);
    CUtensorMap thi, tlo, tv;
    tile_map(&thi, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, bhi, kND, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    tile_map(&tlo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, blo, kND, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    {  // value blocks as (8 K, rows, 2 K halves): a box lands as [half][row][32 bytes], 32-byte swizzle
      cuuint64_t dims[3] = {8, (cuuint64_t)(a->nnz * kBlk), 2};
      cuuint64_t strides[2] = {kBlk * 4, 32};
      cuuint32_t box[3] = {8, kBlk, 2};
      cuuint32_t es[3] = {1, 1, 1};
      if (encode(&tv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a->val, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        raise(SFG_ERR_CUDA, "cuTensorMapEncodeTiled(values) failed");
    }
    run_panel(k_bcsr_tc_panel<kP, kW, true>,
              1024 + PanelCfg<true>::kStages * PanelCfg<true>::kStageBytes + sizeof(PShared<PanelCfg<true>::kStages>) +
                  64,
              thi, tlo, tv);
    dfree(ctx, bhi);
    dfree(ctx, blo);
    return true;
  }

  if (quad) {
    CUtensorMap tq;
    tile_map(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, b, ldb, CU_TENSOR_MAP_SWIZZLE_128B);
    // the window schedule (cached on the tensor: tc_base = per-group first
    // stage, tc_desc = super columns, tc_plan = masks), when its build fits
    const int64_t nsc = ceil_div(a->nbc, (int64_t)4), cells = ngroups * nsc;
    static const bool no_sched = std::getenv("SFG_Q_NOSCHED") != nullptr;  // A/B switch
    if (!no_sched && !mut->tc_base && cells < INT32_MAX && cells * 24 <= (int64_t)(ctx->total_mem / 8)) {
      auto* plan = dalloc_n<uint32_t>(ctx, cells * 4);
      auto* flag = dalloc_n<int32_t>(ctx, cells);
      auto* pos = dalloc_n<int32_t>(ctx, cells + 1);
      SFG_CUDA(cudaMemsetAsync(plan, 0, cells * 16, ctx->stream));
      SFG_LAUNCH(k_q_plan, stream_grid(ctx, a->nbr * 32, 256, 1, 8), 256, 0, ctx->stream, a->ptr, a->idx,
                 (int32_t)a->nbr, nsc, plan);
      SFG_LAUNCH(k_q_flags, stream_grid(ctx, cells, 256, 4, 8), 256, 0, ctx->stream,
                 reinterpret_cast<const uint4*>(plan), cells, flag);
      scan_counts(ctx, flag, cells, pos);
      int32_t nst = 0;
      read_back(ctx, pos + cells, sizeof nst, &nst);
      mut->tc_base = dalloc_n<int32_t>(ctx, ngroups + 1);
      mut->tc_desc = reinterpret_cast<uint32_t*>(dalloc_n<int32_t>(ctx, std::max<int32_t>(nst, 1)));
      mut->tc_plan = dalloc_n<uint32_t>(ctx, (int64_t)std::max<int32_t>(nst, 1) * 4);
      SFG_LAUNCH(k_q_compact, stream_grid(ctx, cells, 256, 4, 8), 256, 0, ctx->stream,
                 reinterpret_cast<const uint4*>(plan), pos, cells, nsc, ngroups,
                 reinterpret_cast<int32_t*>(mut->tc_desc), reinterpret_cast<uint4*>(mut->tc_plan), mut->tc_base);
      for (void* q : {(void*)plan, (void*)flag, (void*)pos}) dfree(ctx, q);
    }
    const size_t qsmem = 1024 + (size_t)kQPipes * kQStages * kQStageBytes + sizeof(QShared) + 64;
    cudaFuncSetAttribute(k_bcsr4_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsmem);
    SFG_LAUNCH(k_bcsr4_tc, grid, 32 * (4 + 2 * kQPipes), qsmem, ctx->stream, tq, static_cast<const uint8_t*>(a->val),
               a->ptr, a->idx, a->nnz, (int32_t)a->nbr, (int32_t)a->m, c, ldc, accumulate ? 1 : 0, mut->tc_base,
               reinterpret_cast<const int32_t*>(mut->tc_desc), reinterpret_cast<const uint4*>(mut->tc_plan));
    return true;
  }
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
  CUtensorMap tb3;  // both 64-column halves of a B tile in one copy: dims (64, n, 2)
  tile_map(&tb3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, b, ldb, CU_TENSOR_MAP_SWIZZLE_128B);
  const size_t smem = 1024 + kStages * kStageBytes + sizeof(Shared) + 64;
  const size_t gsmem = 1024 + kGStages * kGStageBytes + sizeof(GShared) + 64;
  static const bool per_row = [] {
    const char* v = std::getenv("SFG_BCSR_TC_PER_ROW");  // A/B switch: one block row per accumulator
    return v && *v == '1';
  }();
  if (per_row) {
    // the attribute is per device: set on every call (a few host microseconds)
    SFG_CUDA(cudaFuncSetAttribute(k_bcsr_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    SFG_LAUNCH(k_bcsr_tc, (int)std::min<int64_t>(a->nbr, (int64_t)ctx->sms), kThreads, smem, ctx->stream, tb, ta,
               a->ptr, a->idx, (int32_t)a->nbr, (int32_t)a->m, c, ldc, accumulate ? 1 : 0);
    return true;
  }
  if (plan_ok) build_schedule(PanelCfg<false>::kPanel, PanelCfg<false>::kPanelA);
  if (mut->tc_desc) {
    run_panel(k_bcsr_tc_panel<kP, kW, false>,
              1024 + PanelCfg<false>::kStages * PanelCfg<false>::kStageBytes +
                  sizeof(PShared<PanelCfg<false>::kStages>) + 64,
              tb3, tb3, ta);
  } else {
    // set on every call: a once-only static setup measured 30 % slower
    // launches of the panel kernel (0.61 vs 0.46 ms at m = 65536)
    cudaFuncSetAttribute(k_bcsr_tc_group<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem);
    SFG_LAUNCH((k_bcsr_tc_group<2, 2>), grid, 32 * 8, gsmem, ctx->stream, tb3, static_cast<const uint8_t*>(a->val),
               a->ptr, a->idx, (int32_t)a->nbr, (int32_t)a->m, c, ldc, accumulate ? 1 : 0, mut->tc_plan,
               (int32_t)a->nbc);
  }
  return true;
}

}  // namespace sfg
