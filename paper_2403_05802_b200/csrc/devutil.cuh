// devutil.cuh — device helpers: streaming loads, warp/block scans, and the
// single-pass decoupled look-back tile prefix (CUB-free).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace sfg {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- loads
// Streaming loads for data read exactly once: no L1 allocation.
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int ld_stream(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_stream(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
// Streaming stores: evict-first.
__device__ __forceinline__ void st_stream(int4* p, int4 v) {
  asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w));
}
__device__ __forceinline__ void st_stream(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w));
}

// ---------------------------------------------------------------- warp ops
template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(kFull, v, o);
    v = v > w ? v : w;
  }
  return v;
}

// Inclusive warp scan.
template <class T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T w = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += w;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix, *total gets the block sum. `smem` holds >= 33 elements.
template <class T, int kThreads>
__device__ __forceinline__ T block_exclusive_scan(T v, T* smem, T* total) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) smem[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < kThreads / 32 ? smem[lane] : T(0);
    T wi = warp_inclusive_scan(w);
    smem[lane] = wi - w;
    if (lane == 31) smem[32] = wi;
  }
  __syncthreads();
  T out = smem[warp] + inc - v;
  *total = smem[32];
  __syncthreads();
  return out;
}

// -------------------------------------------------- decoupled look-back
// Tile status word: [63:34] epoch, [33:32] state (1 aggregate, 2 inclusive
// prefix), [31:0] value. The epoch makes stale words from earlier launches
// read as "not ready", so the status array never needs clearing. Tiles are
// indexed by blockIdx.x: a tile only waits on lower-indexed CTAs, which
// were dispatched before it, so the look-back always makes progress.
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long lb_pack(uint32_t epoch, uint32_t state, uint32_t v) {
  return (static_cast<unsigned long long>(((epoch & 0x3fffffffu) << 2) | state) << 32) | v;
}

// Called by every thread of the CTA. Returns the exclusive prefix (sum of
// all earlier tiles' aggregates). Aggregates must fit in 32 bits.
__device__ __forceinline__ uint32_t lookback_prefix(unsigned long long* status, uint32_t epoch,
                                                    int tile, uint32_t aggregate,
                                                    uint32_t* smem_slot) {
  if (threadIdx.x < 32) {
    int lane = threadIdx.x;
    uint32_t ep = epoch & 0x3fffffffu;
    if (tile == 0) {
      if (lane == 0) {
        st_relaxed(&status[0], lb_pack(epoch, 2, aggregate));
        *smem_slot = 0;
      }
    } else {
      if (lane == 0) st_relaxed(&status[tile], lb_pack(epoch, 1, aggregate));
      uint32_t excl = 0;
      int look = tile - 1;
      while (true) {
        int i = look - lane;
        uint32_t st = 2, v = 0;
        if (i >= 0) {
          unsigned long long w;
          do {
            w = ld_relaxed(&status[i]);
            uint32_t hi = static_cast<uint32_t>(w >> 32);
            st = (hi >> 2) == ep ? (hi & 3u) : 0u;
          } while (st == 0);
          v = static_cast<uint32_t>(w);
        }
        unsigned pmask = __ballot_sync(kFull, st == 2);
        int stop = pmask ? __ffs(pmask) - 1 : 31;
        uint32_t c = lane <= stop ? v : 0u;
        excl += warp_sum(c);
        if (pmask) break;
        look -= 32;
      }
      if (lane == 0) {
        st_relaxed(&status[tile], lb_pack(epoch, 2, excl + aggregate));
        *smem_slot = excl;
      }
    }
  }
  __syncthreads();
  uint32_t r = *smem_slot;
  __syncthreads();
  return r;
}

// ---------------------------------------------------- row-pointer gaps
// ptr[lo..hi] = v for the rows between two consecutive sorted entries.
// Gaps longer than a warp are filled cooperatively by the whole warp, so a
// long run of empty rows costs gap/32 iterations, not gap. All 32 lanes
// must call this (warp collectives).
struct Gap {
  int32_t lo, hi, v;  // ptr[lo..hi] = v
};

__device__ __forceinline__ void fill_gaps(Gap (&g)[5], int32_t* __restrict__ ptr) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    int len = g[i].hi - g[i].lo + 1;
    bool big = len > 32;
    if (!big)
      for (int q = g[i].lo; q <= g[i].hi; ++q) ptr[q] = g[i].v;
    unsigned mask = __ballot_sync(kFull, big);
    while (mask) {
      int src = __ffs(mask) - 1;
      mask &= mask - 1;
      int lo = __shfl_sync(kFull, g[i].lo, src), hi = __shfl_sync(kFull, g[i].hi, src);
      int v = __shfl_sync(kFull, g[i].v, src);
      for (int q = lo + lane; q <= hi; q += 32) ptr[q] = v;
    }
  }
}

}  // namespace sfg
