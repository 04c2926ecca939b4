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
__device__ __forceinline__ int2 ld_stream(const int2* p) {
  int2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// (column, value) of entry k: separate arrays (S = 1), or the records of a
// packed (AoS) format — {col, val} (S = 2, one 64-bit load) or {row, col,
// val} (S = 3, col / val pointing at the record's fields).
template <int S>
__device__ __forceinline__ void ld_entry(const int32_t* __restrict__ col, const float* __restrict__ val, int64_t k,
                                         int& c, float& v) {
  if constexpr (S == 2) {
    const int2 q = ld_stream(reinterpret_cast<const int2*>(col) + k);
    c = q.x;
    v = __int_as_float(q.y);
  } else {
    c = ld_stream(col + k * S);
    v = ld_stream(val + k * S);
  }
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

// ---------------------------------------------------- row-pointer writes
// A lane owns N consecutive entries of a sorted row array, rows r[0..N-1],
// entry positions v0..v0+N-1, and `prev` = the row of the entry before
// them. For each entry i it writes ptr[q] = v0 + i for every row q in
// (r[i-1], r[i]] (the rows it opens, including empty rows before it); then
// ptr[q] = end_v for q in (r[N-1], end_hi] (end_hi = r[N-1] for "nothing":
// only the owner of the last entry closes the array up to m).
//
// Up to kInline rows per gap are written as predicated stores with no
// branch; the rest of a longer gap (a run of empty rows) is written by the
// whole warp cooperatively, so a gap of G rows costs G/32 store rounds.
// One ballot per call. All 32 lanes must call this.
template <int N>
__device__ __forceinline__ void write_row_ptr(const int32_t (&r)[N], int32_t prev, int32_t v0,
                                              int32_t end_hi, int32_t end_v,
                                              int32_t* __restrict__ ptr) {
  constexpr int kInline = 2;
  const int lane = threadIdx.x & 31;
  unsigned big = 0;
#pragma unroll
  for (int i = 0; i <= N; ++i) {
    int lo = (i ? r[i - 1] : prev) + 1;
    int hi = i < N ? r[i] : end_hi;
    int v = i < N ? v0 + i : end_v;
#pragma unroll
    for (int j = 0; j < kInline; ++j)
      if (lo + j <= hi) ptr[lo + j] = v;
    if (hi - lo >= kInline) big |= 1u << i;
  }
  unsigned lanes = __ballot_sync(kFull, big != 0);
  while (lanes) {
    int src = __ffs(lanes) - 1;
    lanes &= lanes - 1;
    unsigned which = __shfl_sync(kFull, big, src);
#pragma unroll
    for (int i = 0; i <= N; ++i) {
      if (!(which >> i & 1u)) continue;
      int lo = __shfl_sync(kFull, (i ? r[i - 1] : prev) + 1 + kInline, src);
      int hi = __shfl_sync(kFull, i < N ? r[i] : end_hi, src);
      int v = __shfl_sync(kFull, i < N ? v0 + i : end_v, src);
      for (int q = lo + lane; q <= hi; q += 32) ptr[q] = v;
    }
  }
}

// ------------------------------------------------ chunked row pointers
// A warp owns a chunk of 128*V consecutive sorted entries; lane l holds
// entries base + 128 g + 4 l .. +3 for g < V (coalesced 512 B per group).
// Entries at or past nnz read as the last row.
template <int V>
struct RowChunk {
  int32_t r[V][4];
  int32_t prev;  // row of entry base - 1 (-1 before entry 0)
  bool full;
};

template <int V>
__device__ __forceinline__ void load_row_chunk(const int32_t* __restrict__ row, int64_t nnz,
                                               int64_t base, RowChunk<V>& c) {
  const int lane = threadIdx.x & 31;
  c.full = base + 128 * V <= nnz;
  if (c.full) {
#pragma unroll
    for (int g = 0; g < V; ++g) {
      int4 v = ld_stream(reinterpret_cast<const int4*>(row + base + 128 * g) + lane);
      c.r[g][0] = v.x; c.r[g][1] = v.y; c.r[g][2] = v.z; c.r[g][3] = v.w;
    }
  } else {
    const int32_t last = row[nnz - 1];
#pragma unroll
    for (int g = 0; g < V; ++g)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t e = base + 128 * g + 4 * lane + i;
        c.r[g][i] = e < nnz ? row[e] : last;
      }
  }
  c.prev = base == 0 ? -1 : row[base - 1];  // one broadcast load per warp
}

// Row pointers of the rows this chunk opens: ptr[q] for q in
// (prev, last row] (and up to m for the chunk holding entry nnz - 1) is the
// position of the first entry with row >= q — a lower-bound search over
// the chunk's rows staged in shared memory (s: 128*V words per warp).
// Lanes take consecutive q, so the stores are coalesced and a run of empty
// rows costs one search per 32 rows; no per-gap branches. Warp collective.
template <int kN>
__device__ __forceinline__ void row_ptr_from_smem(const int32_t* __restrict__ s, int32_t prev, int64_t nnz,
                                                  int64_t base, int32_t m, int32_t* __restrict__ ptr) {
  const int lane = threadIdx.x & 31;
  const int32_t last = s[kN - 1];
  const int32_t hi = base + kN >= nnz ? m : last;
  constexpr int kQ = 4;  // independent searches per lane per pass (ILP)
  int32_t q0 = prev + 1;
  while (q0 <= hi) {  // warp-uniform
    int pos[kQ];
#pragma unroll
    for (int j = 0; j < kQ; ++j) pos[j] = 0;
#pragma unroll
    for (int step = kN / 2; step > 0; step >>= 1)
#pragma unroll
      for (int j = 0; j < kQ; ++j)
        if (s[pos[j] + step - 1] < q0 + 32 * j + lane) pos[j] += step;
    int32_t pv0 = 0;
#pragma unroll
    for (int j = 0; j < kQ; ++j) {
      const int32_t q = q0 + 32 * j + lane;
      if (pos[j] == kN - 1 && s[kN - 1] < q) pos[j] = kN;
      const int64_t v = base + pos[j];
      const int32_t pv = (int32_t)(v < nnz ? v : nnz);
      if (j == 0) pv0 = pv;
      if (q <= hi) ptr[q] = pv;
    }
    const int pfirst = __shfl_sync(kFull, pos[0], 0), plast = __shfl_sync(kFull, pos[kQ - 1], 31);
    if (pfirst == plast && q0 + 32 * kQ - 1 < hi) {
      // the whole pass falls in one run of empty rows ending at row
      // s[pfirst]: fill the rest of the run without searching
      const int32_t end = pfirst < kN ? s[pfirst] : hi;
      for (int32_t r = q0 + 32 * kQ + lane; r <= end; r += 32) ptr[r] = pv0;
      q0 = end + 1;
    } else {
      q0 += 32 * kQ;
    }
  }
}

template <int V>
__device__ __forceinline__ void chunk_row_ptr(const RowChunk<V>& c, int64_t nnz, int64_t base,
                                              int32_t m, int32_t* __restrict__ s,
                                              int32_t* __restrict__ ptr) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int g = 0; g < V; ++g)
    reinterpret_cast<int4*>(s + 128 * g)[lane] = make_int4(c.r[g][0], c.r[g][1], c.r[g][2], c.r[g][3]);
  __syncwarp();
  row_ptr_from_smem<128 * V>(s, c.prev, nnz, base, m, ptr);
  __syncwarp();
}

}  // namespace sfg
