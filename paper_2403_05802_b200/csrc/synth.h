/* Deterministic synthetic-matrix generators shared by the CUDA product
 * library (device) and the CPU oracle (host). Integer-only arithmetic, so the
 * host and the device produce bit-identical coordinates and values.
 *
 * These are bench/test infrastructure (SURVEY.md §8d "synthetic input"), not
 * part of the reference algorithm.
 *
 * Values are drawn as +-(0.5 + k*2^-23), k < 2^23: exactly representable in
 * fp32, never zero (SURVEY.md §8c parity trap 1), so the f64 oracle sees the
 * same numbers the fp32 GPU path sees.
 */
#ifndef SFG_SYNTH_H
#define SFG_SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define SFG_HD __host__ __device__ __forceinline__
#else
#define SFG_HD static inline
#endif

/* splitmix64 finaliser: a full-avalanche 64-bit mix. */
SFG_HD uint64_t sfg_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Counter-based hash of (seed, a, b). */
SFG_HD uint64_t sfg_hash3(uint64_t seed, uint64_t a, uint64_t b) {
  return sfg_mix64(sfg_mix64(seed ^ 0x5851F42D4C957F2Dull) ^ sfg_mix64(a * 0x2545F4914F6CDD1Dull + b));
}

/* Uniform integer in [0, n) from the high 32 bits (n < 2^32). */
SFG_HD uint32_t sfg_below(uint64_t h, uint32_t n) {
  return (uint32_t)(((h >> 32) * (uint64_t)n) >> 32);
}

/* Matrix value +-U[0.5, 1.5) on a 2^-23 grid; exact in fp32. */
SFG_HD float sfg_value(uint64_t h) {
  uint32_t k = (uint32_t)(h >> 41);             /* 23 bits */
  float v = 0.5f + (float)k * (1.0f / 8388608.0f);
  return (h & 1ull) ? -v : v;
}

/* Dense-operand value U(0, 1] on a 2^-24 grid; exact in fp32. */
SFG_HD float sfg_dense_value(uint64_t h) {
  uint32_t k = (uint32_t)(h >> 40);             /* 24 bits */
  return (float)(k + 1u) * (1.0f / 16777216.0f);
}

/* Config 1: exactly `per_row` distinct columns in row r, uniform without
 * replacement, returned sorted ascending in cols[0..per_row). */
SFG_HD void sfg_uniform_row(uint64_t seed, uint32_t r, uint32_t ncols, int per_row,
                            uint32_t* cols) {
  int have = 0;
  for (uint32_t t = 0; have < per_row; ++t) {
    uint32_t c = sfg_below(sfg_hash3(seed, r, t), ncols);
    int dup = 0;
    for (int i = 0; i < have; ++i) dup |= (cols[i] == c);
    if (!dup) {
      int i = have++;
      while (i > 0 && cols[i - 1] > c) { cols[i] = cols[i - 1]; --i; }
      cols[i] = c;
    }
  }
}

/* R-MAT quadrant thresholds for (a,b,c,d) = (0.57, 0.19, 0.19, 0.05) on a
 * 2^32 grid: floor(0.57*2^32), +floor(0.19*2^32), +floor(0.19*2^32). */
#define SFG_RMAT_A 2448131358u
#define SFG_RMAT_AB 3264175144u
#define SFG_RMAT_ABC 4080218930u

/* R-MAT edge e of a 2^scale x 2^scale graph, no vertex permutation. Packed
 * key = row << 32 | col, so sorting keys sorts by (row, col). */
SFG_HD uint64_t sfg_rmat_edge(uint64_t seed, uint64_t e, int scale) {
  uint32_t r = 0, c = 0;
  for (int l = 0; l < scale; ++l) {
    uint32_t u = (uint32_t)(sfg_hash3(seed, e, (uint64_t)l) >> 32);
    uint32_t bit = 1u << (scale - 1 - l);
    if (u >= SFG_RMAT_A) {
      if (u < SFG_RMAT_AB) c |= bit;
      else if (u < SFG_RMAT_ABC) r |= bit;
      else { r |= bit; c |= bit; }
    }
  }
  return ((uint64_t)r << 32) | c;
}

/* Config 3: coordinate k i.i.d. uniform over an M x N grid. */
SFG_HD uint64_t sfg_uniform_coord(uint64_t seed, uint64_t k, uint32_t m, uint32_t n) {
  uint64_t h1 = sfg_hash3(seed, k, 0x11);
  uint64_t h2 = sfg_hash3(seed, k, 0x22);
  return ((uint64_t)sfg_below(h1, m) << 32) | sfg_below(h2, n);
}

/* Value of the entry at (r, c): a function of the coordinate, so a dedup
 * that keeps any copy keeps the same value. */
SFG_HD float sfg_coord_value(uint64_t seed, uint32_t r, uint32_t c) {
  return sfg_value(sfg_hash3(seed ^ 0xA5A5A5A5ull, r, c));
}

#endif /* SFG_SYNTH_H */

/* Config 4: block (br, bc) of a block-sparse matrix is present with
 * probability p = thresh / 2^32; values are coordinate-hashed like the other
 * generators, so the block-sparse matrix equals its COO expansion. */
#ifndef SFG_SYNTH_BLOCKS
#define SFG_SYNTH_BLOCKS
SFG_HD int sfg_block_present(uint64_t seed, uint32_t br, uint32_t bc, uint32_t thresh) {
  return (uint32_t)(sfg_hash3(seed ^ 0xB10CB10Cull, br, bc) >> 32) < thresh;
}
#endif
