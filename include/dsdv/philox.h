/* Counter-based uniform stream shared bit-for-bit by the sm_100a kernels, the
 * C-ABI host helpers and the CPU oracle (plain C, C++ and CUDA all include it).
 *
 * Replaces the sequential std::mt19937_64 stream of the reference
 * (proj/include/dsd/rng.hpp:34-57) with Philox4x32-10 so that every
 * (sequence, window, slot) draw is addressable without a shared cursor.
 * The 64 -> 53 bit mantissa mapping is the reference's (rng.hpp:38-40):
 *     u = (x >> 11) * 2^-53,   u in [0, 1).
 *
 * Counter layout: c0 = slot, c1 = sequence index, c2/c3 = window (lo/hi);
 * key = seed (lo/hi).
 *
 * Slot map (reference consumption order, verifier.cpp:219,236,246,254):
 *   draft draw at position j        -> slot j                 (j < gamma)
 *   accept test at position j       -> slot gamma + j
 *   extra (residual or bonus) draw  -> slot gamma + (#accept draws)
 *                                    = gamma + k + 1 after a rejection at k,
 *                                      2*gamma after a full window.
 * A stream that hands out consecutive slots therefore replays exactly the
 * draws an unchanged verify_round would pull from a UniformStream.
 */
#ifndef DSDV_PHILOX_H_
#define DSDV_PHILOX_H_

#include <stdint.h>

#if defined(__CUDACC__)
#define DSDV_HD __host__ __device__ __forceinline__
#else
#define DSDV_HD static inline
#endif

#define DSDV_PHILOX_M0 0xD2511F53u
#define DSDV_PHILOX_M1 0xCD9E8D57u
#define DSDV_PHILOX_W0 0x9E3779B9u
#define DSDV_PHILOX_W1 0xBB67AE85u

typedef struct {
  uint32_t v[4];
} dsdv_philox_out;

DSDV_HD uint32_t dsdv_mulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * (uint64_t)b) >> 32);
#endif
}

/* Philox4x32 with 10 rounds (Salmon et al., SC'11). */
DSDV_HD dsdv_philox_out dsdv_philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                           uint32_t c3, uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = dsdv_mulhi32(DSDV_PHILOX_M0, c0);
    const uint32_t lo0 = DSDV_PHILOX_M0 * c0;
    const uint32_t hi1 = dsdv_mulhi32(DSDV_PHILOX_M1, c2);
    const uint32_t lo1 = DSDV_PHILOX_M1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += DSDV_PHILOX_W0;
    k1 += DSDV_PHILOX_W1;
  }
  dsdv_philox_out o;
  o.v[0] = c0;
  o.v[1] = c1;
  o.v[2] = c2;
  o.v[3] = c3;
  return o;
}

/* 64 random bits for (seed, window, sequence, slot). */
DSDV_HD uint64_t dsdv_philox_bits(uint64_t seed, uint64_t window, uint32_t sequence,
                                  uint32_t slot) {
  const dsdv_philox_out o =
      dsdv_philox4x32_10(slot, sequence, (uint32_t)window, (uint32_t)(window >> 32),
                         (uint32_t)seed, (uint32_t)(seed >> 32));
  return ((uint64_t)o.v[1] << 32) | (uint64_t)o.v[0];
}

/* Uniform in [0, 1) with the reference's 53-bit mapping (rng.hpp:39). */
DSDV_HD double dsdv_philox_uniform(uint64_t seed, uint64_t window, uint32_t sequence,
                                   uint32_t slot) {
  return (double)(dsdv_philox_bits(seed, window, sequence, slot) >> 11) *
         1.1102230246251565404236316680908203125e-16; /* 2^-53 */
}

#endif /* DSDV_PHILOX_H_ */
