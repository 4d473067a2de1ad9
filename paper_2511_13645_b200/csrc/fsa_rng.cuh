// fsa_rng.cuh — the per-seed stream contract of FuseSampleAgg, host+device.
//
// Bit-exact restatement of the reference's determinism contract:
//   * stream derivation  z = base + GOLDEN*(1 + root*ROOT + hop*HOP + index*INDEX)  (mod 2^64)
//     then the splitmix64 finaliser, 0 -> GOLDEN escape
//       reference: pkg/src/fsa/rng.py:95-104 (derive_stream), rng.py:38-43 (splitmix64),
//                  rng.py:27-28,64-68 (zero escape), kernels.py:26-49 (_splitmix/_derive)
//   * generator          xorshift64 with shift triple (13, 7, 17); the returned value is the
//                        new state      rng.py:46-52, kernels.py:33-38
//   * reduction          plain `state % (i+1)`   rng.py:75-83, kernels.py:63-65
//
// On top of the contract this header carries the two facts that make the sampler parallel
// on a GPU (both exact, both covered by golden tests):
//   (a) xorshift64 is linear over GF(2)^64, so T^n can be applied with precomputed nibble
//       tables for T^(2^e)  -> any lane can jump to any draw of any chain;
//   (b) `x % m` for m < 2^30 is computed exactly with a Barrett reciprocal R = floor(2^64/m)
//       using four 32-bit multiplies and two conditional subtractions.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define FSA_HD __host__ __device__ __forceinline__
#else
#define FSA_HD inline
#endif

namespace fsa {

constexpr uint64_t GOLDEN     = 0x9E3779B97F4A7C15ull;
constexpr uint64_t MIX1       = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t MIX2       = 0x94D049BB133111EBull;
constexpr uint64_t ROOT_MULT  = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t HOP_MULT   = 0x94D049BB133111EBull;
constexpr uint64_t INDEX_MULT = 0xD6E8FEB86659FD93ull;

FSA_HD uint64_t splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
}

FSA_HD uint64_t xorshift64(uint64_t x) {
  x ^= x << 13;
  x ^= x >> 7;
  x ^= x << 17;
  return x;
}

// Inverse of xorshift64 (used only by host-side table checks).
FSA_HD uint64_t xorshift64_inv(uint64_t x) {
  x ^= x << 17; x ^= x << 34;
  x ^= x >> 7;  x ^= x >> 14; x ^= x >> 28; x ^= x >> 56;
  x ^= x << 13; x ^= x << 26; x ^= x << 52;
  return x;
}

// derive_stream(base, root, hop, index).state  — rng.py:95-104 / kernels.py:41-49.
// `root` is the position of the seed in the (global) batch, not the node id.
FSA_HD uint64_t derive_state(uint64_t base_seed, uint64_t root, uint64_t hop, uint64_t index) {
  uint64_t z = base_seed + GOLDEN * (1ull + root * ROOT_MULT + hop * HOP_MULT + index * INDEX_MULT);
  uint64_t s = splitmix64(z);
  return s == 0 ? GOLDEN : s;
}

// R = floor(2^64 / m) for 2 <= m < 2^32.
FSA_HD uint64_t barrett_recip(uint32_t m) {
  uint64_t r = 0xFFFFFFFFFFFFFFFFull / m;
  if ((m & (m - 1u)) == 0u) r += 1;  // m | 2^64 only for powers of two
  return r;
}

#if defined(__CUDACC__)
// x mod m, exact for 2 <= m <= 2^30, R = barrett_recip(m).
// q~ = floor((x*R - xl*Rl) / 2^64) satisfies q* - 2 <= q~ <= q*, so r~ = x - q~*m lies in
// [0, 3m) < 2^32 and is recovered from the low 32 bits alone; two conditional subtractions
// (unsigned min with the wrapped difference) give r exactly.
__device__ __forceinline__ uint32_t mod_barrett(uint64_t x, uint64_t R, uint32_t m) {
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
  const uint32_t Rl = (uint32_t)R, Rh = (uint32_t)(R >> 32);
  const uint64_t s = (uint64_t)xh * Rl + (uint64_t)xl * Rh;  // mod 2^64 on purpose
  const uint32_t ql = xh * Rh + (uint32_t)(s >> 32);
  uint32_t r = xl - ql * m;
  r = min(r, r - m);
  r = min(r, r - m);
  return r;
}
#endif

}  // namespace fsa
