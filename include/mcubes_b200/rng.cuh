// SPDX-License-Identifier: Apache-2.0
//
// Counter-based sample streams.  Both kinds are pure functions of
// (seed, iteration, cube, sample, axis), so the stream never depends on which
// thread, block or GPU draws a point.
//
//  * compat: the reference's keyed SplitMix64 chain, bit for bit
//    (rng.hpp:26-68).  Pure integer work (IMAD/LOP3/SHF), off the FP64 pipe.
//  * philox: Philox4x32-10 keyed by (seed, iteration), counter (cube lo,
//    cube hi, sample, block of 4 axes) -- the north-star stream, 32-bit
//    uniforms.  Not bitwise comparable with the reference; validated
//    statistically (and bit for bit against its C twin in oracle/).
#pragma once

#include <cstdint>

#include "config.cuh"

namespace mcubes::gpu::rng {

inline constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ull;

/// z * C mod 2^64.  On the device as one IMAD.WIDE.U32 and two IMAD into its
/// high word (the compiler's own lowering spends a fourth instruction on
/// adding the cross products separately).
template <std::uint64_t C>
MCB_HD std::uint64_t mul_const(std::uint64_t z) {
#if defined(__CUDA_ARCH__)
  std::uint64_t r;
  asm("{\n\t.reg .u32 zl, zh, rl, rh;\n\t"
      "mov.b64 {zl, zh}, %1;\n\t"
      "mul.wide.u32 %0, zl, %2;\n\t"
      "mov.b64 {rl, rh}, %0;\n\t"
      "mad.lo.u32 rh, zh, %2, rh;\n\t"
      "mad.lo.u32 rh, zl, %3, rh;\n\t"
      "mov.b64 %0, {rl, rh};\n\t}"
      : "=l"(r)
      : "l"(z), "n"(static_cast<std::uint32_t>(C)), "n"(static_cast<std::uint32_t>(C >> 32)));
  return r;
#else
  return z * C;
#endif
}

/// SplitMix64 finalizer (rng.hpp:29-33).
MCB_HD std::uint64_t avalanche(std::uint64_t z) {
  z = mul_const<0xbf58476d1ce4e5b9ull>(z ^ (z >> 30));
  z = mul_const<0x94d049bb133111ebull>(z ^ (z >> 27));
  return z ^ (z >> 31);
}

/// Absorb one key field (rng.hpp:37-39).
MCB_HD std::uint64_t feed(std::uint64_t h, std::uint64_t v) { return avalanche(h + kGamma + v); }

MCB_HD std::uint64_t iteration_root(std::uint64_t seed, std::uint64_t it) {  // rng.hpp:47-50
  return feed(feed(0, seed), it);
}

/// to_unit (rng.hpp:41-43): double(h >> 11) * 2^-53 -- one I2F.F64.U64 (XU
/// pipe) and a DMUL, exact since h >> 11 < 2^53.
MCB_HD double to_unit(std::uint64_t h) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(__ull2double_rn(h >> 11), 0x1.0p-53);
#else
  return static_cast<double>(h >> 11) * 0x1.0p-53;
#endif
}

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al. 2011 (Random123).  The kernel applies it with the per-round
// keys precomputed on the host (engine.cuh set_round_keys, sampler.cuh
// philox_rk); the C twin is oracle/mcubes_oracle.c philox4x32_10.
struct U4 {
  std::uint32_t x, y, z, w;
};
inline constexpr std::uint32_t kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;
inline constexpr std::uint32_t kPhiloxW0 = 0x9E3779B9u, kPhiloxW1 = 0xBB67AE85u;

}  // namespace mcubes::gpu::rng
