// SPDX-License-Identifier: Apache-2.0
//
// Counter-based sample streams.  Both kinds are pure functions of
// (seed, iteration, cube, sample, axis), so the stream never depends on which
// thread, block or GPU draws a point.
//
//  * compat: the reference's keyed SplitMix64 chain, bit for bit
//    (rng.hpp:26-68).  Pure integer work (IMAD/LOP3/SHF), off the FP64 pipe.
//  * philox: Philox4x32-10 keyed by (seed, iteration), counter
//    (cube, sample, axis pair) -- the north-star stream.  Not bitwise
//    comparable with the reference; validated statistically.
#pragma once

#include <cstdint>

#include "config.cuh"

namespace mcubes::gpu::rng {

inline constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ull;

/// SplitMix64 finalizer (rng.hpp:29-33).
MCB_HD std::uint64_t avalanche(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/// Absorb one key field (rng.hpp:37-39).
MCB_HD std::uint64_t feed(std::uint64_t h, std::uint64_t v) { return avalanche(h + kGamma + v); }

MCB_HD std::uint64_t iteration_root(std::uint64_t seed, std::uint64_t it) {  // rng.hpp:47-50
  return feed(feed(0, seed), it);
}

/// to_unit (rng.hpp:41-43): double(h >> 11) * 2^-53, computed without an
/// integer->double conversion.  With x = h >> 11 (53 bits), b = bit 52 of x and
/// D = 0.5 * (1 + low52(x) * 2^-52) (built from bits, exponent -1):
/// b = 1: x*2^-53 = D exactly;  b = 0: x*2^-53 = D - 0.5 exactly (Sterbenz).
MCB_HD double to_unit(std::uint64_t h) {
#if defined(__CUDA_ARCH__) && !defined(MCB_TOUNIT_BITS)
  // one I2F.F64.U64 (XU pipe) + DMUL: exact since h >> 11 < 2^53 (measured faster
  // than the bit-built form below, which -DMCB_TOUNIT_BITS selects)
  return __dmul_rn(__ull2double_rn(h >> 11), 0x1.0p-53);
#elif defined(__CUDA_ARCH__)
  const std::uint32_t hi = static_cast<std::uint32_t>(h >> 32);
  const std::uint32_t lo = static_cast<std::uint32_t>(h);
  const std::uint32_t dhi = 0x3FE00000u | ((hi >> 11) & 0x000FFFFFu);
  const std::uint32_t dlo = __funnelshift_r(lo, hi, 11);
  const double D = __hiloint2double(static_cast<int>(dhi), static_cast<int>(dlo));
  // b = top bit of h; subtract 0.5 when it is clear
  const std::uint32_t subhi = (static_cast<std::int32_t>(hi) >> 31) ? 0u : 0xBFE00000u;
  return __dadd_rn(D, __hiloint2double(static_cast<int>(subhi), 0));
#else
  return static_cast<double>(h >> 11) * 0x1.0p-53;
#endif
}

// ---------------------------------------------------------------- Philox4x32-10
struct U4 {
  std::uint32_t x, y, z, w;
};

MCB_HD void mulhilo(std::uint32_t a, std::uint32_t b, std::uint32_t& hi, std::uint32_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umulhi(a, b);
#else
  const std::uint64_t p = static_cast<std::uint64_t>(a) * b;
  lo = static_cast<std::uint32_t>(p);
  hi = static_cast<std::uint32_t>(p >> 32);
#endif
}

MCB_HD U4 philox4x32_10(U4 c, std::uint32_t k0, std::uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    std::uint32_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2511F53u, c.x, hi0, lo0);
    mulhilo(0xCD9E8D57u, c.z, hi1, lo1);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

/// Two uniforms in [0,1) (53 bits each) for axes (2q, 2q+1) of sample k of
/// cube t; key = iteration_root(seed, iteration).
MCB_HD void philox_pair(std::uint64_t key, std::uint64_t t, std::uint32_t k, std::uint32_t q,
                        double& r0, double& r1) {
  const U4 o = philox4x32_10(U4{static_cast<std::uint32_t>(t), static_cast<std::uint32_t>(t >> 32), k, q},
                             static_cast<std::uint32_t>(key), static_cast<std::uint32_t>(key >> 32));
  r0 = to_unit((static_cast<std::uint64_t>(o.x) << 32) | o.y);
  r1 = to_unit((static_cast<std::uint64_t>(o.z) << 32) | o.w);
}

}  // namespace mcubes::gpu::rng
