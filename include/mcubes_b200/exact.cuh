// SPDX-License-Identifier: Apache-2.0
//
// Exact, order-independent accumulation of doubles on the GPU.
//
// The reference makes every cross-cube reduction exact with a 34-limb
// fixed-point superaccumulator (exact_sum.hpp:12-27), which is what makes its
// results independent of thread count and batch size.  The B200 path keeps
// that contract with a representation that suits shared memory: kXWords
// 32-bit words per accumulator, word w holding radix-2^32 digit w of the exact
// integer sum in units of 2^-1074 (the same weight convention as ExactSum).
// A deposit is three native 32-bit shared-memory atomics whose returned old
// values carry exactly into the next word, so the final integer is the exact
// sum no matter how warps interleave: bitwise-identical results for any launch
// geometry, any cube partition across GPUs, and equal to the reference's
// ExactSum::value() after rounding.
//
// Exchange format (per-block partials, the NCCL all-reduce buffer and the
// oracle's mcubes_oracle.c): kXWords unsigned 64-bit words per accumulator,
// each an unnormalised sum of radix-2^32 digits.  Integer sums of that form are
// associative, so the cross-GPU all-reduce is exact too.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#include "config.cuh"

namespace mcubes::gpu::exact {

/// Digits of |v| * 2^1074: word index and the three radix-2^32 digits.
struct Digits {
  std::uint32_t w, d0, d1, d2;
};

MCB_HD bool split(double v, Digits& out) {
  std::uint64_t bits;
#ifdef __CUDA_ARCH__
  bits = static_cast<std::uint64_t>(__double_as_longlong(v));
#else
  std::memcpy(&bits, &v, 8);
#endif
  bits &= 0x7fffffffffffffffull;
  if (!bits) return false;
  const std::uint32_t hi = static_cast<std::uint32_t>(bits >> 32);
  const std::uint32_t lo = static_cast<std::uint32_t>(bits);
  const std::uint32_t be = hi >> 20;
  // exact_sum.hpp:106-110: implicit bit for normals, LSB weight 2^(pos-1074)
  const std::uint32_t m1 = (hi & 0x000FFFFFu) | (be ? 0x00100000u : 0u);
  const std::uint32_t pos = be ? be - 1 : 0;
  const std::uint32_t off = pos & 31u;
  out.w = pos >> 5;
#ifdef __CUDA_ARCH__
  out.d0 = lo << off;
  out.d1 = __funnelshift_l(lo, m1, off);
  out.d2 = __funnelshift_l(m1, 0u, off);
#else
  const unsigned __int128 sh = static_cast<unsigned __int128>((static_cast<std::uint64_t>(m1) << 32) | lo) << off;
  out.d0 = static_cast<std::uint32_t>(sh);
  out.d1 = static_cast<std::uint32_t>(sh >> 32);
  out.d2 = static_cast<std::uint32_t>(sh >> 64);
#endif
  return true;
}

#ifdef __CUDACC__
/// Rare tail of a deposit: a carry out of the third word ripples upward.
template <int kTag = 0>
__device__ __noinline__ void carry_up(std::uint32_t* p, std::uint32_t* end) {
  for (; p < end; ++p)
    if (atomicAdd(p, 1u) != 0xffffffffu) break;
}

/// Add pre-split digits at p = acc + dg.w (three word atomics, carries
/// travel through the returned old values).  Branch-free except for the
/// ~2^-11-probability ripple out of the top word.
__device__ __forceinline__ void add_digits(std::uint32_t* p, std::uint32_t* end, const Digits& dg) {
  const std::uint32_t o0 = atomicAdd(p, dg.d0);
  const std::uint32_t c0 = (o0 + dg.d0) < o0 ? 1u : 0u;
  const std::uint32_t t1 = dg.d1 + c0;  // wraps to 0 only if d1 == 0xffffffff and c0
  const std::uint32_t o1 = atomicAdd(p + 1, t1);
  const std::uint32_t c1 = ((t1 < c0) || ((o1 + t1) < o1)) ? 1u : 0u;
  const std::uint32_t t2 = dg.d2 + c1;  // d2 < 2^21: never wraps
  const std::uint32_t o2 = atomicAdd(p + 2, t2);
  if ((o2 + t2) < o2) carry_up(p + 3, end);
}

/// Deposit the same digits into N accumulators (one per axis) -- the
/// sampler's bin update, where every axis receives the same (f J)^2
/// (sampler.hpp:173-176).  The atomics are issued word-major across the N
/// accumulators, so a sample pays three shared-memory round trips instead of
/// 3N, and the rare ripple out of the top word is one check per sample.
/// p[j] = accumulator j + dg.w.
template <int N>
__device__ __forceinline__ void add_digits_n(std::uint32_t* const (&p)[N], std::uint32_t* end, const Digits& dg) {
  std::uint32_t c[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const std::uint32_t o = atomicAdd(p[j], dg.d0);
    c[j] = (o + dg.d0) < o ? 1u : 0u;
  }
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const std::uint32_t t = dg.d1 + c[j];  // wraps to 0 only if d1 == 0xffffffff and a carry in
    const std::uint32_t o = atomicAdd(p[j] + 1, t);
    c[j] = static_cast<std::uint32_t>(t < c[j]) | static_cast<std::uint32_t>((o + t) < o);
  }
  std::uint32_t ripple = 0;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const std::uint32_t t = dg.d2 + c[j];  // d2 < 2^21: never wraps
    const std::uint32_t o = atomicAdd(p[j] + 2, t);
    ripple |= static_cast<std::uint32_t>((o + t) < o) << j;
  }
  if (ripple) {
#pragma unroll
    for (int j = 0; j < N; ++j)
      if ((ripple >> j) & 1u) carry_up(p[j] + 3, end);
  }
}

/// Add |v| exactly into a shared-memory accumulator of kXWords u32 words.
/// Carries travel through the atomics' returned old values, so concurrent
/// deposits from any lanes/warps compose to the exact total.
__device__ __forceinline__ void add_shared(std::uint32_t* acc, double v) {
  Digits dg;
  if (!split(v, dg)) return;
  std::uint32_t* p = acc + dg.w;
  std::uint32_t o = atomicAdd(p, dg.d0);
  std::uint32_t c = (o + dg.d0) < o;
  const std::uint32_t t1 = dg.d1 + c;
  c = t1 < c;  // d1 == 0xffffffff and a carry in
  if (t1) {
    o = atomicAdd(p + 1, t1);
    c += (o + t1) < o;
  }
  const std::uint32_t t2 = dg.d2 + c;  // d2 < 2^21: never wraps
  if (t2) {
    o = atomicAdd(p + 2, t2);
    if ((o + t2) < o) {
      for (std::uint32_t k = dg.w + 3; k < static_cast<std::uint32_t>(kXWords); ++k)
        if (atomicAdd(acc + k, 1u) != 0xffffffffu) break;
    }
  }
}
#endif

/// Round the exact integer (pos - neg) * 2^-1074 to the nearest double, ties
/// to even -- ExactSum::value() (exact_sum.hpp:137-179).  Inputs are
/// unnormalised u64 digit sums (the exchange format); neg may be null.
MCB_HD double round_words(const unsigned long long* pos, const unsigned long long* neg) {
  std::uint32_t a[kXWords], b[kXWords];
  unsigned long long ca = 0, cb = 0;
  for (int i = 0; i < kXWords; ++i) {
    ca += pos[i];
    a[i] = static_cast<std::uint32_t>(ca);
    ca >>= 32;
    cb += neg ? neg[i] : 0ull;
    b[i] = static_cast<std::uint32_t>(cb);
    cb >>= 32;
  }
  int cmp = 0;
  for (int i = kXWords - 1; i >= 0 && cmp == 0; --i) cmp = a[i] < b[i] ? -1 : (a[i] > b[i] ? 1 : 0);
  if (cmp == 0) return 0.0;
  std::uint32_t* big = cmp > 0 ? a : b;
  const std::uint32_t* small = cmp > 0 ? b : a;
  std::uint32_t br = 0;
  for (int i = 0; i < kXWords; ++i) {
    const std::uint64_t d = static_cast<std::uint64_t>(big[i]) - small[i] - br;
    big[i] = static_cast<std::uint32_t>(d);
    br = static_cast<std::uint32_t>(d >> 63);
  }
  int top = -1;
  for (int i = kXWords - 1; i >= 0; --i)
    if (big[i]) {
#ifdef __CUDA_ARCH__
      top = 32 * i + 31 - __clz(big[i]);
#else
      top = 32 * i + 31 - __builtin_clz(big[i]);
#endif
      break;
    }
  auto bit = [&](int p) -> std::uint32_t { return (big[p >> 5] >> (p & 31)) & 1u; };
  double r;
  if (top <= 52) {
    const std::uint64_t v = static_cast<std::uint64_t>(big[0]) | (static_cast<std::uint64_t>(big[1]) << 32);
    r = std::ldexp(static_cast<double>(v), -1074);  // exact (sub)normal
  } else {
    // 53-bit window [top-52, top], guard bit, sticky (exact_sum.hpp:160-176)
    const int lo = top - 52;
    const int wi = lo >> 5, sh = lo & 31;
    std::uint64_t mant = static_cast<std::uint64_t>(big[wi]) >> sh;
    mant |= static_cast<std::uint64_t>(wi + 1 < kXWords ? big[wi + 1] : 0u) << (32 - sh);
    if (sh && wi + 2 < kXWords) mant |= static_cast<std::uint64_t>(big[wi + 2]) << (64 - sh);
    mant &= (1ull << 53) - 1;
    const int gpos = top - 53;
    const std::uint32_t guard = bit(gpos);
    bool sticky = false;
    if (gpos > 0) {
      const int gw = gpos >> 5, gb = gpos & 31;
      if (gb) sticky = (big[gw] & ((1u << gb) - 1u)) != 0;
      for (int k = 0; k < gw && !sticky; ++k) sticky = big[k] != 0;
    }
    int e = top - 52 - 1074;
    if (guard && (sticky || (mant & 1))) {
      if (++mant == (1ull << 53)) {
        mant >>= 1;
        ++e;
      }
    }
    r = std::ldexp(static_cast<double>(mant), e);
  }
  return cmp > 0 ? r : -r;
}

/// Host-side exact add into exchange-format words (used by host tools/tests).
inline void add_words(unsigned long long* acc, double v) {
  Digits dg;
  if (!split(v, dg)) return;
  acc[dg.w] += dg.d0;
  acc[dg.w + 1] += dg.d1;
  acc[dg.w + 2] += dg.d2;
}

}  // namespace mcubes::gpu::exact
