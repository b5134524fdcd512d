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
// Exchange format (K1's flush target, the NCCL all-reduce buffer and the
// oracle's mcubes_oracle.c): kXWords unsigned 64-bit words per accumulator,
// each an unnormalised sum of radix-2^32 digits.  Integer sums of that form are
// associative, so the cross-GPU all-reduce is exact too.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <utility>

#include "config.cuh"

namespace mcubes::gpu::exact {

/// Digits of |v| * 2^1074: word index and the three radix-2^32 digits.
struct Digits {
  std::uint32_t w, d0, d1, d2;
  std::uint32_t be;  ///< biased exponent field (0x7ff: the addend was +-inf -- ExactSum::add throws)
};

MCB_HD bool split(double v, Digits& out) {
  std::uint64_t bits;
#ifdef __CUDA_ARCH__
  bits = static_cast<std::uint64_t>(__double_as_longlong(v));
#else
  std::memcpy(&bits, &v, 8);
#endif
  bits &= 0x7fffffffffffffffull;
  out.be = static_cast<std::uint32_t>(bits >> 52);
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
// ---- exact deposits on 32-bit shared-window addresses (atom.shared): no
// 64-bit generic-pointer arithmetic per axis; constant per-axis row offsets
// fold into the instruction's immediate.
// No "memory" clobber: the accumulators are only read after __syncthreads(),
// and atomics to distinct words commute, so the compiler may schedule other
// loads and arithmetic around them.
__device__ __forceinline__ std::uint32_t atoms_add(std::uint32_t addr, std::uint32_t v) {
  std::uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v));
  return old;
}

/// Rare tail of a deposit: a carry out of the top word ripples upward, at
/// most to the accumulator's last word (`end` = one past it; a carry past it
/// would need a sum beyond 2^1070, more than any block's deposits can reach).
/// The bound is derived in this rare path from the deposit address and word
/// index (acc_top), so the hot path keeps no extra live value.
template <int kTag = 0>
__device__ __noinline__ void carry_up_s(std::uint32_t addr, std::uint32_t end) {
  for (; addr < end; addr += 4)
    if (atoms_add(addr, 1u) != 0xffffffffu) break;
}

/// One past the last word of the accumulator whose word w sits at address a.
__device__ __forceinline__ std::uint32_t acc_top(std::uint32_t a, std::uint32_t w) { return a + 4u * (kXWords - w); }

/// Deposit the same digits into N accumulators (one per axis) -- the
/// sampler's bin update, where every axis receives the same (f J)^2
/// (sampler.hpp:173-176) -- at shared-window byte addresses a[j]
/// (= accumulator j + 4 dg.w).  The atomics are issued word-major across the N
/// accumulators, so a sample pays three shared-memory round trips instead of
/// 3N; carries travel through the returned old words (PTX add.cc/addc: IADD3
/// with predicate carry-out / IADD3.X), and the rare ripple out of the top
/// word is one check per sample.
template <int N>
__device__ __forceinline__ void add_digits_s(const std::uint32_t (&a)[N], const Digits& dg) {
  std::uint32_t t1[N], u[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const std::uint32_t o = atoms_add(a[j], dg.d0);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %2, %3;\n\taddc.cc.u32 %0, %4, 0;\n\taddc.u32 %1, %5, 0;\n\t}"
        : "=r"(t1[j]), "=r"(u[j])
        : "r"(o), "r"(dg.d0), "r"(dg.d1), "r"(dg.d2));
  }
  std::uint32_t t2[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const std::uint32_t o = atoms_add(a[j] + 4, t1[j]);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %3, 0;\n\t}" : "=r"(t2[j]) : "r"(o), "r"(t1[j]), "r"(u[j]));
  }
  std::uint32_t ripple = 0;  // bit (N-1-j) = carry out of axis j's top word
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const std::uint32_t o = atoms_add(a[j] + 8, t2[j]);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}" : "+r"(ripple) : "r"(o), "r"(t2[j]));
  }
  if (ripple) {
#pragma unroll
    for (int j = 0; j < N; ++j)
      if ((ripple >> (N - 1 - j)) & 1u) carry_up_s(a[j] + 12, acc_top(a[j], dg.w));
  }
}

// ---- Philox path bin deposits: (f J)^2 rounded to 24 significant bits.
// The bins only steer the grid adaptation, and shared 32-bit atomics are the
// K1 throughput ceiling (~7.4 lane-ops/clk/SM on B200, tools/microbench/
// atoms.cu, conflict-free or not).  With a 24-bit significand (float
// precision, 6e-8 relative per addend -- far below the Monte Carlo noise of a
// bin) a deposit spans at most two words, only one when it sits at a word
// offset <= 8, and the carry out of the upper word is rare (its digit is
// < 2^23).  The rounding is a pure function of the value and the integer sums
// stay exact, so results remain independent of launch geometry and GPU count.

/// Two digits of RN24(|v|) * 2^1074 (round-half-up on the 53-bit significand).
struct Digits2 {
  std::uint32_t w, d0, d1;
  std::uint32_t be;  ///< biased exponent after rounding (0x7ff: +-inf, or rounded up to 2^1024)
};

inline constexpr int kBinDrop = 29;  ///< significand bits dropped: 53 - 24

MCB_HD std::uint64_t round_bin_bits(std::uint64_t bits) {
  return (bits + (1ull << (kBinDrop - 1))) & ~((1ull << kBinDrop) - 1);  // carries into the exponent
}

MCB_HD bool split_r24(double v, Digits2& out) {
  std::uint64_t bits;
#ifdef __CUDA_ARCH__
  bits = static_cast<std::uint64_t>(__double_as_longlong(v));
#else
  std::memcpy(&bits, &v, 8);
#endif
  bits &= 0x7fffffffffffffffull;
  out.be = 0;
  if (!bits) return false;
  bits = round_bin_bits(bits);
  const std::uint32_t hi = static_cast<std::uint32_t>(bits >> 32);
  const std::uint32_t be = hi >> 20;
  out.be = be;
  // 24-bit significand m = (implicit:hi[19:0]:lo[31:29]), its LSB at bit pos + 29
  const std::uint32_t m = (((hi & 0x000FFFFFu) | (be ? 0x00100000u : 0u)) << 3) |
                          (static_cast<std::uint32_t>(bits) >> kBinDrop);
  const std::uint32_t pos = (be ? be - 1 : 0) + kBinDrop;
  const std::uint32_t off = pos & 31u;
  out.w = pos >> 5;
  out.d0 = m << off;
#ifdef __CUDA_ARCH__
  out.d1 = __funnelshift_l(m, 0u, off);
#else
  out.d1 = off ? m >> (32 - off) : 0u;
#endif
  return true;
}

#ifdef __CUDACC__
/// Deposit RN24 digits into N accumulators at shared-window addresses a[j]
/// (= accumulator j + 4 dg.w): two word atomics (predicating the upper one
/// off when its addend is zero measured slower), a rare ripple above.
template <int N>
__device__ __forceinline__ void add_digits2_s(const std::uint32_t (&a)[N], const Digits2& dg) {
  std::uint32_t t1[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const std::uint32_t o = atoms_add(a[j], dg.d0);
    // t1 = d1 + carry(o + d0)   (d1 < 2^23: never wraps)
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %3, 0;\n\t}" : "=r"(t1[j]) : "r"(o), "r"(dg.d0), "r"(dg.d1));
  }
  std::uint32_t ripple = 0;
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const std::uint32_t o = atoms_add(a[j] + 4, t1[j]);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}" : "+r"(ripple) : "r"(o), "r"(t1[j]));
  }
  if (ripple) {
#pragma unroll
    for (int j = 0; j < N; ++j)
      if ((ripple >> (N - 1 - j)) & 1u && atoms_add(a[j] + 8, 1u) == 0xffffffffu) carry_up_s(a[j] + 12, acc_top(a[j], dg.w));
  }
}
#endif

#ifdef __CUDACC__
/// atom.shared.add at a register address plus a compile-time byte offset
/// (folded into the instruction: [R + imm]).
template <std::uint32_t Off>
__device__ __forceinline__ std::uint32_t atoms_add_at(std::uint32_t addr, std::uint32_t v) {
  std::uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1+%2], %3;" : "=r"(old) : "r"(addr), "n"(Off), "r"(v));
  return old;
}

/// add_digits2_s for the N axes of one sample when the axis stride kRow is a
/// compile-time constant: base[j] = word-w address of bin[j] in axis 0's row;
/// axis j's row offset j*kRow rides in the atomics' immediates, so a deposit
/// costs one IMAD of address arithmetic per axis.
template <int N, std::uint32_t kRow>
__device__ __forceinline__ void add_digits2_rows(const std::uint32_t (&base)[N], const Digits2& dg) {
  std::uint32_t t1[N];
  [&]<std::size_t... J>(std::index_sequence<J...>) {
    ((void)[&] {
      const std::uint32_t o = atoms_add_at<static_cast<std::uint32_t>(J) * kRow>(base[J], dg.d0);
      asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %3, 0;\n\t}"
          : "=r"(t1[J]) : "r"(o), "r"(dg.d0), "r"(dg.d1));
    }(), ...);
  }(std::make_index_sequence<N>{});
  std::uint32_t ripple = 0;
  [&]<std::size_t... J>(std::index_sequence<J...>) {
    ((void)[&] {
      const std::uint32_t o = atoms_add_at<static_cast<std::uint32_t>(J) * kRow + 4u>(base[J], t1[J]);
      asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}" : "+r"(ripple) : "r"(o), "r"(t1[J]));
    }(), ...);
  }(std::make_index_sequence<N>{});
  if (ripple) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const std::uint32_t a = base[j] + static_cast<std::uint32_t>(j) * kRow;
      if ((ripple >> (N - 1 - j)) & 1u && atoms_add(a + 8, 1u) == 0xffffffffu) carry_up_s(a + 12, acc_top(a, dg.w));
    }
  }
}
#endif

#ifdef __CUDACC__
/// add_digits_s (three words, the exact addend) with the axis row offsets
/// j*kRow as immediates, as add_digits2_rows: the Philox stream with exact bins.
template <int N, std::uint32_t kRow>
__device__ __forceinline__ void add_digits_rows(const std::uint32_t (&base)[N], const Digits& dg) {
  std::uint32_t t1[N], u[N];
  [&]<std::size_t... J>(std::index_sequence<J...>) {
    ((void)[&] {
      const std::uint32_t o = atoms_add_at<static_cast<std::uint32_t>(J) * kRow>(base[J], dg.d0);
      asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %2, %3;\n\taddc.cc.u32 %0, %4, 0;\n\taddc.u32 %1, %5, 0;\n\t}"
          : "=r"(t1[J]), "=r"(u[J])
          : "r"(o), "r"(dg.d0), "r"(dg.d1), "r"(dg.d2));
    }(), ...);
  }(std::make_index_sequence<N>{});
  std::uint32_t t2[N];
  [&]<std::size_t... J>(std::index_sequence<J...>) {
    ((void)[&] {
      const std::uint32_t o = atoms_add_at<static_cast<std::uint32_t>(J) * kRow + 4u>(base[J], t1[J]);
      asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %3, 0;\n\t}"
          : "=r"(t2[J]) : "r"(o), "r"(t1[J]), "r"(u[J]));
    }(), ...);
  }(std::make_index_sequence<N>{});
  std::uint32_t ripple = 0;
  [&]<std::size_t... J>(std::index_sequence<J...>) {
    ((void)[&] {
      const std::uint32_t o = atoms_add_at<static_cast<std::uint32_t>(J) * kRow + 8u>(base[J], t2[J]);
      asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}" : "+r"(ripple) : "r"(o), "r"(t2[J]));
    }(), ...);
  }(std::make_index_sequence<N>{});
  if (ripple) {
#pragma unroll
    for (int j = 0; j < N; ++j)
      if ((ripple >> (N - 1 - j)) & 1u) {
        const std::uint32_t a = base[j] + static_cast<std::uint32_t>(j) * kRow;
        carry_up_s(a + 12, acc_top(a, dg.w));
      }
  }
}
#endif

/// Two independent exact adds (the per-cube estimate and variance) at
/// shared-window addresses a_s / b_s (accumulator bases), issued interleaved
/// so their atomic round trips overlap.
__device__ __forceinline__ void add_shared2_s(std::uint32_t a_s, double a, std::uint32_t b_s, double b) {
  Digits da, db;
  const bool ha = split(a, da), hb = split(b, db);
  if (ha && hb) {
    const std::uint32_t pa = a_s + 4u * da.w, pb = b_s + 4u * db.w;
    // the two accumulators receive different digits: interleave by hand
    std::uint32_t ta, ua, tb, ub;
    std::uint32_t o = atoms_add(pa, da.d0);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %2, %3;\n\taddc.cc.u32 %0, %4, 0;\n\taddc.u32 %1, %5, 0;\n\t}"
        : "=r"(ta), "=r"(ua) : "r"(o), "r"(da.d0), "r"(da.d1), "r"(da.d2));
    o = atoms_add(pb, db.d0);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %2, %3;\n\taddc.cc.u32 %0, %4, 0;\n\taddc.u32 %1, %5, 0;\n\t}"
        : "=r"(tb), "=r"(ub) : "r"(o), "r"(db.d0), "r"(db.d1), "r"(db.d2));
    o = atoms_add(pa + 4, ta);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %3, 0;\n\t}" : "=r"(ta) : "r"(o), "r"(ta), "r"(ua));
    o = atoms_add(pb + 4, tb);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %3, 0;\n\t}" : "=r"(tb) : "r"(o), "r"(tb), "r"(ub));
    std::uint32_t ra = 0, rb = 0;
    o = atoms_add(pa + 8, ta);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, 0, 0;\n\t}" : "=r"(ra) : "r"(o), "r"(ta));
    o = atoms_add(pb + 8, tb);
    asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, 0, 0;\n\t}" : "=r"(rb) : "r"(o), "r"(tb));
    if (ra | rb) {
      if (ra) carry_up_s(pa + 12, acc_top(pa, da.w));
      if (rb) carry_up_s(pb + 12, acc_top(pb, db.w));
    }
  } else if (ha) {
    const std::uint32_t pa[1] = {a_s + 4u * da.w};
    add_digits_s<1>(pa, da);
  } else if (hb) {
    const std::uint32_t pb[1] = {b_s + 4u * db.w};
    add_digits_s<1>(pb, db);
  }
}

#endif

/// Round the exact integer (pos - neg) * 2^-1074 to the nearest double, ties
/// to even -- ExactSum::value() (exact_sum.hpp:65-109).  Inputs are
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
    // 53-bit window [top-52, top], guard bit, sticky (exact_sum.hpp:91-104)
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

#ifdef __CUDACC__
namespace warpx {
// Warp-cooperative exact rounding.  Lane l holds words w = l + 32k, k = 0..2
// (kXWords = 67 <= 96).  Carries/borrows move up one word per step through
// shuffles; a step clears all carries unless a run of all-ones words is met,
// so the loops finish in ~2-3 steps.

__device__ __forceinline__ unsigned long long up1(unsigned long long x0, unsigned long long x1,
                                                  unsigned long long x2, int k, int lane) {
  // value of register k from the previous word (w - 1)
  const unsigned long long src = k == 0 ? x0 : (k == 1 ? x1 : x2);
  const unsigned long long prev_lane = __shfl_up_sync(0xffffffffu, src, 1);
  const unsigned long long wrap = __shfl_sync(0xffffffffu, k == 0 ? 0ull : (k == 1 ? x0 : x1), 31);
  return lane == 0 ? (k == 0 ? 0ull : wrap) : prev_lane;
}

/// Normalise unsigned digit sums into radix-2^32 digits (v[k] < 2^32).
__device__ __forceinline__ void normalise(unsigned long long (&v)[3], int lane) {
  while (true) {
    unsigned long long c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      c[k] = v[k] >> 32;
      v[k] &= 0xffffffffull;
    }
    const bool any = (c[0] | c[1] | c[2]) != 0;
    if (!__any_sync(0xffffffffu, any)) return;
    unsigned long long in[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) in[k] = up1(c[0], c[1], c[2], k, lane);
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] += in[k];
  }
}

/// a -= b for normalised digits with a >= b.
__device__ __forceinline__ void subtract(unsigned long long (&a)[3], const unsigned long long (&b)[3], int lane) {
  long long d[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) d[k] = static_cast<long long>(a[k]) - static_cast<long long>(b[k]);
  while (true) {
    unsigned long long br[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      br[k] = d[k] < 0 ? 1ull : 0ull;
      d[k] += static_cast<long long>(br[k]) << 32;
    }
    if (!__any_sync(0xffffffffu, (br[0] | br[1] | br[2]) != 0)) break;
    unsigned long long in[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) in[k] = up1(br[0], br[1], br[2], k, lane);
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] -= static_cast<long long>(in[k]);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) a[k] = static_cast<unsigned long long>(d[k]);
}

/// Highest word index whose predicate holds (-1 if none); uniform across the warp.
__device__ __forceinline__ int top_word(bool p0, bool p1, bool p2) {
  const unsigned m2 = __ballot_sync(0xffffffffu, p2), m1 = __ballot_sync(0xffffffffu, p1),
                 m0 = __ballot_sync(0xffffffffu, p0);
  if (m2) return 64 + 31 - __clz(m2);
  if (m1) return 32 + 31 - __clz(m1);
  if (m0) return 31 - __clz(m0);
  return -1;
}

/// Digit w (uniform) broadcast to all lanes.
__device__ __forceinline__ unsigned long long digit(const unsigned long long (&v)[3], int w) {
  if (w < 0) return 0ull;
  const int k = w >> 5;
  const unsigned long long x = k == 0 ? v[0] : (k == 1 ? v[1] : v[2]);
  return __shfl_sync(0xffffffffu, x, w & 31);
}
}  // namespace warpx

/// Warp-cooperative form of round_words: RN-even of (pos - neg) * 2^-1074
/// (ExactSum::value(), exact_sum.hpp:65-109).  All 32 lanes call it; every
/// lane returns the result.
__device__ __forceinline__ double warp_round_words(const unsigned long long* pos, const unsigned long long* neg) {
  const int lane = threadIdx.x & 31;
  unsigned long long a[3], b[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int w = lane + 32 * k;
    a[k] = w < kXWords ? pos[w] : 0ull;
    b[k] = (w < kXWords && neg) ? neg[w] : 0ull;
  }
  warpx::normalise(a, lane);
  bool negative = false;
  if (neg) {
    warpx::normalise(b, lane);
    const int dw = warpx::top_word(a[0] != b[0], a[1] != b[1], a[2] != b[2]);
    if (dw < 0) return 0.0;
    if (warpx::digit(a, dw) < warpx::digit(b, dw)) {
      negative = true;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const unsigned long long t = a[k];
        a[k] = b[k];
        b[k] = t;
      }
    }
    warpx::subtract(a, b, lane);
  }
  const int tw = warpx::top_word(a[0] != 0, a[1] != 0, a[2] != 0);
  if (tw < 0) return 0.0;
  const unsigned long long d2 = warpx::digit(a, tw), d1 = warpx::digit(a, tw - 1), d0 = warpx::digit(a, tw - 2);
  // any nonzero digit below the 3-word window
  const int lw = tw - 3;
  const unsigned below = __ballot_sync(0xffffffffu, (lane <= lw && a[0] != 0) || (lane + 32 <= lw && a[1] != 0) ||
                                                         (lane + 64 <= lw && a[2] != 0));
  double r;
  const int top = 32 * tw + 31 - __clz(static_cast<unsigned>(d2));
  if (top <= 52) {
    const unsigned long long v = warpx::digit(a, 0) | (warpx::digit(a, 1) << 32);
    r = ldexp(static_cast<double>(v), -1074);
  } else {
    // 96-bit window X = d2:d1:d0 covering bit positions [32(tw-2), 32(tw+1))
    const int base = 32 * (tw - 2);
    const int lo = top - 52 - base;  // window-relative position of the mantissa LSB (may be < 0 if tw < 2)
    const unsigned __int128 X = (static_cast<unsigned __int128>(d2) << 64) | (static_cast<unsigned __int128>(d1) << 32) | d0;
    unsigned long long mant;
    bool guard, sticky = below != 0;
    if (lo >= 1) {
      mant = static_cast<unsigned long long>(X >> lo) & ((1ull << 53) - 1);
      guard = ((X >> (lo - 1)) & 1) != 0;
      if (lo >= 2) sticky = sticky || (X & ((static_cast<unsigned __int128>(1) << (lo - 1)) - 1)) != 0;
    } else {  // only when the value is tiny (tw < 2): the whole number is in the window
      mant = static_cast<unsigned long long>(X >> (lo > 0 ? lo : 0));
      guard = false;
    }
    int e = top - 52 - 1074;
    if (guard && (sticky || (mant & 1))) {
      if (++mant == (1ull << 53)) {
        mant >>= 1;
        ++e;
      }
    }
    r = ldexp(static_cast<double>(mant), e);
  }
  return negative ? -r : r;
}
#endif

/// Host-side exact add into exchange-format words (used by host tools/tests).
inline void add_words(unsigned long long* acc, double v) {
  Digits dg;
  if (!split(v, dg)) return;
  acc[dg.w] += dg.d0;
  acc[dg.w + 1] += dg.d1;
  acc[dg.w + 2] += dg.d2;
}

}  // namespace mcubes::gpu::exact
