// SPDX-License-Identifier: Apache-2.0
//
// K1-WS: the Philox-path sampling kernel with warp-specialised exact bin
// deposits (adjusting iterations, all axes).
//
//
// ARCHIVED EXPERIMENT (not built): measured slower than the single-role K1
// because the shared-memory atomic unit, not latency, bounds the deposits
// (DESIGN.md section 4).  Compile with -I include/mcubes_b200.
// In K1 every warp alternates a compute phase (Philox, transform, integrand)
// and a deposit phase whose three dependent shared-memory atomic rounds per
// axis (carries travel through the returned old words, exact.cuh) leave the
// warp waiting.  Here the block is split:
//
//  * kWsProducers PRODUCER warps walk the cubes exactly as K1 does, deposit
//    the per-cube estimate/variance themselves (once per cube), and for every
//    sample hand the split (f J)^2 -- word base address and three radix-2^32
//    digits -- plus the D bin indices to their consumer through a
//    shared-memory ring of kWsSlots warp-wide slots (mbarrier full/empty
//    handshakes, one arrival per lane);
//  * kWsConsumers CONSUMER warps drain the rings of kWsProducers/kWsConsumers
//    producers each and perform the exact deposits for all of those records at
//    once, so each atomic round has NQ*D independent atomics in flight.
//
// The deposited integers are the same as K1's (exact sums), so results are
// bitwise identical to K1-philox for any launch geometry.
#pragma once

#include <cstdint>

#include "config.cuh"
#include "exact.cuh"
#include "sampler.cuh"

namespace mcubes::gpu {

#ifndef MCB_WS_PRODUCERS
#define MCB_WS_PRODUCERS 24
#endif
#ifndef MCB_WS_CONSUMERS
#define MCB_WS_CONSUMERS 8
#endif
inline constexpr int kWsProducers = MCB_WS_PRODUCERS;
inline constexpr int kWsConsumers = MCB_WS_CONSUMERS;
inline constexpr int kWsSlots = 4;  ///< ring depth per producer warp
inline constexpr int kWsThreads = 32 * (kWsProducers + kWsConsumers);
static_assert(kWsProducers % kWsConsumers == 0, "each consumer serves the same number of producers");

/// Record sentinels in the word-base field (real bases are > 1: the grid
/// table precedes the accumulators in shared memory).
inline constexpr std::uint32_t kWsNone = 0;  ///< sample deposits nothing ((f J)^2 == 0 or non-finite)
inline constexpr std::uint32_t kWsEnd = 1;   ///< producer finished

/// Dynamic shared memory of K1-WS.
inline std::size_t sample_ws_smem_bytes(int D, std::uint32_t nb) {
  const std::size_t base = sample_smem_bytes(D, nb, static_cast<std::uint32_t>(D));
  const std::size_t ring = static_cast<std::size_t>(kWsProducers) * kWsSlots * 32 * (16 + 8);
  const std::size_t bars = static_cast<std::size_t>(kWsProducers) * kWsSlots * 2 * 8;
  return base + ring + bars;
}

namespace ws {
__device__ __forceinline__ void bar_init(std::uint32_t addr, std::uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(std::uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void bar_wait(std::uint32_t addr, std::uint32_t parity) {
  std::uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
/// Predicated shared atomic add (no-op, old = 0 when !on).
__device__ __forceinline__ std::uint32_t atoms_add_if(std::uint32_t addr, std::uint32_t v, std::uint32_t on) {
  std::uint32_t old = 0;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q atom.shared.add.u32 %0, [%1], %2;\n\t}"
               : "+r"(old)
               : "r"(addr), "r"(v), "r"(on));
  return old;
}
}  // namespace ws

template <class F, int D, int NB>
__global__ void __launch_bounds__(kWsThreads, 1) vsample_ws_kernel(const SampleArgs a, const F f) {
  static_assert(D >= 2 && D <= 8, "bin indices are packed as 8 bytes");
  if (a.stop && *a.stop) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const std::uint32_t nb = NB ? static_cast<std::uint32_t>(NB) : a.nb;
  double2* LW = reinterpret_cast<double2*>(smem);
  double* rcp = reinterpret_cast<double*>(LW + D * nb);
  std::uint32_t* acc = reinterpret_cast<std::uint32_t*>(rcp + kRcpSmem);
  const int nacc = block_accs(static_cast<std::uint32_t>(D), nb);
  unsigned char* after = smem + sample_smem_bytes(D, nb, static_cast<std::uint32_t>(D));
  uint4* ring4 = reinterpret_cast<uint4*>(after);                                  // [P][S][32]
  uint2* ringb = reinterpret_cast<uint2*>(ring4 + kWsProducers * kWsSlots * 32);    // [P][S][32]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(ringb + kWsProducers * kWsSlots * 32);
  const std::uint32_t bars_s = static_cast<std::uint32_t>(__cvta_generic_to_shared(bars));
  auto full_bar = [&](int q, int s) { return bars_s + 8u * static_cast<std::uint32_t>(q * kWsSlots + s); };
  auto empty_bar = [&](int q, int s) {
    return bars_s + 8u * static_cast<std::uint32_t>(kWsProducers * kWsSlots + q * kWsSlots + s);
  };
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;

  {  // zero the accumulators, stage the grid and the Welford reciprocals, init the barriers
    const int nwords = nacc * kXWords;
    for (int i = tid; i < nwords; i += nt) acc[i] = 0u;
    stage_grid_fast<D>(LW, a);
    for (int i = tid; i < kRcpSmem; i += nt) rcp[i] = i ? 1.0 / static_cast<double>(i) : 0.0;
    if (tid == 0)
      for (int i = 0; i < 2 * kWsProducers * kWsSlots; ++i) ws::bar_init(bars_s + 8u * i, 32);
  }
  __syncthreads();

  std::uint32_t* bins = acc + kScalarAccs * kLaneCopies * kXWords;
  const std::uint32_t bins_s = static_cast<std::uint32_t>(__cvta_generic_to_shared(bins));
  const std::uint32_t end_s = static_cast<std::uint32_t>(__cvta_generic_to_shared(acc + nacc * kXWords));
  constexpr std::uint32_t kCell = 4u * kXWords;

  if (warp < kWsProducers) {
    // ------------------------------------------------------------ producer
    std::uint32_t* est_pos = acc + (0 * kLaneCopies + lane) * kXWords;
    std::uint32_t* est_neg = acc + (1 * kLaneCopies + lane) * kXWords;
    std::uint32_t* var_acc = acc + (2 * kLaneCopies + lane) * kXWords;
    const std::uint64_t T = static_cast<std::uint64_t>(gridDim.x) * (32 * kWsProducers);
    CubeWalk<D> cw;
    bool active = cw.init(a, static_cast<std::uint64_t>(blockIdx.x) * (32 * kWsProducers) + warp * 32 + lane);
    std::uint32_t seq = 0;
    uint4* my4 = ring4 + warp * kWsSlots * 32 + lane;
    uint2* myb = ringb + warp * kWsSlots * 32 + lane;
    auto enqueue = [&](std::uint32_t wb, const exact::Digits& dg, const std::uint32_t (&bin)[D]) {
      const int s = static_cast<int>(seq % kWsSlots);
      const std::uint32_t k = seq / kWsSlots;
      if (k > 0) ws::bar_wait(empty_bar(warp, s), (k - 1) & 1u);
      std::uint32_t b0 = 0, b1 = 0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (j < 4) b0 |= bin[j] << (8 * j);
        else b1 |= bin[j] << (8 * (j - 4));
      }
      my4[s * 32] = make_uint4(wb, dg.d0, dg.d1, dg.d2);
      myb[s * 32] = make_uint2(b0, b1);
      ws::bar_arrive(full_bar(warp, s));
      ++seq;
    };
    const std::uint32_t p = static_cast<std::uint32_t>(a.p);
    while (__any_sync(0xffffffffu, active)) {
      const std::uint64_t t = cw.t;
      double sum = 0.0, mean = 0.0, m2 = 0.0;
      for (std::uint32_t k = 0; k < p; ++k) {
        double x[D];
        std::uint32_t bin[D];
        double fx = 0.0, fj = 0.0;
        exact::Digits dg{0, 0, 0, 0};
        std::uint32_t wb = kWsNone;
        if (active) {
          fj = sample_point_fast<F, D, NB>(a, f, LW, cw.dig, t, k, x, bin, fx);
          if (!isfinite(fj)) {
            atomicMin(a.err_key, static_cast<unsigned long long>(t * a.p + k));
          } else {
            sum = __dadd_rn(sum, fj);
            const std::uint32_t nk = k + 1;
            const double y = nk < static_cast<std::uint32_t>(kRcpSmem) ? rcp[nk] : __drcp_rn(static_cast<double>(nk));
            const double dd = __dsub_rn(fj, mean);
            mean = __fma_rn(dd, y, mean);
            m2 = __fma_rn(dd, __dsub_rn(fj, mean), m2);
            if (exact::split(__dmul_rn(fj, fj), dg)) wb = bins_s + 4u * dg.w;
          }
        }
        if (wb == kWsNone) {
#pragma unroll
          for (int j = 0; j < D; ++j) bin[j] = 0;
        }
        enqueue(wb, dg, bin);
      }
      if (active) {
        sum = __dmul_rn(sum, a.scale);
        double var = __dmul_rn(m2, a.rcp_pp1);
        if (!(var > 0.0)) var = 0.0;
        std::uint32_t* const est_acc = sum < 0.0 ? est_neg : est_pos;
        exact::add_shared2(est_acc, sum, var_acc, var, est_acc + kXWords, var_acc + kXWords);
        bool all_axes;
        active = cw.next(a, T, all_axes);
      }
    }
    const std::uint32_t bz[D] = {};
    enqueue(kWsEnd, exact::Digits{0, 0, 0, 0}, bz);
  } else {
    // ------------------------------------------------------------ consumer
    constexpr int NQ = kWsProducers / kWsConsumers;
    const int c = warp - kWsProducers;
    std::uint32_t seq = 0;  // all producers of a consumer advance in lock step
    std::uint32_t live = (1u << NQ) - 1u;
    while (live) {
      const int s = static_cast<int>(seq % kWsSlots);
      const std::uint32_t par = (seq / kWsSlots) & 1u;
      uint4 r[NQ];
      uint2 rb[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        r[i] = make_uint4(kWsNone, 0, 0, 0);
        rb[i] = make_uint2(0, 0);
        if ((live >> i) & 1u) {
          const int q = c + i * kWsConsumers;
          ws::bar_wait(full_bar(q, s), par);
          r[i] = ring4[(q * kWsSlots + s) * 32 + lane];
          rb[i] = ringb[(q * kWsSlots + s) * 32 + lane];
          ws::bar_arrive(empty_bar(q, s));
          if (r[i].x == kWsEnd) {  // warp-uniform: every lane of the producer wrote it
            live &= ~(1u << i);
            r[i].x = kWsNone;
          }
        }
      }
      ++seq;
      // exact deposits of NQ records x D axes, word-major (exact.cuh add_digits_s)
      std::uint32_t ad[NQ][D], on[NQ], t1[NQ][D], u[NQ][D];
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        on[i] = r[i].x > kWsEnd ? 1u : 0u;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const std::uint32_t b = ((j < 4 ? rb[i].x : rb[i].y) >> (8 * (j & 3))) & 0xffu;
          ad[i][j] = r[i].x + b * kCell + static_cast<std::uint32_t>(j) * nb * kCell;
        }
      }
#pragma unroll
      for (int i = 0; i < NQ; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const std::uint32_t o = ws::atoms_add_if(ad[i][j], r[i].y, on[i]);
          asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %2, %3;\n\taddc.cc.u32 %0, %4, 0;\n\taddc.u32 %1, %5, 0;\n\t}"
              : "=r"(t1[i][j]), "=r"(u[i][j])
              : "r"(o), "r"(r[i].y), "r"(r[i].z), "r"(r[i].w));
        }
#pragma unroll
      for (int i = 0; i < NQ; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const std::uint32_t o = ws::atoms_add_if(ad[i][j] + 4, t1[i][j], on[i]);
          asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %3, 0;\n\t}"
              : "=r"(t1[i][j])
              : "r"(o), "r"(t1[i][j]), "r"(u[i][j]));
        }
      std::uint32_t ripple[NQ];
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        ripple[i] = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const std::uint32_t o = ws::atoms_add_if(ad[i][j] + 8, t1[i][j], on[i]);
          asm("{\n\t.reg .u32 z;\n\tadd.cc.u32 z, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}"
              : "+r"(ripple[i])
              : "r"(o), "r"(t1[i][j]));
        }
      }
#pragma unroll
      for (int i = 0; i < NQ; ++i)
        if (ripple[i]) {
#pragma unroll
          for (int j = 0; j < D; ++j)
            if ((ripple[i] >> (D - 1 - j)) & 1u) exact::carry_up_s(ad[i][j] + 12, end_s);
        }
    }
  }
  __syncthreads();

  // per-block partials (same layout as K1)
  const int nbins = static_cast<int>(D * nb);
  std::uint32_t* out = a.partials + static_cast<std::size_t>(blockIdx.x) * kXWords * nbins;
  for (int i = tid; i < nbins * kXWords; i += nt) {
    const int w = i / nbins, cc = i % nbins;
    out[i] = bins[cc * kXWords + w];
  }
  unsigned long long* sout = a.scal_partials + static_cast<std::size_t>(blockIdx.x) * kScalarAccs * kXWords;
  for (int i = tid; i < kScalarAccs * kXWords; i += nt) {
    const int kind = i / kXWords, w = i % kXWords;
    const std::uint32_t* src = acc + kind * kLaneCopies * kXWords + w;
    unsigned long long s = 0;
#pragma unroll 8
    for (int l = 0; l < kLaneCopies; ++l) s += src[l * kXWords];
    sout[i] = s;
  }
}

}  // namespace mcubes::gpu
