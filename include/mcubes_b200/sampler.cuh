// SPDX-License-Identifier: Apache-2.0
//
// K1: the m-Cubes sampling kernel (V-Sample / V-Sample-No-Adjust).
//
// Replaces run_cube + sample_all_cubes (sampler.hpp:147-181, 213-278) and the
// paper's atomics-based CUDA V-Sample.  Design (DESIGN.md
// section 4):
//
//  * Persistent grid: one block per SM (1024 threads on the Philox path, 768
//    on compat).  Each thread walks its share of the linear work index n in
//    whole rows along axis 0 (row mode) or cube by cube (CubeWalk below); the
//    n -> cube map is a bijection that spreads neighbouring lanes over distinct
//    bins on every axis and depends on (m, g, d) only.
//  * The grid lives in shared memory as per-bin {left, width} (compat) or
//    {left - i*width, width} (Philox: the point is one FMA) pairs.
//  * compat reproduces the reference arithmetic exactly: SplitMix keyed
//    stream, (digit + r) / g, the bin map and jacobian of grid.hpp:204-224,
//    Welford (sampler.hpp:93-104); IEEE divisions by the launch constants use
//    Markstein's correction with a correctly rounded reciprocal
//    (q0 = a*y; r = fma(-q0, b, a); q = fma(r, y, q0)), i.e. the same bits as a/b.
//    Philox: Philox4x32-10 keyed by the iteration, 32-bit uniforms, FMA
//    transform, restated bit for bit by oracle/mcubes_oracle.c run_cube_philox.
//  * Estimates and variances are summed EXACTLY into shared-memory
//    superaccumulators (exact.cuh), the d x n_bins contributions (f*J)^2 too
//    (compat: exact values; Philox: rounded to 24 significant bits first).  No
//    global atomics per sample; results independent of launch geometry and of
//    how cubes are split across GPUs, and equal to the reference's ExactSum.
//  * At the end each block adds its nonzero accumulator words into the
//    exchange buffer (exact 64-bit integer atomics; see the flush below).
#pragma once

#include <cooperative_groups.h>

#include <cmath>
#include <cstdint>
#include <span>
#include <type_traits>

#include "config.cuh"
#include "exact.cuh"
#include "integrands.cuh"
#include "rng.cuh"

namespace mcubes::gpu {

/// Shared-memory Welford reciprocal table length (RN(1/n), n < kRcpSmem).
inline constexpr int kRcpSmem = 64;

struct SampleArgs {
  const double* edges;  ///< device, dims x nb right edges (grid.hpp:303 layout)
  const double* lower;  ///< device, dims
  std::uint32_t dims, nb;
  std::uint32_t bin_axes;  ///< 0 = frozen (v_sample_no_adjust), 1 = axis0_only, dims = all_axes
  /// Axes [bin_lo, bin_lo + bin_n) deposit bins in this launch.  A shape
  /// whose bin_axes x (n_bins + 1) exact accumulators exceed one CTA's shared
  /// memory is sampled in several passes over the same (keyed, hence
  /// identical) points, each holding the histograms of a subset of the axes;
  /// the first pass (`scalars`) also sums the estimate, the variance and the
  /// sample counts.  Single pass: bin_lo = 0, bin_n = bin_axes, scalars = 1.
  std::uint32_t bin_lo, bin_n;
  std::uint32_t scalars;
  std::uint32_t publish;  ///< peer exchange: this (last) pass publishes the iteration flag
  std::uint64_t m, p, g;
  double nbd;      ///< double(nb)
  double gd;       ///< double(g)
  double rcp_g;    ///< RN(1/g)
  double scale;    ///< 1.0 / (double(m) * double(p))   (sampler.hpp:293)
  double pp1;      ///< double(p) * double(p - 1)       (sampler.hpp:178)
  double rcp_pp1;  ///< RN(1/pp1)
  double cs;       ///< philox: nb / (g * 2^32)   (32-bit uniform -> bin coordinate)
  double nbg;      ///< philox: nb / g            (cube digit -> bin coordinate)
  double nbpow;    ///< philox: nb^D              (jacobian = nb^D * prod widths)
  std::uint64_t iter_root;  ///< compat: iteration_root(seed, it); philox: the key
  std::uint64_t n0, n1;     ///< this launch's slice of the linear work index
  std::uint64_t A;          ///< cube mode: cube(n) = n*A mod m; row mode: rho(r) = r*A mod R
  std::uint64_t stepT;      ///< (gridDim*blockDim*A) mod m
  std::uint64_t step_digits[kMaxDims];  ///< cube mode: base-g digits of stepT (axis 0 first);
                                        ///< row mode: digits of stepR at axes 1..D-1
  std::uint32_t row_mode;               ///< 1 = walk whole rows along axis 0 (see K1)
  std::uint64_t R;                      ///< rows m / g
  std::uint64_t stepR;                  ///< row mode: (T*A) mod R, A = A' = 1 + g + ... + g^(D-2)
  std::uint32_t round_keys[20];         ///< philox: (k0, k1) of rounds 0..9 (uniform; folded into LOP3)
  unsigned long long* words;  ///< exchange accumulators (zeroed): every block adds its nonzero words here;
                              ///< words[-3..-1]: overflowed addends, finite and non-finite samples (kXHeader)
  std::uint32_t nb_out;       ///< n_bins of the exchange layout (the padding cell folds into bin nb_out-1)
  std::uint32_t tab_copies;   ///< copies of the grid table in shared memory (runtime-n_bins kernels; 0 = 1)
  unsigned long long* err_key;  ///< min over non-finite samples of t*p + k (init all-ones)
  const int* stop;              ///< nullable; nonzero = run finished, skip
  PeerArgs peer;                ///< multi-GPU exchange over peer memory (peer.npeers == 0: local words)
};

/// Accumulator slots in one block's partial.
MCB_HD constexpr int block_accs(std::uint32_t bin_axes, std::uint32_t nb) {
  return kScalarAccs * kLaneCopies + static_cast<int>(bin_axes * nb);
}

/// Dynamic shared memory of K1 for a given shape, with `copies` interleaved
/// copies of the grid table (see stage_grid).
MCB_HD constexpr std::size_t sample_smem_bytes(int D, std::uint32_t nb, std::uint32_t bin_axes, std::uint32_t copies = 1) {
  const std::size_t grid = 2 * sizeof(double) * static_cast<std::size_t>(D) * nb * copies;  // {left, width}
  const std::size_t rcp = sizeof(double) * kRcpSmem;
  std::size_t acc = sizeof(std::uint32_t) * static_cast<std::size_t>(block_accs(bin_axes, nb)) * kXWords;
  acc = (acc + 15) & ~std::size_t{15};
  return grid + rcp + acc;
}

/// 128-bit shared load at a 32-bit shared-window byte address.
__device__ __forceinline__ double2 lds_d2(std::uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}

/// Correctly rounded a / b given y = RN(1/b) (Markstein).
__device__ __forceinline__ double div_rn(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, y, q0);
}

/// Dynamic shared memory K1 may use (the opt-in maximum less a margin for
/// its few static shared variables).
inline constexpr std::size_t kK1SmemBudget = 227 * 1024 - 1024;

/// Grid-table copies of the compile-time-n_bins kernels: the most (8, 4, 2)
/// that fit next to every axis' histograms, else 1.
#ifndef MCB_K1_TAB_COPIES_MAX
#define MCB_K1_TAB_COPIES_MAX 8
#endif
constexpr std::uint32_t fixed_tab_copies(int D, std::uint32_t pnb) {
  for (std::uint32_t c = MCB_K1_TAB_COPIES_MAX; c > 1; c >>= 1)
    if (sample_smem_bytes(D, pnb, static_cast<std::uint32_t>(D), c) <= kK1SmemBudget) return c;
  return 1;
}

template <int D>
using DigitT = std::conditional_t<(D <= 2), std::uint64_t, std::uint32_t>;

/// Stage the grid as per-bin {left edge, width} pairs (one 128-bit LDS per
/// axis per sample).  width = right - left exactly as grid.hpp:218-219.
///
/// The table is stored C times, interleaved: entry e's copies fill C
/// consecutive 16-byte slots, and lane l reads copy l mod C.  A 128-bit
/// shared load is served a quarter-warp (8 lanes, 128 B) per wavefront; the
/// 8 lanes of a quarter then always sit in 8 distinct bank groups whatever
/// bins they hit, so a table lookup costs the minimum 4 wavefronts instead of
/// ~9 for random bins in one copy (ncu: the table lookups were 54 % of a
/// saturated shared-memory pipe).
template <int D>
__device__ __forceinline__ void stage_grid(double2* LW, const SampleArgs& a, std::uint32_t C) {
  const std::uint32_t nb = a.nb;
  for (std::uint32_t idx = threadIdx.x; idx < D * nb; idx += blockDim.x) {
    const std::uint32_t j = idx / nb, i = idx % nb;
    const double* row = a.edges + static_cast<std::size_t>(j) * nb;
    const double left = i == 0 ? a.lower[j] : row[i - 1];
    const double2 v = make_double2(left, __dsub_rn(row[i], left));
    for (std::uint32_t c = 0; c < C; ++c) LW[idx * C + c] = v;
  }
}

/// Philox path: per-bin {A, width} with A = left - i*width, so the point is
/// one FMA of the bin coordinate z: x = A + z*width (= left + (z-i)*width up
/// to one rounding).
/// The table has nb + 1 entries per axis: entry nb repeats bin nb-1, so a
/// bin coordinate that rounds up to exactly nb (possible only for g >= 2^20)
/// needs no clamp -- its deposit lands in a padding cell that K1's flush folds into
/// bin nb-1 (philox_pnb).
template <int D>
__device__ __forceinline__ void stage_grid_fast(double2* LW, const SampleArgs& a, std::uint32_t C) {
  const std::uint32_t nb = a.nb, pnb = nb + 1;
  for (std::uint32_t idx = threadIdx.x; idx < D * pnb; idx += blockDim.x) {
    const std::uint32_t j = idx / pnb, i0 = idx % pnb, i = i0 < nb ? i0 : nb - 1;
    const double* row = a.edges + static_cast<std::size_t>(j) * nb;
    const double left = i == 0 ? a.lower[j] : row[i - 1];
    const double w = __dsub_rn(row[i], left);
    const double2 v = make_double2(__fma_rn(-static_cast<double>(i), w, left), w);
    for (std::uint32_t c = 0; c < C; ++c) LW[idx * C + c] = v;
  }
}

/// Philox4x32-10 with the per-round keys read from the launch parameters
/// (constant bank), so a round is two IMAD.WIDE + two LOP3.
__device__ __forceinline__ rng::U4 philox_rk(rng::U4 c, const std::uint32_t (&rk)[20]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const std::uint64_t p0 = static_cast<std::uint64_t>(rng::kPhiloxM0) * c.x;
    const std::uint64_t p1 = static_cast<std::uint64_t>(rng::kPhiloxM1) * c.z;
    c = rng::U4{static_cast<std::uint32_t>(p1 >> 32) ^ c.y ^ rk[2 * r], static_cast<std::uint32_t>(p1),
                static_cast<std::uint32_t>(p0 >> 32) ^ c.w ^ rk[2 * r + 1], static_cast<std::uint32_t>(p0)};
  }
  return c;
}

/// Philox path, one sample: D uniforms from ceil(D/4) Philox4x32-10 blocks
/// keyed by the iteration with counter (cube, sample, block); bin coordinate
/// z = (digit + u) * nb / g as one FMA from the per-cube base; point and
/// jacobian from the {A, width} table.  Returns f*J.
template <class F, int D, int NB, class Dig>
__device__ __forceinline__ double sample_point_fast(const SampleArgs& a, const F& f, std::uint32_t lw_s,
                                                    std::uint32_t C, const Dig (&dig)[D], std::uint64_t t,
                                                    std::uint32_t k, double (&x)[D], std::uint32_t (&bin)[D],
                                                    double& fx) {
  const std::uint32_t pnb = (NB ? static_cast<std::uint32_t>(NB) : a.nb) + 1;  // padded table (stage_grid_fast)
  std::uint32_t r[(D + 3) & ~3];
#pragma unroll
  for (int q = 0; q < (D + 3) / 4; ++q) {
    const rng::U4 o = philox_rk(
        rng::U4{static_cast<std::uint32_t>(t), static_cast<std::uint32_t>(t >> 32), k, static_cast<std::uint32_t>(q)},
        a.round_keys);
    r[4 * q] = o.x;
    r[4 * q + 1] = o.y;
    r[4 * q + 2] = o.z;
    r[4 * q + 3] = o.w;
  }
  double jw = 1.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    // bin coordinate z = (digit + r / 2^32) * nb / g.  For 32-bit digits the
    // 64-bit integer digit:r (the register pair itself) converts exactly
    // (digit < 2^21), so z is one I2F.U64 and one DMUL: z = RN((digit 2^32 + r) cs).
    double z;
    if constexpr (sizeof(Dig) == 4) {
      // 2^52 + digit:r is the double with words {0x43300000 | digit, r}
      // (digit < 2^20); subtracting 2^52 is exact (no I2F on the XU pipe)
      z = __dmul_rn(__dadd_rn(__hiloint2double(static_cast<int>(0x43300000u | dig[j]), static_cast<int>(r[j])),
                              -0x1p52),
                    a.cs);
    } else {
      z = __fma_rn(__uint2double_rn(r[j]), a.cs, __dmul_rn(__ull2double_rn(dig[j]), a.nbg));
    }
    const std::uint32_t i = __double2uint_rz(z);  // 0 <= z <= nb: no clamp (padded table)
    const double2 lw = lds_d2(lw_s + (static_cast<std::uint32_t>(j) * pnb + i) * C * 16u);  // lane's copy
    x[j] = __fma_rn(z, lw.y, lw.x);
    jw = j == 0 ? lw.y : __dmul_rn(jw, lw.y);
    bin[j] = i;
  }
  fx = static_cast<double>(f(std::span<const double>(x, D)));
  return __dmul_rn(fx, __dmul_rn(jw, a.nbpow));
}

/// One sample: point, jacobian, bins and f*J of sample k of a cube
/// (sampler.hpp:163-170 with transform_impl, grid.hpp:204-224).
template <class F, int D, int NB>
__device__ __forceinline__ double sample_point(const SampleArgs& a, const F& f, std::uint32_t lw_s, std::uint32_t C,
                                               const double (&dg)[D], std::uint64_t croot, std::uint32_t k,
                                               double (&x)[D], std::uint32_t (&bin)[D], double& fx) {
  const std::uint32_t nb = NB ? static_cast<std::uint32_t>(NB) : a.nb, nbm1 = nb - 1;
  double r[D];
  const std::uint64_t proot = rng::feed(croot, k);  // rng.hpp:55-58
#pragma unroll
  for (int j = 0; j < D; ++j) r[j] = rng::to_unit(rng::feed(proot, static_cast<std::uint64_t>(j)));
  double jac = 1.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    // u_j = (digit_j + r_j) / g  (sampler.hpp:165-166)
    const double u = div_rn(__dadd_rn(dg[j], r[j]), a.gd, a.rcp_g);
    // transform_impl (grid.hpp:209-222)
    const double z = __dmul_rn(u, a.nbd);
    std::uint32_t i = __double2uint_rz(z);
    i = i < nbm1 ? i : nbm1;
    const double2 lw = lds_d2(lw_s + (static_cast<std::uint32_t>(j) * nb + i) * C * 16u);  // lane's copy
    x[j] = __dadd_rn(lw.x, __dmul_rn(__dsub_rn(z, static_cast<double>(i)), lw.y));
    jac = __dmul_rn(jac, __dmul_rn(a.nbd, lw.y));
    bin[j] = i;
  }
  fx = static_cast<double>(f(std::span<const double>(x, D)));
  return __dmul_rn(fx, jac);
}

/// The work-index -> cube walk of one K1 thread (results do not depend on
/// it: the sums are exact and the stream is keyed by cube).
///  cube mode: linear index n -> cube t = n*A mod m, thread stride T, all
///    digits advanced per cube by an odometer add of (T*A mod m).
///  row mode (m/g >= 2^20 rows): n = r*g + e; row r maps to the digits of
///    axes 1..D-1 of rho = r*A' mod (m/g), and the thread walks the whole row
///    along axis 0 with d0 = (e + digit1(rho)) mod g, so per cube only axis 0
///    changes; rows advance by an odometer add of (T*A' mod m/g).
///  Both spread neighbouring lanes over distinct bins on every axis.
template <int D, bool kShareIndex = false>
struct CubeWalk {
  using Dig = DigitT<D>;
  Dig dig[D];
  std::uint64_t t = 0, rp = 0, rowbase = 0, rho = 0, n_ = 0;
  /// The cube-mode linear work index.  kShareIndex keeps it in rp (the row
  /// counter of row mode; a runtime flag selects the walk): one register
  /// pair fewer -- measured +2.3 % on compat, -1.1 % on Philox (register
  /// allocation at the cap), so the kernel picks it per stream.
  __device__ __forceinline__ std::uint64_t& n() {
    if constexpr (kShareIndex) return rp;
    else return n_;
  }
  std::uint32_t e = 0, e_end = 0;
  bool rows = false;

  __device__ __forceinline__ void odometer(const SampleArgs& a, int j0) {  // dig[j0..] += step_digits[j0..]
    const Dig g = static_cast<Dig>(a.g);
    if constexpr (sizeof(Dig) == 4) {
      // v = dig + step + carry (< 2g < 2^31); w = v - g; digit = min(v, w)
      // unsigned; carry = w >= 0, folded into the next axis' add
      std::uint32_t borrow = 1;  // 1 - carry
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (j < j0) continue;
        const std::uint32_t v = dig[j] + static_cast<std::uint32_t>(a.step_digits[j]) + 1u - borrow;
        const std::uint32_t w = v - g;
        dig[j] = v < w ? v : w;
        borrow = w >> 31;
      }
    } else {
      Dig carry = 0;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        if (j < j0) continue;
        const Dig v = dig[j] + static_cast<Dig>(a.step_digits[j]) + carry;
        carry = v >= g ? 1 : 0;
        dig[j] = carry ? v - g : v;
      }
    }
  }
  /// start of a row: e range clipped to [n0, n1), axis-0 digit, cube index
  __device__ __forceinline__ void row_start(const SampleArgs& a) {
    const Dig g = static_cast<Dig>(a.g);
    const std::uint64_t r0 = rp * a.g;
    e = r0 < a.n0 ? static_cast<std::uint32_t>(a.n0 - r0) : 0u;
    e_end = static_cast<std::uint32_t>(a.n1 - r0 < a.g ? a.n1 - r0 : a.g);
    Dig d0 = static_cast<Dig>(e) + dig[D >= 2 ? 1 : 0];
    if (d0 >= g) d0 -= g;
    dig[0] = d0;
    rowbase = rho * a.g;
    t = rowbase + d0;
  }
  /// First cube of global thread gtid; false if it has none.
  __device__ __forceinline__ bool init(const SampleArgs& a, std::uint64_t gtid) {
    rows = a.row_mode != 0 && D >= 2;
    if (rows) {
      rp = a.n0 / a.g + gtid;
      if (rp * a.g >= a.n1) return false;
      rho = static_cast<std::uint64_t>((static_cast<unsigned __int128>(rp) * a.A) % a.R);
      std::uint64_t tt = rho;
#pragma unroll
      for (int j = 1; j < D; ++j) {
        dig[j] = static_cast<Dig>(tt % a.g);
        tt /= a.g;
      }
      row_start(a);
      return true;
    }
    n() = a.n0 + gtid;
    if (n() >= a.n1) return false;
    t = static_cast<std::uint64_t>((static_cast<unsigned __int128>(n() % a.m) * a.A) % a.m);
    std::uint64_t tt = t;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      dig[j] = static_cast<Dig>(tt % a.g);
      tt /= a.g;
    }
    return true;
  }
  /// Advance by the thread stride T; false when done.  all_axes = false when
  /// only dig[0] changed.
  __device__ __forceinline__ bool next(const SampleArgs& a, std::uint64_t T, bool& all_axes) {
    all_axes = true;
    if (rows) {
      if (++e < e_end) {  // along the row: only axis 0 moves
        Dig d0 = dig[0] + 1;
        if (d0 == static_cast<Dig>(a.g)) d0 = 0;
        dig[0] = d0;
        t = rowbase + d0;
        all_axes = false;
        return true;
      }
      rp += T;
      if (rp * a.g >= a.n1) return false;
      odometer(a, 1);  // rho += T*A' (mod m/g) on the digits of axes 1..D-1
      rho += a.stepR;
      if (rho >= a.R) rho -= a.R;
      row_start(a);
      return true;
    }
    n() += T;
    if (n() >= a.n1) return false;
    // cube (n + T)*A mod m: odometer add of stepT's digits
    t += a.stepT;
    if (t >= a.m) t -= a.m;
    odometer(a, 0);
    return true;
  }
};

#ifdef MCB_K1_TIMING
// latency probe (tools/latbench.cu): %globaltimer at K1's phases, min/max over blocks
__device__ unsigned long long g_k1_times[8];
#define MCB_K1_STAMP(i, op)                                  \
  if (threadIdx.x == 0) {                                    \
    unsigned long long t_;                                   \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));   \
    op(&g_k1_times[i], t_);                                  \
  }
#else
#define MCB_K1_STAMP(i, op)
#endif

/// K1.  NB = n_bins when known at compile time (50, the reference default
/// and every BASELINE config), 0 = runtime n_bins.
template <class F, int D, RngKind R, int NB = 0>
__global__ void __launch_bounds__(sample_threads(R, D), 1) vsample_kernel(const SampleArgs a, const F f) {
  pdl_trigger();  // the finish kernel may launch now; it waits for this grid to complete
  MCB_K1_STAMP(0, atomicMin)
  MCB_K1_STAMP(1, atomicMax)
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned int nonfinite_s;        // this block's non-finite samples (flushed with the words)
  __shared__ unsigned long long cubes_s;      // cubes this block visited (-> the device-counted sample total)
  __shared__ unsigned int overflow_s;         // addends that overflowed to inf (words[-3])
  // cells per axis: n_bins, plus one padding cell on the Philox path (see stage_grid_fast)
  const std::uint32_t nb = (NB ? static_cast<std::uint32_t>(NB) : a.nb) + (philox_stream(R) ? 1u : 0u);
  double2* LW = reinterpret_cast<double2*>(smem);
  // grid-table copies (stage_grid): compile-time for the fixed-n_bins kernels
  constexpr std::uint32_t kFixedC = NB ? fixed_tab_copies(D, static_cast<std::uint32_t>(NB) + (philox_stream(R) ? 1u : 0u)) : 0u;
  const std::uint32_t C = kFixedC ? kFixedC : (a.tab_copies ? a.tab_copies : 1u);
  double* rcp = reinterpret_cast<double*>(LW + D * nb * C);
  std::uint32_t* acc = reinterpret_cast<std::uint32_t*>(rcp + kRcpSmem);
  const int nacc = block_accs(a.bin_n, nb);
  const int tid = threadIdx.x, nt = blockDim.x;

  {  // zero the accumulators, stage the grid and the Welford reciprocals
    const int nwords = nacc * kXWords;
    for (int i = tid; i < nwords; i += nt) acc[i] = 0u;
    for (int i = tid; i < kRcpSmem; i += nt) rcp[i] = i ? 1.0 / static_cast<double>(i) : 0.0;
    if (tid == 0) {
      nonfinite_s = 0u;
      overflow_s = 0u;
      cubes_s = 0ull;
    }
    pdl_wait();  // the grid, the stop flag and the exchange words come from the previous kernels
    if (a.stop && *a.stop) return;  // (uniform across the block)
    if constexpr (R == RngKind::compat) stage_grid<D>(LW, a, C);
    else stage_grid_fast<D>(LW, a, C);
  }
  __syncthreads();
  MCB_K1_STAMP(2, atomicMax)

  const int lane = tid & 31;
  // this lane's table copy (stage_grid), as a 32-bit shared-window byte address
  const std::uint32_t lw_s = static_cast<std::uint32_t>(__cvta_generic_to_shared(LW)) + 16u * (static_cast<std::uint32_t>(lane) & (C - 1));
  std::uint32_t* bins = acc + kScalarAccs * kLaneCopies * kXWords;
  // 32-bit shared-window byte addresses of the accumulators
  const std::uint32_t acc_s = static_cast<std::uint32_t>(__cvta_generic_to_shared(acc));
  constexpr std::uint32_t kAccBytes = 4u * kXWords;
  const std::uint32_t est_pos_s = acc_s + (0 * kLaneCopies + lane) * kAccBytes;
  const std::uint32_t est_neg_s = acc_s + (1 * kLaneCopies + lane) * kAccBytes;
  const std::uint32_t var_s = acc_s + (2 * kLaneCopies + lane) * kAccBytes;
  const std::uint32_t bins_s = acc_s + kScalarAccs * kLaneCopies * kAccBytes;
  // The compile-time-n_bins kernels (NB != 0) run every shape in one pass
  // (launch_k1 sends multi-pass shapes to NB = 0), so their pass logic folds away.
  constexpr bool kOnePass = NB != 0;
  const std::uint32_t bin_n = kOnePass ? a.bin_axes : a.bin_n, bin_lo = kOnePass ? 0u : a.bin_lo;
  const bool scalars = kOnePass || a.scalars != 0;
  // An exact addend that overflowed to +-inf ((f J)^2, a cube's sum or
  // variance): the reference's ExactSum::add throws (exact_sum.hpp:34).  Its
  // digits are deposited like any other (they stay inside the accumulator);
  // the flag is counted once per thread at the end and the finish kernel
  // stops the run with that error.
  bool ovf = false;
  constexpr std::uint32_t kCell = 4u * kXWords;  // bytes per accumulator

  // sampler.hpp:173-176: the same (f J)^2 on every axis -- split it once,
  // deposit word-major across the axes
  // (compat: the exact (f J)^2, as the reference's ExactBins; philox: rounded
  // to 24 significant bits -- one or two word atomics instead of three, exact.cuh)
  constexpr bool kR24 = R == RngKind::philox;  // 24-bit bin addends (else exact, as ExactBins)
  auto deposit = [&](double fj, const std::uint32_t (&bin)[D]) {
    using Dg = std::conditional_t<kR24, exact::Digits2, exact::Digits>;
    Dg dgt;
    bool nz;
    const double sq = __dmul_rn(fj, fj);
    if constexpr (kR24) nz = exact::split_r24(sq, dgt);
    else nz = exact::split(sq, dgt);
    // (f J)^2 overflowed (|f J| > ~1.3e154; with 24-bit addends also a value
    // that RN24 rounds up to 2^1024)
    ovf |= dgt.be == 0x7ffu;
    if (nz) {
      const std::uint32_t wb = bins_s + 4u * dgt.w;
      if (bin_n == static_cast<std::uint32_t>(D)) {  // every axis in one pass (the common case)
        if constexpr (philox_stream(R) && NB != 0) {  // row offsets as immediates
          std::uint32_t base[D];
#pragma unroll
          for (int j = 0; j < D; ++j) base[j] = wb + bin[j] * kCell;
          if constexpr (kR24) exact::add_digits2_rows<D, static_cast<std::uint32_t>(NB + 1) * kCell>(base, dgt);
          else exact::add_digits_rows<D, static_cast<std::uint32_t>(NB + 1) * kCell>(base, dgt);
        } else {
          std::uint32_t ad[D];
#pragma unroll
          for (int j = 0; j < D; ++j) ad[j] = wb + bin[j] * kCell + static_cast<std::uint32_t>(j) * nb * kCell;
          if constexpr (kR24) exact::add_digits2_s<D>(ad, dgt);
          else exact::add_digits_s<D>(ad, dgt);
        }
      } else if (kOnePass || (bin_n == 1 && bin_lo == 0)) {  // BinUpdate::axis0_only
        const std::uint32_t ad[1] = {wb + bin[0] * kCell};
        if constexpr (kR24) exact::add_digits2_s<1>(ad, dgt);
        else exact::add_digits_s<1>(ad, dgt);
      } else {  // a pass over axes [bin_lo, bin_lo + bin_n) (compile-time axis index, runtime predicate)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const std::uint32_t rel = static_cast<std::uint32_t>(j) - bin_lo;
          if (rel < bin_n) {
            const std::uint32_t ad[1] = {wb + bin[j] * kCell + rel * nb * kCell};
            if constexpr (kR24) exact::add_digits2_s<1>(ad, dgt);
            else exact::add_digits_s<1>(ad, dgt);
          }
        }
      }
    }
  };

  const std::uint64_t T = static_cast<std::uint64_t>(gridDim.x) * nt;
  CubeWalk<D, R == RngKind::compat> cw;
  bool active = cw.init(a, static_cast<std::uint64_t>(blockIdx.x) * nt + tid);
  // compat: per-axis cube coordinate double(digit) (the philox path reads the digits)
  double cd[R == RngKind::compat ? D : 1];
  auto coord = [&](int j) {
    if constexpr (R == RngKind::compat) cd[j] = static_cast<double>(cw.dig[j]);
  };
#pragma unroll
  for (int j = 0; j < D; ++j) coord(j);

  const std::uint32_t p = static_cast<std::uint32_t>(a.p);
  std::uint32_t ncubes = 0;  // cubes this thread visited (counted, not derived: the coverage check)
  while (active) {
    const std::uint64_t t = cw.t;
    ncubes += scalars ? 1u : 0u;
    double sum, var;
    if constexpr (R == RngKind::compat) {
      const std::uint64_t croot = rng::feed(a.iter_root, t);  // rng.hpp:51-54
      double mean = 0.0, m2 = 0.0;
      sum = 0.0;
      for (std::uint32_t k = 0; k < p; ++k) {
        double x[D];
        std::uint32_t bin[D];
        double fx;
        const double fj = sample_point<F, D, NB>(a, f, lw_s, C, cd, croot, k, x, bin, fx);
        if (!isfinite(fj)) {  // sampler.hpp:170 -- the first failure in serial order is reported
          atomicMin(a.err_key, static_cast<unsigned long long>(t * a.p + k));
          if (scalars) atomicAdd(&nonfinite_s, 1u);  // exchanged with the words: all ranks stop together
          continue;
        }
        sum = __dadd_rn(sum, __dmul_rn(fj, a.scale));
        // Welford (sampler.hpp:98-103)
        const std::uint32_t nk = k + 1;
        const double dd = __dsub_rn(fj, mean);
        const double q = nk < static_cast<std::uint32_t>(kRcpSmem) ? div_rn(dd, static_cast<double>(nk), rcp[nk])
                                                                   : __ddiv_rn(dd, static_cast<double>(nk));
        mean = __dadd_rn(mean, q);
        m2 = __dadd_rn(m2, __dmul_rn(dd, __dsub_rn(fj, mean)));
        if (bin_n) deposit(fj, bin);
      }
      var = div_rn(m2, a.pp1, a.rcp_pp1);  // sampler.hpp:178-179
    } else {
      // Philox path: same estimator (sum of f*J, Welford variance of the
      // mean), FMA-contracted arithmetic; validated statistically.
      double mean = 0.0, m2 = 0.0;
      sum = 0.0;
      for (std::uint32_t k = 0; k < p; ++k) {
        double x[D];
        std::uint32_t bin[D];
        double fx;
        const double fj = sample_point_fast<F, D, NB>(a, f, lw_s, C, cw.dig, t, k, x, bin, fx);
        if (!isfinite(fj)) {
          atomicMin(a.err_key, static_cast<unsigned long long>(t * a.p + k));
          if (scalars) atomicAdd(&nonfinite_s, 1u);  // exchanged with the words: all ranks stop together
          continue;
        }
        sum = __dadd_rn(sum, fj);
        // Welford with y = RN(1/n): mean += (f - mean) * y
        const std::uint32_t nk = k + 1;
        double y;
        if (nk <= 2) y = nk == 1 ? 1.0 : 0.5;  // p = 2 (every BASELINE shape above 1e6 calls): no LDS
        else y = nk < static_cast<std::uint32_t>(kRcpSmem) ? rcp[nk] : __drcp_rn(static_cast<double>(nk));
        const double dd = __dsub_rn(fj, mean);
        mean = __fma_rn(dd, y, mean);
        m2 = __fma_rn(dd, __dsub_rn(fj, mean), m2);
        if (bin_n) deposit(fj, bin);
      }
      sum = __dmul_rn(sum, a.scale);
      var = __dmul_rn(m2, a.rcp_pp1);
    }
    if (!(var > 0.0)) var = 0.0;  // sampler.hpp:179 (a NaN variance becomes 0, an infinite one stays)
    if (scalars) {
      ovf |= !(fabs(sum) < INFINITY) || !(var < INFINITY);  // ExactSum::add would throw (exact_sum.hpp:34)
      exact::add_shared2_s(sum < 0.0 ? est_neg_s : est_pos_s, sum, var_s, var);
    }

    bool all_axes;
    active = cw.next(a, T, all_axes);
    if (all_axes) {
#pragma unroll
      for (int j = 0; j < D; ++j) coord(j);
    } else {
      coord(0);
    }
  }
  MCB_K1_STAMP(3, atomicMin)
  if (ovf) atomicAdd(&overflow_s, 1u);
  {  // the block's visited-cube count (warp sums in u64: a thread's count fits u32, a block's may not)
    unsigned long long c = ncubes;
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((tid & 31) == 0 && c) atomicAdd(&cubes_s, c);
  }
  __syncthreads();
  MCB_K1_STAMP(4, atomicMax)

  // Flush: the block's nonzero words go straight into the exchange buffer as
  // exact 64-bit integer adds -- a few thousand per block per iteration,
  // against the ~10^8 shared-memory deposits they summarise -- so no
  // per-block partials are written and no separate reduction pass reads them
  // back.  Integer addition is order-free: bit-reproducible for any launch
  // geometry and GPU count.  (The reference merges per-worker ExactSums in
  // worker order, sampler.hpp:272-276; the integer sum is the same.)
  // With the peer-memory exchange every word goes to every rank's buffer
  // (system-scope reductions over NVLink), otherwise to the local buffer
  // that a collective then all-reduces.
  const int npeers = a.peer.npeers;
  auto add_word = [&](std::ptrdiff_t idx, unsigned long long v) {
    if (npeers == 0) {
      red_add_gpu(a.words + idx, v);
    } else {
      for (int q = 0; q < npeers; ++q) red_add_sys(a.peer.words[q] + idx, v);
    }
  };
  {
    // In a 2-CTA cluster each CTA adds BOTH CTAs' words (its own + its
    // partner's over DSMEM; the u64 sums of two u32 words are exact) for one
    // half of the words: half the global reductions per SM.
    namespace cg = cooperative_groups;
    const cg::cluster_group cluster = cg::this_cluster();
    const unsigned csize = cluster.num_blocks();
    const unsigned crank = cluster.block_rank();
    const std::uint32_t* peer_acc = acc;
    if (csize == 2) {
      cluster.sync();  // the partner's accumulators are final
      peer_acc = cluster.map_shared_rank(acc, crank ^ 1u);
    }
    const std::uint32_t* peer_bins = peer_acc + kScalarAccs * kLaneCopies * kXWords;
    const int ncells = static_cast<int>(a.bin_n * nb);
    const int nbw = ncells * kXWords;
    auto flush_bin_word = [&](int i, unsigned long long v) {  // block word i (cell-major) -> exchange slot
      const int c = i / kXWords, w = i - c * kXWords;
      const int ax = c / static_cast<int>(nb), cell = c - ax * static_cast<int>(nb);
      const int slot = (static_cast<int>(a.bin_lo) + ax) * static_cast<int>(a.nb_out) +
                       min(cell, static_cast<int>(a.nb_out) - 1);
      add_word(static_cast<std::ptrdiff_t>(kScalarAccs + slot) * kXWords + w, v);
    };
    const int b0 = csize == 2 ? (crank ? nbw / 2 : 0) : 0, b1 = csize == 2 ? (crank ? nbw : nbw / 2) : nbw;
    for (int i = b0 + tid; i < b1; i += nt) {
      const unsigned long long v = static_cast<unsigned long long>(bins[i]) +
                                   (csize == 2 ? static_cast<unsigned long long>(peer_bins[i]) : 0ull);
      if (v) flush_bin_word(i, v);
    }
    // est+/est-/var: the 32 lane copies (of both CTAs) folded into u64 word sums (< 2^38, exact)
    const int nsw = scalars ? kScalarAccs * kXWords : 0;  // later passes deposit bins only
    const int s0 = csize == 2 ? (crank ? nsw / 2 : 0) : 0, s1 = csize == 2 ? (crank ? nsw : nsw / 2) : nsw;
    for (int i = s0 + tid; i < s1; i += nt) {
      const int kind = i / kXWords, w = i % kXWords;
      const std::uint32_t* src = acc + kind * kLaneCopies * kXWords + w;
      const std::uint32_t* psrc = peer_acc + kind * kLaneCopies * kXWords + w;
      unsigned long long sum = 0;
#pragma unroll 8
      for (int l = 0; l < kLaneCopies; ++l) sum += src[l * kXWords];
      if (csize == 2) {
#pragma unroll 8
        for (int l = 0; l < kLaneCopies; ++l) sum += psrc[l * kXWords];
      }
      if (sum) add_word(i, sum);
    }
    if (tid == 0 && nonfinite_s) add_word(-1, nonfinite_s);  // words[-1]: the non-finite count (own CTA's)
    if (tid == 0 && overflow_s) add_word(-3, overflow_s);    // words[-3]: overflowed addends (own CTA's)
    // words[-2]: finite samples taken = visited cubes * p - non-finite samples (own CTA's); the
    // finish kernel turns it into the write count (samples * bin_axes, sampler.hpp:116-119)
    if (tid == 0 && cubes_s) add_word(-2, cubes_s * a.p - nonfinite_s);
    if (csize == 2) cluster.sync();  // the partner has finished reading this CTA's accumulators
  }
  if (npeers && a.publish) {
    // Publish "this rank's words are in": every thread's reductions are
    // ordered before the block's arrival (fence.sc.sys + barrier); the last
    // block to arrive releases the iteration's flag into every rank's slot.
    __threadfence_system();
    __syncthreads();
    if (tid == 0 && atomicAdd(a.peer.counter, 1u) == gridDim.x - 1) {
      *a.peer.counter = 0u;  // ready for the next launch (stream order)
      __threadfence_system();
      for (int q = 0; q < npeers; ++q) st_release_sys(a.peer.flags[q], a.peer.flag);
    }
  }
  MCB_K1_STAMP(5, atomicMax)
}

/// Recompute one sample (cube t, sample k) -- used to report the point of a
/// NonFiniteSample (sampler.hpp:31-48) after the failing iteration.
template <class F, int D, RngKind R>
__global__ void sample_point_kernel(const SampleArgs a, const F f, std::uint64_t t, std::uint64_t k,
                                    double* out_x, double* out_fx) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* LW = reinterpret_cast<double2*>(smem);
  if constexpr (R == RngKind::compat) stage_grid<D>(LW, a, 1);
  else stage_grid_fast<D>(LW, a, 1);
  __syncthreads();
  if (threadIdx.x != 0) return;
  double dg[D];
  std::uint64_t tt = t;
  for (int j = 0; j < D; ++j) {
    dg[j] = static_cast<double>(tt % a.g);
    tt /= a.g;
  }
  double x[D];
  std::uint32_t bin[D];
  double fx;
  if constexpr (R == RngKind::compat) {
    sample_point<F, D, 0>(a, f, static_cast<std::uint32_t>(__cvta_generic_to_shared(LW)), 1, dg, rng::feed(a.iter_root, t), static_cast<std::uint32_t>(k), x, bin, fx);
  } else {
    DigitT<D> dig[D];
    std::uint64_t t2 = t;
    for (int j = 0; j < D; ++j) {
      dig[j] = static_cast<DigitT<D>>(t2 % a.g);
      t2 /= a.g;
    }
    sample_point_fast<F, D, 0>(a, f, static_cast<std::uint32_t>(__cvta_generic_to_shared(LW)), 1, dig, t, static_cast<std::uint32_t>(k), x, bin, fx);
  }
  for (int j = 0; j < D; ++j) out_x[j] = x[j];
  *out_fx = fx;
}

}  // namespace mcubes::gpu
