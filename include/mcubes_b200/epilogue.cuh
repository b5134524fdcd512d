// SPDX-License-Identifier: Apache-2.0
//
// The fused "finish" kernel K3b+K4 (exact rounding, on-device grid
// adaptation, inverse-variance combination, chi^2 and the convergence gate).
// Together with K1 -- whose blocks add their exact accumulators into the
// exchange buffer (unnormalised u64 digit sums: integer, so exact and
// order-free; under multi-GPU this buffer is what NCCL all-reduces) -- it makes
// one m-Cubes iteration with no host round trip.  The finish kernel rounds each accumulator to
// the nearest double exactly like ExactSum::value() (exact_sum.hpp:65-109),
// producing v_sample's outputs (sampler.hpp:322-332), then replaces
// Grid::adjusted / adjusted_symmetric (grid.hpp:104-146, 232-297),
// weighted_estimate and check_convergence (driver.hpp:146-178) and the loop
// bookkeeping of integrate (driver.hpp:227-256).
#pragma once

#include <cmath>
#include <cstdint>

#include "config.cuh"
#include "exact.cuh"

namespace mcubes::gpu {

/// Device-resident run state for integrate(): K1 exits early once `stop` is set.
struct RunState {
  int stop;
  int converged;
  int failed;  ///< 1: a non-finite sample was seen (err_key holds the first one); 2: an exact addend overflowed
  std::uint32_t iterations_used;
  std::uint32_t failed_iteration;
  std::uint32_t pad;
  double estimate, sigma, chi2_dof;
  unsigned long long samples;     ///< finite samples taken over the run (device-counted by K1)
  unsigned long long bin_writes;  ///< contribution deposits over the run (samples * bin_axes per iteration)
};

/// Exchange-buffer slots: est+, est-, var, then bin_axes*nb bins.
MCB_HD int exchange_accs(std::uint32_t bin_axes, std::uint32_t nb) {
  return kScalarAccs + static_cast<int>(bin_axes * nb);
}

// ------------------------------------------------------------------ grid adaptation
/// adjust_axis (grid.hpp:232-297) by one warp, in shared memory.
///
/// The reference's rebinning walk is sequential; here it is reformulated so
/// every output edge is found in parallel with exactly the reference's
/// floating-point values:
///   * the running sums the walk accumulates -- cum after each old bin,
///     P[k+1] = RN(P[k] + imp[k]), and the targets T[i] = RN(T[i-1] + share)
///     -- are computed sequentially by lane 0 in the reference's order;
///   * the walk stops output i at the first k with imp[k] != 0 and
///     P[k+1] >= T[i] (or n-1).  Because T is non-decreasing, that is the
///     same k the sequential loop reaches from the previous output's k;
///   * the edge is left + width * ((T[i] - P[k]) / imp[k]) as in the reference.
/// The nextafter repair passes run sequentially only if some edge needs one.
/// scratch: kAdjustScratch * n doubles.  contrib must be finite and >= 0.
#ifdef MCB_FINISH_TIMING
// latency probe (tools/latbench.cu): %globaltimer at the finish kernel's phases
__device__ unsigned long long g_fin_times[16];
__device__ __forceinline__ unsigned long long fin_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define MCB_FIN_STAMP(i) g_fin_times[i] = fin_now()
#define MCB_FIN_STAMP_MAX(i) atomicMax(&g_fin_times[i], fin_now())
#else
#define MCB_FIN_STAMP(i)
#define MCB_FIN_STAMP_MAX(i)
#endif
#ifdef MCB_FINISH_TIMING
#define MCB_ADJ_STAMP(i) if (threadIdx.x == 0) g_fin_times[8 + (i)] = fin_now()
#else
#define MCB_ADJ_STAMP(i)
#endif

inline constexpr int kAdjustScratch = 6;  ///< doubles per bin of per-warp scratch

__device__ inline void adjust_axis_warp(double* edges_g, const double* edges_in, double lo, double hi,
                                        const double* contrib, std::uint32_t n, double alpha, double* scratch) {
  const int lane = threadIdx.x & 31;
  double* edges = scratch;
  double* smooth = scratch + n;
  double* imp = scratch + 2 * n;
  double* P = scratch + 3 * n;      // n + 1 entries: cum before bin k
  double* T = scratch + 4 * n + 1;  // n - 1 targets
  bool any_local = false;
  for (std::uint32_t i = lane; i < n; i += 32) {
    edges[i] = edges_in[i];
    any_local |= contrib[i] != 0.0;
  }
  const bool any = __any_sync(0xffffffffu, any_local);
  MCB_ADJ_STAMP(0);
  if (!any || n == 1) return;  // nothing observed: leave the axis alone
  for (std::uint32_t i = lane; i < n; i += 32) {
    double s;
    if (i == 0) s = 0.5 * (contrib[0] + contrib[1]);
    else if (i + 1 == n) s = 0.5 * (contrib[n - 2] + contrib[n - 1]);
    else s = (contrib[i - 1] + contrib[i] + contrib[i + 1]) / 3.0;
    smooth[i] = s;
  }
  __syncwarp();
  double total = 0.0;
  if (lane == 0) {
#pragma unroll 8
    for (std::uint32_t i = 0; i < n; ++i) total += smooth[i];
  }
  total = __shfl_sync(0xffffffffu, total, 0);
  MCB_ADJ_STAMP(1);
  for (std::uint32_t i = lane; i < n; i += 32) {
    const double c = smooth[i] / total;
    double r = 0.0;
    if (c == 1.0) r = 1.0;
    else if (c > 0.0) r = pow((c - 1.0) / log(c), alpha);
    imp[i] = r;
  }
  __syncwarp();
  MCB_ADJ_STAMP(2);
  if (lane == 0) {  // the reference's sequential accumulations, in its order
    // rtot (grid.hpp:252-264) and the walk's cum (grid.hpp:268-278) add the
    // same imp[] in the same order, so one pass yields both: P[n] == rtot.
    // (imp is loaded eight at a time ahead of the stores into P: the compiler
    // cannot move a load above a possibly aliasing shared store, which would
    // put a shared-memory round trip on every step of the dependent chain)
    double cum = 0.0;
    P[0] = 0.0;
    std::uint32_t k = 0;
    for (; k + 8 <= n; k += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = imp[k + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        cum += v[q];
        P[k + 1 + q] = cum;
      }
    }
    for (; k < n; ++k) {
      cum += imp[k];
      P[k + 1] = cum;
    }
    const double share = cum / static_cast<double>(n);
    double target = 0.0;
#pragma unroll 8
    for (std::uint32_t i = 0; i + 1 < n; ++i) {
      target += share;
      T[i] = target;
    }
  }
  __syncwarp();
  MCB_ADJ_STAMP(3);
  double* out = smooth;  // smooth is dead: reuse it as the output row
  for (std::uint32_t i = lane; i + 1 < n; i += 32) {
    const double t = T[i];
    // first k in [0, n-1) with imp[k] != 0 and P[k+1] >= t, else n-1: binary
    // search the monotone P for the first P[k+1] >= t, then step over
    // zero-importance bins (whose P[k+1] == P[k]).
    std::uint32_t lo_k = 0, hi_k = n - 1;
    while (lo_k < hi_k) {
      const std::uint32_t mid = (lo_k + hi_k) >> 1;
      if (P[mid + 1] < t) lo_k = mid + 1;
      else hi_k = mid;
    }
    std::uint32_t k = lo_k;
    while (k + 1 < n && (imp[k] == 0.0 || P[k + 1] < t)) ++k;
    const double left = k == 0 ? lo : edges[k - 1];
    const double width = edges[k] - left;
    out[i] = left + width * ((t - P[k]) / imp[k]);
  }
  __syncwarp();
  MCB_ADJ_STAMP(4);
  bool bad = false;
  for (std::uint32_t i = lane; i + 1 < n; i += 32) {
    const double prev = i == 0 ? lo : out[i - 1];
    const double next = i + 2 == n ? hi : out[i + 1];
    bad |= !(out[i] > prev) || !(out[i] < next);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) {  // repair passes (grid.hpp:285-294)
    double prev = lo;
    for (std::uint32_t i = 0; i + 1 < n; ++i) {
      if (!(out[i] > prev)) out[i] = nextafter(prev, INFINITY);
      prev = out[i];
    }
    double next = hi;
    for (std::uint32_t i = n - 1; i-- > 0;) {
      if (!(out[i] < next)) out[i] = nextafter(next, -INFINITY);
      next = out[i];
    }
  }
  __syncwarp();
  MCB_ADJ_STAMP(5);
  for (std::uint32_t i = lane; i < n; i += 32) edges_g[i] = i + 1 < n ? out[i] : hi;
  __syncwarp();
  MCB_ADJ_STAMP(6);
}

struct AdjustArgs {
  std::uint32_t dims, nb;
  const double* lower;
  const double* upper;
  double* edges;          ///< in/out, dims x nb
  const double* contrib;  ///< dims x nb (symmetric: row 0 only is read)
  double alpha;
  int symmetric;
  double* contrib_scratch;  ///< device dims x nb: finish-kernel staging when no contrib output is kept
};

/// Grid::adjusted / adjusted_symmetric: warp j adapts axis j (symmetric: warp
/// 0 adapts axis 0, then all warps replicate it).  `contrib` and `edges_in`
/// (the current edges, a copy of a.edges or a.edges itself) may point to
/// shared or global memory.  scratch: nwarps * kAdjustScratch * nb doubles.
__device__ inline void adjust_grid_block(const AdjustArgs& a, const double* contrib, const double* edges_in,
                                         double* scratch_all, int adj_warps) {
  const int warp = threadIdx.x >> 5;
  double* scratch = scratch_all + static_cast<std::size_t>(warp) * kAdjustScratch * a.nb;
  const std::uint32_t axes = a.symmetric ? 1u : a.dims;
  if (warp < adj_warps)
    for (std::uint32_t j = warp; j < axes; j += adj_warps)
      adjust_axis_warp(a.edges + static_cast<std::size_t>(j) * a.nb, edges_in + static_cast<std::size_t>(j) * a.nb,
                       a.lower[j], a.upper[j], contrib + static_cast<std::size_t>(j) * a.nb, a.nb, a.alpha, scratch);
  if (!a.symmetric) return;
  __syncthreads();
  const double* row0 = a.edges;
  for (std::uint32_t idx = threadIdx.x; idx < (a.dims - 1) * a.nb; idx += blockDim.x) {
    const std::uint32_t j = 1 + idx / a.nb, i = idx % a.nb;
    double* row = a.edges + static_cast<std::size_t>(j) * a.nb;
    if (a.lower[j] == a.lower[0] && a.upper[j] == a.upper[0]) {
      row[i] = row0[i];  // grid.hpp:131-135: verbatim copy keeps axes bit-identical
    } else if (i + 1 < a.nb) {
      const double range0 = a.upper[0] - a.lower[0];
      const double range = a.upper[j] - a.lower[j];
      row[i] = a.lower[j] + ((row0[i] - a.lower[0]) / range0) * range;
    } else {
      row[i] = a.upper[j];
    }
  }
}

/// Named barrier over the first `nthreads` threads of the block (a multiple of 32).
__device__ __forceinline__ void bar_sync_n(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

/// Shared-memory doubles adjust_grid_par needs beyond the staged contributions and edges.
MCB_HD std::size_t adjust_par_scratch(std::uint32_t dims, std::uint32_t nb) {
  return static_cast<std::size_t>(dims) * (kAdjustScratch * nb + 4);
}

/// Grid::adjusted (grid.hpp:232-297), every axis at once across the first
/// `nthreads` threads of the block: the element-wise steps (smoothing, the
/// importance r_i, the equal-share walk, the monotonicity check) run one
/// element per thread, and the three order-dependent sums of each axis (the
/// smoothed total, the cumulative importance, the targets) run one axis per
/// lane of warp 0 -- the reference's sequential accumulations in its order,
/// all axes in lockstep.  Bitwise the same edges as adjust_axis_warp.
/// contrib_s and edges_s are staged in shared memory; scratch:
/// adjust_par_scratch(dims, nb) doubles.
__device__ inline void adjust_grid_par(const AdjustArgs& a, const double* contrib_s, const double* edges_s,
                                       double* scratch, int nthreads) {
  const std::uint32_t n = a.nb, D = a.dims;
  const int tid = threadIdx.x;
  double* tot = scratch + static_cast<std::size_t>(D) * kAdjustScratch * n;
  double* lo = tot + D;
  double* hi = lo + D;
  int* any = reinterpret_cast<int*>(hi + D);
  int* bad = any + D;
  auto smooth_of = [&](std::uint32_t j) { return scratch + static_cast<std::size_t>(j) * kAdjustScratch * n; };
  if (tid < static_cast<int>(D)) {
    lo[tid] = a.lower[tid];
    hi[tid] = a.upper[tid];
    any[tid] = 0;
    bad[tid] = 0;
  }
  bar_sync_n(1, nthreads);
  MCB_ADJ_STAMP(0);
  const std::uint32_t total_el = D * n;
  for (std::uint32_t idx = tid; idx < total_el; idx += nthreads) {  // smoothing (grid.hpp:240-252)
    const std::uint32_t j = idx / n, i = idx - j * n;
    const double* c = contrib_s + static_cast<std::size_t>(j) * n;
    if (c[i] != 0.0) any[j] = 1;
    if (n == 1) continue;
    double v;
    if (i == 0) v = 0.5 * (c[0] + c[1]);
    else if (i + 1 == n) v = 0.5 * (c[n - 2] + c[n - 1]);
    else v = (c[i - 1] + c[i] + c[i + 1]) / 3.0;
    smooth_of(j)[i] = v;
  }
  bar_sync_n(1, nthreads);
  MCB_ADJ_STAMP(1);
  if (n == 1) return;  // a single bin has no interior edge
  if (tid < static_cast<int>(D) && any[tid]) {  // the smoothed total, in order
    const double* sm = smooth_of(tid);
    double t = 0.0;
#pragma unroll 8
    for (std::uint32_t i = 0; i < n; ++i) t += sm[i];
    tot[tid] = t;
  }
  bar_sync_n(1, nthreads);
  MCB_ADJ_STAMP(2);
  for (std::uint32_t idx = tid; idx < total_el; idx += nthreads) {  // importance (grid.hpp:255-262)
    const std::uint32_t j = idx / n, i = idx - j * n;
    if (!any[j]) continue;
    double* sm = smooth_of(j);
    const double c = sm[i] / tot[j];
    double r = 0.0;
    if (c == 1.0) r = 1.0;
    else if (c > 0.0) r = pow((c - 1.0) / log(c), a.alpha);
    sm[n + i] = r;
  }
  bar_sync_n(1, nthreads);
  MCB_ADJ_STAMP(3);
  if (tid < static_cast<int>(D) && any[tid]) {  // cumulative importance and targets, in order
    double* sm = smooth_of(tid);
    const double* imp = sm + n;
    double* P = sm + 2 * n;
    double* T = sm + 3 * n + 1;
    double cum = 0.0;
    P[0] = 0.0;
    std::uint32_t k = 0;
    for (; k + 8 <= n; k += 8) {  // loads ahead of the (possibly aliasing) stores
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = imp[k + q];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        cum += v[q];
        P[k + 1 + q] = cum;
      }
    }
    for (; k < n; ++k) {
      cum += imp[k];
      P[k + 1] = cum;
    }
    const double share = cum / static_cast<double>(n);
    double target = 0.0;
#pragma unroll 8
    for (std::uint32_t i = 0; i + 1 < n; ++i) {
      target += share;
      T[i] = target;
    }
  }
  bar_sync_n(1, nthreads);
  MCB_ADJ_STAMP(4);
  const std::uint32_t walk_el = D * (n - 1);
  for (std::uint32_t idx = tid; idx < walk_el; idx += nthreads) {  // the equal-share walk (grid.hpp:263-284)
    const std::uint32_t j = idx / (n - 1), i = idx - j * (n - 1);
    if (!any[j]) continue;
    double* sm = smooth_of(j);
    const double* imp = sm + n;
    const double* P = sm + 2 * n;
    const double t = sm[3 * n + 1 + i];
    std::uint32_t lo_k = 0, hi_k = n - 1;
    while (lo_k < hi_k) {
      const std::uint32_t mid = (lo_k + hi_k) >> 1;
      if (P[mid + 1] < t) lo_k = mid + 1;
      else hi_k = mid;
    }
    std::uint32_t k = lo_k;
    while (k + 1 < n && (imp[k] == 0.0 || P[k + 1] < t)) ++k;
    const double* ed = edges_s + static_cast<std::size_t>(j) * n;
    const double left = k == 0 ? lo[j] : ed[k - 1];
    const double width = ed[k] - left;
    sm[4 * n + i] = left + width * ((t - P[k]) / imp[k]);  // out row (after T)
  }
  bar_sync_n(1, nthreads);
  MCB_ADJ_STAMP(5);
  for (std::uint32_t idx = tid; idx < walk_el; idx += nthreads) {  // strictly increasing?
    const std::uint32_t j = idx / (n - 1), i = idx - j * (n - 1);
    if (!any[j]) continue;
    const double* out = smooth_of(j) + 4 * n;
    const double prev = i == 0 ? lo[j] : out[i - 1];
    const double next = i + 2 == n ? hi[j] : out[i + 1];
    if (!(out[i] > prev) || !(out[i] < next)) bad[j] = 1;
  }
  bar_sync_n(1, nthreads);
  if (tid < static_cast<int>(D) && any[tid] && bad[tid]) {  // repair passes (grid.hpp:285-294)
    double* out = smooth_of(tid) + 4 * n;
    double prev = lo[tid];
    for (std::uint32_t i = 0; i + 1 < n; ++i) {
      if (!(out[i] > prev)) out[i] = nextafter(prev, INFINITY);
      prev = out[i];
    }
    double next = hi[tid];
    for (std::uint32_t i = n - 1; i-- > 0;) {
      if (!(out[i] < next)) out[i] = nextafter(next, -INFINITY);
      next = out[i];
    }
  }
  bar_sync_n(1, nthreads);
  for (std::uint32_t idx = tid; idx < total_el; idx += nthreads) {
    const std::uint32_t j = idx / n, i = idx - j * n;
    if (!any[j]) continue;
    a.edges[idx] = i + 1 < n ? smooth_of(j)[4 * n + i] : hi[j];
  }
}

template <int kTag = 0>
__global__ void adjust_grid_kernel(const AdjustArgs a) {
  extern __shared__ double adj_scratch[];
  adjust_grid_block(a, a.contrib, a.edges, adj_scratch, blockDim.x >> 5);
}

#ifdef __CUDACC__
/// weighted_estimate_dev by one warp, bit-identical: the loads, reciprocals
/// and per-iteration terms are lane-parallel; the three sums are accumulated
/// by lane 0 in the reference's left-to-right order.  All lanes return the
/// results.
__device__ inline void weighted_estimate_warp(const double* est, const double* var, std::uint32_t n, double& mean,
                                              double& sigma, double& chi2_dof) {
  const int lane = threadIdx.x & 31;
  // first iteration with zero variance (driver.hpp:148-153)
  int zero_at = -1;
  for (std::uint32_t b = 0; b < n && zero_at < 0; b += 32) {
    const std::uint32_t i = b + lane;
    const unsigned z = __ballot_sync(0xffffffffu, i < n && var[i] == 0.0);
    if (z) zero_at = static_cast<int>(b) + __ffs(z) - 1;
  }
  if (zero_at >= 0) {
    mean = est[zero_at];
    sigma = 0.0;
    chi2_dof = 0.0;
    return;
  }
  double sum_w = 0.0, sum_wi = 0.0;
  for (std::uint32_t b = 0; b < n; b += 32) {
    const std::uint32_t i = b + lane;
    const double w = i < n ? 1.0 / var[i] : 0.0;
    const double wi = i < n ? w * est[i] : 0.0;
    const std::uint32_t cnt = n - b < 32 ? n - b : 32;
    for (std::uint32_t l = 0; l < cnt; ++l) {
      const double wl = __shfl_sync(0xffffffffu, w, l), wil = __shfl_sync(0xffffffffu, wi, l);
      sum_w += wl;
      sum_wi += wil;
    }
  }
  mean = sum_wi / sum_w;
  double chi2 = 0.0;
  for (std::uint32_t b = 0; b < n; b += 32) {
    const std::uint32_t i = b + lane;
    double q = 0.0;
    if (i < n) {
      const double d = est[i] - mean;
      q = d * d / var[i];
    }
    const std::uint32_t cnt = n - b < 32 ? n - b : 32;
    for (std::uint32_t l = 0; l < cnt; ++l) chi2 += __shfl_sync(0xffffffffu, q, l);
  }
  const double dof = static_cast<double>(n > 1 ? n - 1 : 1);
  sigma = 1.0 / sqrt(sum_w);
  chi2_dof = chi2 / dof;
}
#endif

/// weighted_estimate (driver.hpp:146-169) -- IEEE ops in the reference's order.
MCB_HD void weighted_estimate_dev(const double* est, const double* var, std::uint32_t n, double& mean,
                                  double& sigma, double& chi2_dof) {
  for (std::uint32_t i = 0; i < n; ++i)
    if (var[i] == 0.0) {
      mean = est[i];
      sigma = 0.0;
      chi2_dof = 0.0;
      return;
    }
  double sum_w = 0.0, sum_wi = 0.0;
  for (std::uint32_t i = 0; i < n; ++i) {
    const double w = 1.0 / var[i];
    sum_w += w;
    sum_wi += w * est[i];
  }
  mean = sum_wi / sum_w;
  double chi2 = 0.0;
  for (std::uint32_t i = 0; i < n; ++i) {
    const double d = est[i] - mean;
    chi2 += d * d / var[i];
  }
  const double dof = static_cast<double>(n > 1 ? n - 1 : 1);
  sigma = 1.0 / sqrt(sum_w);
  chi2_dof = chi2 / dof;
}

/// check_convergence (driver.hpp:173-178).
MCB_HD bool converged_dev(double est, double sigma, double chi2, double tau, double chi2max) {
  const double scale = fabs(est);
  const bool error_ok = scale < 1e-300 ? sigma <= tau : sigma / scale <= tau;
  return error_ok && chi2 <= chi2max;
}

// ------------------------------------------------------------------ finish (K3b + K4)
struct RoundArgs {
  unsigned long long* words;  ///< [exchange_accs][kXWords]; words[-2] the finite-sample count, words[-1] the
                              ///< non-finite count; zeroed by the epilogue when zero_words
  std::uint32_t dims, nb, bin_axes;
  double md2;        ///< double(m) * double(m)  (sampler.hpp:330-331)
  double* est;       ///< 1 double
  double* var;       ///< 1 double
  double* contrib;   ///< dims*nb (nullable: frozen iterations keep only shared copies)
  unsigned long long* counts;  ///< nullable: {samples, writes, overflowed addends, non-finite samples} of this
                               ///< iteration (no epilogue)
  const int* stop;
  int zero_words;  ///< leave the exchange words zeroed for the next K1 flush (integrate loop, compact exchange)
  /// The estimate, variance, contributions and header counts are already in
  /// place (the compact exchange combined every rank's rounded values,
  /// Run::combine): skip the rounding, run the epilogue only.
  int prerounded;
  const unsigned long long* wait_flags;  ///< peer-memory exchange: wait until these nwait flags reach wait_value
  int nwait;
  unsigned long long wait_value;
};

struct EpilogueArgs {
  RunState* st;
  const double* hist_est;
  const double* hist_var;
  const unsigned long long* err_key;
  std::uint32_t it;  ///< 1-based iteration just sampled
  int adjusting;
  int adj_warps;  ///< warps with adaptation scratch (set by launch_finish)
  int adj_par;    ///< 1: adjust_grid_par (all axes block-wide; set by launch_finish when it fits)
  double tau, chi2max;
  AdjustArgs adj;
  int* host_flags;  ///< nullable, host-mapped: [it-1] = 1 (continue) or 2 (stop) once this iteration finished
};

inline constexpr int kFinishThreads = 512;



/// Phase 1 (all blocks): one warp per output value -- warp-cooperative exact
/// rounding of the contributions, the estimate and the variance.
/// Phase 2 (integrate only, the LAST block to finish phase 1): failure check,
/// grid adaptation (contributions staged in shared memory), weighted
/// estimate, chi^2/dof and the convergence gate.  `counter` must be 0 at
/// launch; the last block resets it.
template <int kTag = 0>
__global__ void __launch_bounds__(kFinishThreads) finish_kernel(const RoundArgs r, const EpilogueArgs e,
                                                                int with_epilogue, unsigned int* counter) {
  extern __shared__ double fin_smem[];
  __shared__ bool is_last;
  pdl_trigger();  // the next iteration's K1 may launch (it waits for this grid)
  pdl_wait();     // K1's flushed words (or the all-reduce's) are complete
  if (blockIdx.x == 0 && threadIdx.x == 0) MCB_FIN_STAMP(0);
  const int stop0 = r.stop ? *r.stop : 0;
  __syncthreads();  // every thread reads `stop` before the last block may set it
  if (stop0) return;
  if (r.nwait) {  // peer-memory exchange: every rank's K1 has added its words into ours
    if (threadIdx.x == 0)
      for (int q = 0; q < r.nwait; ++q)
        while (ld_acquire_sys(r.wait_flags + q) < r.wait_value) __nanosleep(64);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int total = static_cast<int>(r.dims * r.nb);
  const int nbins = static_cast<int>(r.bin_axes * r.nb);
  double* contrib_out = r.contrib ? r.contrib : e.adj.contrib_scratch;

  // Each accumulator is read by exactly one warp; with zero_words that warp
  // zeroes its words right after reading them, readying the buffer for the
  // next K1 flush off the epilogue's critical path.
  auto zero_acc = [&](unsigned long long* w0, int naccs) {
    __syncwarp();
    for (int w = lane; w < naccs * kXWords; w += 32) w0[w] = 0ull;
  };
  const int c = blockIdx.x * nwarps + warp;
  if (!r.prerounded && c < total + 2) {
    if (c == total) {
      const double v = exact::warp_round_words(r.words, r.words + kXWords);
      if (lane == 0) *r.est = v;
      if (r.zero_words) zero_acc(r.words, 2);
    } else if (c == total + 1) {
      const double v = exact::warp_round_words(r.words + 2 * kXWords, nullptr) / r.md2;
      if (lane == 0) *r.var = v;
      if (r.zero_words) zero_acc(r.words + 2 * kXWords, 1);
    } else {
      unsigned long long* w = r.words + static_cast<std::size_t>(kScalarAccs + c) * kXWords;
      const double v = c < nbins ? exact::warp_round_words(w, nullptr) : 0.0;
      if (lane == 0 && contrib_out) contrib_out[c] = v;
      if (r.zero_words && c < nbins) zero_acc(w, 1);
    }
  }
  if (!with_epilogue) {
    if (r.counts && blockIdx.x == 0 && threadIdx.x == 0) {
      r.counts[0] = r.words[-2];
      r.counts[1] = r.words[-2] * r.bin_axes;
      r.counts[2] = r.words[-3];
      r.counts[3] = r.words[-1];
      if (r.zero_words) r.words[-1] = r.words[-2] = r.words[-3] = 0ull;
    }
    return;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) MCB_FIN_STAMP_MAX(1);
  if (threadIdx.x == 0) is_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (threadIdx.x == 0) *counter = 0u;
  if (threadIdx.x == 0) MCB_FIN_STAMP(2);

  // contributions and current edges staged together (one global round trip)
  double* contrib_s = fin_smem;
  double* edges_s = fin_smem + static_cast<std::size_t>(r.dims) * r.nb;
  double* scratch = edges_s + static_cast<std::size_t>(r.dims) * r.nb;
  if (e.adjusting)
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      contrib_s[i] = contrib_out[i];
      edges_s[i] = e.adj.edges[i];
    }
  __syncthreads();

  RunState* st = e.st;
  // words[-1] counts non-finite samples over every rank's slice (exchanged
  // with the words), err_key holds this rank's first one
  const unsigned long long nonfinite = r.words[-1], samples = r.words[-2], overflow = r.words[-3];
  __syncthreads();
  if (threadIdx.x == 0) {
    st->samples += samples;  // the write count the reference reports (sampler.hpp:116-119, driver.hpp:242-244)
    st->bin_writes += samples * r.bin_axes;
    if (r.zero_words) r.words[-1] = r.words[-2] = r.words[-3] = 0ull;
  }
  // NonFiniteSample (1) or an overflowed exact addend (2, ExactSum's
  // invalid_argument): abort the run (driver.hpp:231-241 propagate)
  if (*e.err_key != ~0ull || nonfinite != 0 || overflow != 0) {
    if (threadIdx.x == 0) {
      st->failed = (*e.err_key != ~0ull || nonfinite != 0) ? 1 : 2;
      st->failed_iteration = e.it;
      st->stop = 1;
      if (e.host_flags) e.host_flags[e.it - 1] = 2;
    }
    return;
  }
  if (threadIdx.x == 0) MCB_FIN_STAMP(3);
  // The weighted estimate and the convergence gate need only the history, so
  // they run on a warp the adaptation leaves idle, concurrently with it
  // (after it on warp 0 when every warp adapts, or in symmetric mode whose
  // replication step is block-wide).
  auto estimate = [&] {
    double mean, sigma, chi2;
    weighted_estimate_warp(e.hist_est, e.hist_var, e.it, mean, sigma, chi2);
    if (lane != 0) return;
    st->estimate = mean;
    st->sigma = sigma;
    st->chi2_dof = chi2;
    st->iterations_used = e.it;
    if (converged_dev(mean, sigma, chi2, e.tau, e.chi2max)) {
      st->converged = 1;
      st->stop = 1;
    }
    if (e.host_flags) e.host_flags[e.it - 1] = st->stop ? 2 : 1;
    MCB_FIN_STAMP(5);
  };
  const bool par = e.adjusting && e.adj_par;
  const bool concurrent = !e.adjusting || par || (e.adj_warps < nwarps && !e.adj.symmetric);
  const int est_warp = e.adjusting ? nwarps - 1 : 0;
  if (concurrent && warp == est_warp) {
    estimate();
    return;
  }
  if (par) adjust_grid_par(e.adj, contrib_s, edges_s, scratch, (nwarps - 1) * 32);
  else if (e.adjusting) adjust_grid_block(e.adj, contrib_s, edges_s, scratch, e.adj_warps);
  if (threadIdx.x == 0) MCB_FIN_STAMP(4);
  if (!concurrent && warp == 0) estimate();
}

// ------------------------------------------------------------------ compact exchange
/// Layout of one rank's rounded iteration in the compact exchange
/// (Run::round_local): estimate, variance (already / m^2), then four u64
/// counts stored bit for bit in doubles -- finite samples, writes, overflowed
/// addends, non-finite samples -- then the d x n_bins contributions.
inline constexpr int kCompactHead = 6;

/// Combine the G ranks' rounded iterations (gathered[r * len + i], the
/// layout above) in rank order -- sum = v_0 + v_1 + ... + v_{G-1}, the same
/// sequence of IEEE additions on every rank, so every rank holds identical
/// values -- into the run's history slot, contributions and exchange header
/// (the counts the epilogue reads).  SURVEY.md section 8(e)'s all-gather of
/// d x n_bins + 2 doubles, combined in a fixed order.
template <int kTag = 0>
__global__ void combine_kernel(const double* __restrict__ gathered, int nranks, int len, int ncontrib,
                               double* est, double* var, double* contrib, unsigned long long* header,
                               const int* stop) {
  pdl_trigger();
  pdl_wait();
  if (*stop) return;  // the run has finished; later iterations are no-ops
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    if (i >= 2 && i < kCompactHead) {  // counts: exact integer sums
      unsigned long long c = 0;
      for (int q = 0; q < nranks; ++q)
        c += static_cast<unsigned long long>(__double_as_longlong(gathered[static_cast<std::size_t>(q) * len + i]));
      if (i == 2) header[1] = c;  // finite samples   (words[-2])
      if (i == 4) header[0] = c;  // overflowed addends (words[-3])
      if (i == 5) header[2] = c;  // non-finite samples (words[-1])
      continue;
    }
    if (i >= kCompactHead && i - kCompactHead >= ncontrib) continue;  // frozen iteration: no contributions
    double acc = gathered[i];
    for (int q = 1; q < nranks; ++q) acc = __dadd_rn(acc, gathered[static_cast<std::size_t>(q) * len + i]);
    if (i == 0) *est = acc;
    else if (i == 1) *var = acc;
    else contrib[i - kCompactHead] = acc;
  }
}

// ------------------------------------------------------------------ run setup / collect
/// One launch instead of three uploads and three memsets per integrate():
/// grid edges and bounds come straight from pinned host memory (zero-copy),
/// the run state and the exchange words are zeroed, the error key set.
template <int kTag = 0>
__global__ void run_init_kernel(const double* __restrict__ staged, std::uint32_t n_edges, std::uint32_t dims,
                                double* edges, double* lower, double* upper, RunState* st, unsigned long long* err_key,
                                unsigned long long* words, std::uint32_t n_words) {
  pdl_trigger();
  pdl_wait();  // an earlier run on this context may still read the buffers written here
  const std::uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  for (std::uint32_t i = i0; i < n_edges; i += stride) edges[i] = staged[i];
  for (std::uint32_t i = i0; i < dims; i += stride) {
    lower[i] = staged[n_edges + i];
    upper[i] = staged[n_edges + dims + i];
  }
  for (std::uint32_t i = i0; i < n_words; i += stride) words[i] = 0ull;
  if (i0 == 0) {
    *st = RunState{};
    *err_key = ~0ull;
  }
}

/// One launch instead of four device-to-host copies at the end of a run: the
/// run state, the first non-finite key and the history land in pinned host
/// memory (zero-copy writes), read after one stream synchronisation.
template <int kTag = 0>
__global__ void run_collect_kernel(const RunState* st, const unsigned long long* err_key, const double* hist_est,
                                   const double* hist_var, std::uint32_t itmax, unsigned char* out) {
  pdl_trigger();
  pdl_wait();
  const std::uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  auto* hs = reinterpret_cast<double*>(out + sizeof(RunState) + 8);
  const std::uint32_t n = st->iterations_used < itmax ? st->iterations_used : itmax;
  if (i < n) {
    hs[i] = hist_est[i];
    hs[itmax + i] = hist_var[i];
  }
  if (i == 0) {
    *reinterpret_cast<RunState*>(out) = *st;
    *reinterpret_cast<unsigned long long*>(out + sizeof(RunState)) = *err_key;
  }
}

}  // namespace mcubes::gpu
