// SPDX-License-Identifier: Apache-2.0
//
// K3 (cross-block exact reduction + rounding) and K4 (on-device grid
// adaptation, inverse-variance combination, chi^2 and the convergence gate).
// Together with K1 they make one m-Cubes iteration with no host round trip.
//
// K3a sums the per-block partials into the exchange buffer (unnormalised u64
// digit sums -- integer, so exact and order-free; under multi-GPU this buffer
// is what NCCL all-reduces).  K3b rounds each accumulator to the nearest
// double exactly like ExactSum::value() (exact_sum.hpp:137-179) and produces
// v_sample's outputs (sampler.hpp:322-332).  K4 replaces Grid::adjusted /
// adjusted_symmetric (grid.hpp:104-146, 232-297), weighted_estimate and
// check_convergence (driver.hpp:146-178) and the loop bookkeeping of integrate
// (driver.hpp:227-256).
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
  int failed;  ///< a non-finite sample was seen (err_key holds the first one)
  std::uint32_t iterations_used;
  std::uint32_t failed_iteration;
  std::uint32_t pad;
  double estimate, sigma, chi2_dof;
};

/// Exchange-buffer slots: est+, est-, var, then bin_axes*nb bins.
MCB_HD int exchange_accs(std::uint32_t bin_axes, std::uint32_t nb) {
  return kScalarAccs + static_cast<int>(bin_axes * nb);
}

// ------------------------------------------------------------------ K3a
template <int kTag = 0>
__global__ void reduce_partials_kernel(const std::uint32_t* __restrict__ partials, int nblocks,
                                       int nacc, unsigned long long* __restrict__ words,
                                       const int* stop) {
  if (stop && *stop) return;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // = w * nacc + c
  if (idx >= nacc * kXWords) return;
  const int w = idx / nacc, c = idx % nacc;
  const std::size_t bstride = static_cast<std::size_t>(kXWords) * nacc;
  unsigned long long s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int b = 0;
  for (; b + 4 <= nblocks; b += 4) {
    s0 += partials[(b + 0) * bstride + idx];
    s1 += partials[(b + 1) * bstride + idx];
    s2 += partials[(b + 2) * bstride + idx];
    s3 += partials[(b + 3) * bstride + idx];
  }
  for (; b < nblocks; ++b) s0 += partials[b * bstride + idx];
  const unsigned long long s = s0 + s1 + s2 + s3;
  const int lanes = kScalarAccs * kLaneCopies;
  if (c < lanes) {
    if (s) atomicAdd(words + (c / kLaneCopies) * kXWords + w, s);  // integer: order-free
  } else {
    words[(kScalarAccs + (c - lanes)) * kXWords + w] = s;
  }
}

// ------------------------------------------------------------------ K3b
struct RoundArgs {
  const unsigned long long* words;  ///< [exchange_accs][kXWords]
  std::uint32_t dims, nb, bin_axes;
  double md2;        ///< double(m) * double(m)  (sampler.hpp:330-331)
  double* est;       ///< 1 double
  double* var;       ///< 1 double
  double* contrib;   ///< dims*nb (nullable for frozen iterations)
  const int* stop;
};

template <int kTag = 0>
__global__ void round_kernel(const RoundArgs a) {
  if (a.stop && *a.stop) return;
  const int total = static_cast<int>(a.dims * a.nb);
  const int nbins = static_cast<int>(a.bin_axes * a.nb);
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < total + 2; c += gridDim.x * blockDim.x) {
    if (c == total) {
      *a.est = exact::round_words(a.words, a.words + kXWords);
    } else if (c == total + 1) {
      *a.var = exact::round_words(a.words + 2 * kXWords, nullptr) / a.md2;
    } else if (a.contrib) {
      a.contrib[c] = c < nbins ? exact::round_words(a.words + (kScalarAccs + c) * kXWords, nullptr) : 0.0;
    }
  }
}

// ------------------------------------------------------------------ K4 pieces
/// adjust_axis (grid.hpp:232-297) by one warp: the element-wise steps
/// (smoothing, ((c-1)/ln c)^alpha) run lane-parallel, every running sum and
/// the rebinning walk run on lane 0 in the reference's order.
/// scratch: 3*n doubles.  contrib must be finite and >= 0 (checked by callers).
__device__ inline void adjust_axis_warp(double* edges, double lo, double hi, const double* contrib,
                                        std::uint32_t n, double alpha, double* scratch) {
  const int lane = threadIdx.x & 31;
  bool any_local = false;
  for (std::uint32_t i = lane; i < n; i += 32) any_local |= contrib[i] != 0.0;
  const bool any = __any_sync(0xffffffffu, any_local);
  if (!any || n == 1) return;
  double* smooth = scratch;
  double* imp = scratch + n;
  double* out = scratch + 2 * n;
  for (std::uint32_t i = lane; i < n; i += 32) {
    double s;
    if (i == 0) s = 0.5 * (contrib[0] + contrib[1]);
    else if (i + 1 == n) s = 0.5 * (contrib[n - 2] + contrib[n - 1]);
    else s = (contrib[i - 1] + contrib[i] + contrib[i + 1]) / 3.0;
    smooth[i] = s;
  }
  __syncwarp();
  double total = 0.0;
  if (lane == 0)
    for (std::uint32_t i = 0; i < n; ++i) total += smooth[i];
  total = __shfl_sync(0xffffffffu, total, 0);
  for (std::uint32_t i = lane; i < n; i += 32) {
    const double c = smooth[i] / total;
    double r = 0.0;
    if (c == 1.0) r = 1.0;
    else if (c > 0.0) r = pow((c - 1.0) / log(c), alpha);
    imp[i] = r;
  }
  __syncwarp();
  if (lane == 0) {
    double rtot = 0.0;
    for (std::uint32_t i = 0; i < n; ++i) rtot += imp[i];
    const double share = rtot / static_cast<double>(n);
    out[n - 1] = hi;
    double target = 0.0, cum = 0.0;
    std::uint32_t k = 0;
    for (std::uint32_t i = 0; i + 1 < n; ++i) {
      target += share;
      while (k + 1 < n && (imp[k] == 0.0 || cum + imp[k] < target)) {
        cum += imp[k];
        ++k;
      }
      const double left = k == 0 ? lo : edges[k - 1];
      const double width = edges[k] - left;
      out[i] = left + width * ((target - cum) / imp[k]);
    }
    double prev = lo;  // repair passes (grid.hpp:285-294)
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
  for (std::uint32_t i = lane; i < n; i += 32) edges[i] = out[i];
  __syncwarp();
}

struct AdjustArgs {
  std::uint32_t dims, nb;
  const double* lower;
  const double* upper;
  double* edges;          ///< in/out, dims x nb
  const double* contrib;  ///< dims x nb (symmetric: row 0 only is read)
  double alpha;
  int symmetric;
};

/// Grid::adjusted / adjusted_symmetric on device: warp j adapts axis j
/// (symmetric: warp 0 adapts axis 0, then all warps replicate it).
/// Dynamic smem: blockDim/32 * 3*nb doubles.
__device__ inline void adjust_grid_block(const AdjustArgs& a) {
  extern __shared__ double adj_scratch[];
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double* scratch = adj_scratch + static_cast<std::size_t>(warp) * 3 * a.nb;
  const std::uint32_t axes = a.symmetric ? 1u : a.dims;
  for (std::uint32_t j = warp; j < axes; j += nwarps)
    adjust_axis_warp(a.edges + static_cast<std::size_t>(j) * a.nb, a.lower[j], a.upper[j],
                     a.contrib + static_cast<std::size_t>(j) * a.nb, a.nb, a.alpha, scratch);
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

template <int kTag = 0>
__global__ void adjust_grid_kernel(const AdjustArgs a) { adjust_grid_block(a); }

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

struct EpilogueArgs {
  RunState* st;
  const double* hist_est;
  const double* hist_var;
  const unsigned long long* err_key;
  std::uint32_t it;  ///< 1-based iteration just sampled
  int adjusting;
  double tau, chi2max;
  AdjustArgs adj;
};

/// K4: one block; runs after K3b of iteration `it`.
template <int kTag = 0>
__global__ void epilogue_kernel(const EpilogueArgs a) {
  RunState* st = a.st;
  const int stop0 = st->stop;
  __syncthreads();  // every thread reads `stop` before thread 0 may set it
  if (stop0) return;
  if (*a.err_key != ~0ull) {  // NonFiniteSample: abort the run (driver.hpp:231-241 propagate)
    if (threadIdx.x == 0) {
      st->failed = 1;
      st->failed_iteration = a.it;
      st->stop = 1;
    }
    return;
  }
  if (a.adjusting) adjust_grid_block(a.adj);
  if (threadIdx.x == 0) {
    double mean, sigma, chi2;
    weighted_estimate_dev(a.hist_est, a.hist_var, a.it, mean, sigma, chi2);
    st->estimate = mean;
    st->sigma = sigma;
    st->chi2_dof = chi2;
    st->iterations_used = a.it;
    if (converged_dev(mean, sigma, chi2, a.tau, a.chi2max)) {
      st->converged = 1;
      st->stop = 1;
    }
  }
}

}  // namespace mcubes::gpu
