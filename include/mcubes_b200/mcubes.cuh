// SPDX-License-Identifier: Apache-2.0
//
// mcubes_b200: the B200-native drop-in for the reference's header-only
// m-Cubes API (proj/include/mcubes/*.hpp).  Same names, fields, layouts and
// error behaviour in namespace `mcubes`:
//
//   RunConfig, setup, set_batch_size, weighted_estimate, check_convergence,
//   integrate(f, cfg, observer) -> IntegrationResult          (driver.hpp)
//   v_sample, v_sample_no_adjust, SampleOutcome, BinUpdate,
//   NonFiniteSample                                            (sampler.hpp)
//   Grid (transform, adjusted, adjusted_symmetric, write/read) (grid.hpp)
//   BinAccumulator                                             (accumulators.hpp)
//
// The integrand is any trivially copyable functor whose
// `double operator()(std::span<const double>) const` is __host__ __device__
// (gpu::DeviceIntegrand).  The sampling iteration, its exact reductions, the
// grid adaptation and the weighted combination all run on the GPU; compile the
// including translation unit with nvcc -std=c++20 --expt-relaxed-constexpr
// -fmad=false (the analogue of the reference's -ffp-contract=off) for
// bitwise parity with the CPU reference on +-*/ integrands.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <functional>
#include <iomanip>
#include <istream>
#include <limits>
#include <map>
#include <memory>
#include <optional>
#include <ostream>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <utility>
#include <vector>

#include "engine.cuh"
#if MCB_NVTX
#include <nvtx3/nvToolsExt.h>
#endif

namespace mcubes {

// =============================================================== accumulators
/// Per-axis, per-bin totals of (f(x)*J)^2 (accumulators.hpp:18-56).
class BinAccumulator {
 public:
  BinAccumulator(std::uint32_t dims, std::uint32_t n_bins) : dims_(dims), n_bins_(n_bins) {
    if (dims == 0) invalid("dims must be >= 1");
    if (n_bins == 0) invalid("n_bins must be >= 1");
    values_.assign(cells(), 0.0);
  }
  /// The GPU's result: device-rounded cell values and the device-counted writes.
  BinAccumulator(std::uint32_t dims, std::uint32_t n_bins, std::vector<double> values, std::uint64_t writes)
      : dims_(dims), n_bins_(n_bins), values_(std::move(values)), writes_(writes) {
    if (values_.size() != cells()) invalid("value matrix has wrong shape");
  }
  void deposit(std::uint32_t axis, std::uint32_t bin, double v) {
    values_[cell(axis, bin)] += v;
    writes_ += 1;
  }
  [[nodiscard]] double at(std::uint32_t axis, std::uint32_t bin) const { return values_[cell(axis, bin)]; }
  [[nodiscard]] std::span<const double> axis_row(std::uint32_t axis) const {
    if (axis >= dims_) invalid("axis out of range");
    return std::span<const double>(values_).subspan(cell(axis, 0), n_bins_);
  }
  [[nodiscard]] const std::vector<double>& values() const { return values_; }
  [[nodiscard]] std::uint32_t dims() const { return dims_; }
  [[nodiscard]] std::uint32_t n_bins() const { return n_bins_; }
  [[nodiscard]] std::uint64_t writes() const { return writes_; }

 private:
  [[noreturn]] static void invalid(const char* what) {
    throw std::invalid_argument(std::string("BinAccumulator: ") + what);
  }
  [[nodiscard]] std::size_t cells() const { return std::size_t{dims_} * n_bins_; }
  [[nodiscard]] std::size_t cell(std::uint32_t axis, std::uint32_t bin) const {
    return std::size_t{axis} * n_bins_ + bin;  // axis-major, as grid.hpp:303 and sampler.hpp:107-124
  }
  std::uint32_t dims_;
  std::uint32_t n_bins_;
  std::vector<double> values_;
  std::uint64_t writes_ = 0;
};

/// Thrown when f(x)*jacobian is not finite; carries the offending point
/// (sampler.hpp:31-48).  The GPU reports the first failure in serial
/// (cube, sample) order -- what the serial oracle would throw.
class NonFiniteSample : public std::runtime_error {
 public:
  NonFiniteSample(std::vector<double> x, double fx)
      : std::runtime_error(describe(x, fx)), point_(std::move(x)), value_(fx) {}
  [[nodiscard]] const std::vector<double>& point() const { return point_; }
  [[nodiscard]] double value() const { return value_; }

 private:
  static std::string describe(const std::vector<double>& x, double fx) {  // sampler.hpp:31-48's message
    std::ostringstream msg;
    msg << "integrand produced non-finite value " << fx << " at x = (";
    const char* sep = "";
    for (const double xj : x) {
      msg << sep << xj;
      sep = ", ";
    }
    msg << ')';
    return msg.str();
  }
  std::vector<double> point_;
  double value_;
};

enum class BinUpdate : std::uint8_t { all_axes, axis0_only };

struct SampleOutcome {
  double raw_estimate;
  double raw_variance;
  BinAccumulator contributions;
};

struct EstimateVariance {
  double raw_estimate;
  double raw_variance;
};

namespace gpu {

/// NVTX range for profilers (nsys / ncu --nvtx): the whole integrate() and
/// each enqueued iteration.  No-ops unless a tool is attached; MCB_NVTX=0 at
/// build time removes them.
struct NvtxRange {
  explicit NvtxRange(const char* name) {
#if MCB_NVTX
    nvtxRangePushA(name);
#else
    (void)name;
#endif
  }
  ~NvtxRange() {
#if MCB_NVTX
    nvtxRangePop();
#endif
  }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


/// One context per (host thread, device), created on first use.
inline Context& default_context() {
  int dev = 0;
  MCB_CUDA(cudaGetDevice(&dev));
  thread_local std::map<int, std::unique_ptr<Context>> ctxs;
  auto& c = ctxs[dev];
  if (!c) c = std::make_unique<Context>(dev);
  return *c;
}

/// Type-erased launchers of one integrand: lets the (non-template)
/// orchestration below serve every functor type.
struct IntegrandOps {
  std::function<Launch(Context&, const Shape&, std::uint32_t, std::uint64_t, std::uint64_t, std::uint64_t,
                       const int*, unsigned long long*, unsigned long long*)>  // ..., stop, err_key, exchange words
      k1;
  std::function<void(Context&, const Shape&, std::uint64_t, std::uint64_t, std::uint64_t, double*, double*)> point;
  RngKind rng = RngKind::compat;
};

template <DeviceIntegrand F, RngKind R = RngKind::compat>
IntegrandOps make_ops(const F& f) {
  IntegrandOps ops;
  ops.k1 = [f](Context& c, const Shape& sh, std::uint32_t ba, std::uint64_t root, std::uint64_t n0,
               std::uint64_t n1, const int* stop, unsigned long long* err, unsigned long long* words) {
    return dispatch_k1<F, R>(c, f, sh, ba, root, n0, n1, stop, err, words);
  };
  ops.point = [f](Context& c, const Shape& sh, std::uint64_t root, std::uint64_t t, std::uint64_t k, double* x,
                  double* fx) { dispatch_point<F, R>(c, f, sh, root, t, k, x, fx); };
  ops.rng = R;
  return ops;
}

/// make_ops for a stream chosen at run time.
template <DeviceIntegrand F>
IntegrandOps make_ops_for(const F& f, RngKind r) {
  switch (r) {
    case RngKind::philox: return make_ops<F, RngKind::philox>(f);
    case RngKind::philox_exact: return make_ops<F, RngKind::philox_exact>(f);
    default: return make_ops<F, RngKind::compat>(f);
  }
}

/// Per-iteration key: the reference's iteration root (rng.hpp:47-50); the
/// Philox stream uses the same 64-bit value as its key.
inline std::uint64_t iteration_key(std::uint64_t seed, std::uint64_t it) { return rng::iteration_root(seed, it); }

inline void upload(Context& ctx, DevBuf<double>& buf, const double* host, std::size_t n) {
  MCB_CUDA(cudaMemcpyAsync(buf.ensure(n), host, sizeof(double) * n, cudaMemcpyHostToDevice, ctx.stream()));
}

inline void download(Context& ctx, double* host, const double* dev, std::size_t n) {
  MCB_CUDA(cudaMemcpyAsync(host, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream()));
}

[[noreturn]] inline void throw_nonfinite(Context& ctx, const IntegrandOps& ops, const Shape& sh,
                                         std::uint64_t iter_root, unsigned long long key) {
  double* dx = ctx.point.ensure(sh.dims + 1);
  ops.point(ctx, sh, iter_root, key / sh.p, key % sh.p, dx, dx + sh.dims);
  std::vector<double> hx(sh.dims + 1);
  download(ctx, hx.data(), dx, sh.dims + 1);
  ctx.sync();
  const double fx = hx[sh.dims];
  hx.resize(sh.dims);
  throw NonFiniteSample(std::move(hx), fx);
}

/// An exact addend ((f J)^2, a cube's sum or variance) overflowed to inf:
/// the reference's ExactSum::add throws this (exact_sum.hpp:34).
[[noreturn]] inline void throw_overflow() { throw std::invalid_argument("ExactSum: non-finite addend"); }

}  // namespace gpu

// ====================================================================== grid
/// Per-axis importance grid (grid.hpp:19-176): right edges only, d x n_bins
/// row-major, implicit left edge at `lower`.
class Grid {
 public:
  /// The uniform grid (grid.hpp:30-50): n_bins equal bins per axis, edge i
  /// at lower + (i + 1) * width, the last edge exactly the upper bound.
  Grid(std::uint32_t dims, std::uint32_t n_bins, std::span<const double> lower, std::span<const double> upper)
      : dims_(dims), n_bins_(n_bins), lower_(lower.begin(), lower.end()), upper_(upper.begin(), upper.end()) {
    const auto need = [](bool ok, const char* what) {
      if (!ok) throw std::invalid_argument(std::string("Grid: ") + what);
    };
    need(dims_ != 0, "dims must be >= 1");
    need(n_bins_ >= 2, "n_bins must be >= 2");
    need(lower_.size() == dims_ && upper_.size() == dims_, "bounds must have one entry per axis");
    for (std::uint32_t j = 0; j < dims_; ++j)
      need(lower_[j] < upper_[j] && std::isfinite(lower_[j]) && std::isfinite(upper_[j]),
           "requires finite lower < upper on every axis");
    edges_.reserve(std::size_t{dims_} * n_bins_);
    for (std::uint32_t j = 0; j < dims_; ++j) {
      const double step = (upper_[j] - lower_[j]) / static_cast<double>(n_bins_);
      for (std::uint32_t k = 1; k < n_bins_; ++k) edges_.push_back(lower_[j] + static_cast<double>(k) * step);
      edges_.push_back(upper_[j]);
    }
  }

  /// From raw edges (validated like Grid::read, grid.hpp:161-175).
  static Grid from_edges(std::uint32_t dims, std::uint32_t n_bins, std::vector<double> lower,
                         std::vector<double> upper, std::vector<double> edges) {
    if (dims == 0 || n_bins < 2) throw std::invalid_argument("Grid::read: malformed header");
    if (lower.size() != dims || upper.size() != dims || edges.size() != std::size_t{dims} * n_bins)
      throw std::invalid_argument("Grid: bounds must have one entry per axis");
    return Grid(dims, n_bins, std::move(lower), std::move(upper), std::move(edges));
  }

  [[nodiscard]] std::uint32_t dims() const { return dims_; }
  [[nodiscard]] std::uint32_t n_bins() const { return n_bins_; }
  [[nodiscard]] double lower(std::uint32_t axis) const { return lower_[axis]; }
  [[nodiscard]] double upper(std::uint32_t axis) const { return upper_[axis]; }
  [[nodiscard]] std::span<const double> edges(std::uint32_t axis) const {
    return {edges_.data() + std::size_t{axis} * n_bins_, n_bins_};
  }
  [[nodiscard]] const std::vector<double>& raw_edges() const { return edges_; }
  [[nodiscard]] const std::vector<double>& lowers() const { return lower_; }
  [[nodiscard]] const std::vector<double>& uppers() const { return upper_; }

  /// grid.hpp:61-67: the bin of unit coordinate u, clamped to [0, n_bins - 1]
  /// (u <= 0 or NaN -> 0).
  [[nodiscard]] std::uint32_t bin_index(double u) const { return clamp_bin(u * static_cast<double>(n_bins_)); }
  void bin_indices(std::span<const double> u, std::span<std::uint32_t> out) const {
    for (std::uint32_t j = 0; j < dims_; ++j) out[j] = bin_index(u[j]);
  }

  /// Host form of the map the sampling kernel applies (grid.hpp:204-224).
  double transform(std::span<const double> u, std::span<double> x) const { return transform_impl<false>(u, x, {}); }
  double transform(std::span<const double> u, std::span<double> x, std::span<std::uint32_t> bins) const {
    return transform_impl<true>(u, x, bins);
  }

  /// One adaptation step (grid.hpp:104-114), computed on the GPU.
  [[nodiscard]] Grid adjusted(const BinAccumulator& contributions, double alpha) const {
    if (contributions.dims() != dims_ || contributions.n_bins() != n_bins_)
      throw std::invalid_argument("Grid::adjusted: contribution shape mismatch");
    require_valid_alpha(alpha);
    check_contrib(contributions.values());
    return adjust_on_device(contributions.values(), alpha, false);
  }

  /// Symmetric-integrand adaptation (grid.hpp:122-146), computed on the GPU.
  [[nodiscard]] Grid adjusted_symmetric(std::span<const double> axis0_contributions, double alpha) const {
    if (axis0_contributions.size() != n_bins_)
      throw std::invalid_argument("Grid::adjusted_symmetric: contribution shape mismatch");
    require_valid_alpha(alpha);
    std::vector<double> c(std::size_t{dims_} * n_bins_, 0.0);
    std::copy(axis0_contributions.begin(), axis0_contributions.end(), c.begin());
    check_contrib(c);
    return adjust_on_device(c, alpha, true);
  }

  /// Plain-text checkpoint (grid.hpp:148-158): a "dims n_bins" header, then
  /// one line per axis -- lower, upper and the n_bins right edges -- at 17
  /// significant digits, which round-trip every double.
  void write(std::ostream& os) const {
    const std::streamsize saved = os.precision(17);
    os << dims_ << ' ' << n_bins_ << '\n';
    for (std::uint32_t j = 0; j < dims_; ++j) {
      std::span<const double> row = edges(j);
      os << lower_[j] << ' ' << upper_[j];
      for (std::size_t k = 0; k < row.size(); ++k) os << ' ' << row[k];
      os << '\n';
    }
    os.precision(saved);
  }

  /// grid.hpp:161-174: parses write()'s format; a truncated or non-numeric
  /// header, bound pair or edge list raises invalid_argument, as the reference.
  static Grid read(std::istream& is) {
    const auto fail = [](const char* what) { throw std::invalid_argument(std::string("Grid::read: ") + what); };
    std::uint32_t dims = 0, n_bins = 0;
    is >> dims >> n_bins;
    if (!is || dims == 0 || n_bins < 2) fail("malformed header");
    std::vector<double> lower(dims), upper(dims), edges;
    edges.reserve(std::size_t{dims} * n_bins);
    for (std::uint32_t j = 0; j < dims; ++j) {
      is >> lower[j] >> upper[j];
      if (!is) fail("malformed axis bounds");
      for (std::uint32_t k = 0; k < n_bins; ++k) {
        double e;
        if (!(is >> e)) fail("malformed edge list");
        edges.push_back(e);
      }
    }
    return Grid(dims, n_bins, std::move(lower), std::move(upper), std::move(edges));
  }

  friend bool operator==(const Grid&, const Grid&) = default;

 private:
  Grid(std::uint32_t dims, std::uint32_t n_bins, std::vector<double> lower, std::vector<double> upper,
       std::vector<double> raw_edges)
      : dims_(dims), n_bins_(n_bins), lower_(std::move(lower)), upper_(std::move(upper)), edges_(std::move(raw_edges)) {
    // grid.hpp:61-67 invariants of a checkpointed grid: per axis, lower < e_0 < ... < e_{n-1} = upper
    for (std::uint32_t j = 0; j < dims_; ++j) {
      if (!(lower_[j] < upper_[j])) throw std::invalid_argument("Grid: requires lower < upper on every axis");
      const std::span<const double> row = edges(j);
      for (std::size_t k = 0; k < row.size(); ++k)
        if (!(row[k] > (k ? row[k - 1] : lower_[j]))) throw std::invalid_argument("Grid: edges must increase strictly");
      if (row[row.size() - 1] != upper_[j]) throw std::invalid_argument("Grid: last edge must equal the upper bound");
    }
  }

  static void require_valid_alpha(double alpha) {
    if (!(alpha >= 0.0) || !std::isfinite(alpha))
      throw std::invalid_argument("Grid: damping exponent alpha must be finite and >= 0");
  }
  static void check_contrib(const std::vector<double>& c) {
    for (const double v : c)
      if (v < 0.0 || !std::isfinite(v)) throw std::invalid_argument("Grid: contributions must be finite and >= 0");
  }

  Grid adjust_on_device(const std::vector<double>& contrib, double alpha, bool symmetric) const {
    gpu::Context& ctx = gpu::default_context();
    ctx.activate();
    const std::size_t n = std::size_t{dims_} * n_bins_;
    gpu::upload(ctx, ctx.edges, edges_.data(), n);
    gpu::upload(ctx, ctx.contrib, contrib.data(), n);
    gpu::upload(ctx, ctx.lower, lower_.data(), dims_);
    gpu::upload(ctx, ctx.upper, upper_.data(), dims_);
    gpu::AdjustArgs a{dims_, n_bins_, ctx.lower.get(), ctx.upper.get(), ctx.edges.get(), ctx.contrib.get(), alpha,
                      symmetric ? 1 : 0};
    gpu::launch_adjust(ctx, a);
    Grid g(*this);
    gpu::download(ctx, g.edges_.data(), ctx.edges.get(), n);
    ctx.sync();
    return g;
  }

  /// Bin of the bin coordinate z = u * n_bins: floor(z) inside, 0 for z <= 0
  /// (or NaN), n_bins - 1 for z >= n_bins (grid.hpp:61-67, 209-213).
  [[nodiscard]] std::uint32_t clamp_bin(double z) const {
    if (z >= static_cast<double>(n_bins_)) return n_bins_ - 1;
    return z > 0.0 ? static_cast<std::uint32_t>(z) : 0u;
  }

  /// The host form of the map K1 applies (grid.hpp:204-224), operation for
  /// operation the same IEEE arithmetic: x = left + (z - bin) * width and the
  /// jacobian as the running product of n_bins * width, axis by axis.
  template <bool kWantBins>
  double transform_impl(std::span<const double> u, std::span<double> x, std::span<std::uint32_t> bins) const {
    const double nb = static_cast<double>(n_bins_);
    double jac = 1.0;
    for (std::uint32_t j = 0; j < dims_; ++j) {
      const double z = u[j] * nb;
      const std::uint32_t b = clamp_bin(z);
      const std::span<const double> row = edges(j);
      const double left = b ? row[b - 1] : lower_[j];
      const double width = row[b] - left;
      x[j] = left + (z - static_cast<double>(b)) * width;
      jac *= nb * width;
      if constexpr (kWantBins) bins[j] = b;
    }
    return jac;
  }

  std::uint32_t dims_;
  std::uint32_t n_bins_;
  std::vector<double> lower_;
  std::vector<double> upper_;
  std::vector<double> edges_;
};

// =================================================================== sampler
/// Unit-space position of a point in cube t (sampler.hpp:75-87).
inline void cube_unit_point(std::uint64_t t, std::uint64_t g, std::uint32_t dims, std::span<const double> r,
                            std::span<double> u) {
  const auto fail = [](const char* what) { throw std::invalid_argument(std::string("cube_unit_point: ") + what); };
  if (g == 0) fail("g must be >= 1");
  if (r.size() != dims || u.size() != dims) fail("r and u must have one entry per axis");
  // t in base g, axis 0 the fastest digit: u_j = (digit_j + r_j) / g
  std::uint64_t rest = t;
  for (std::uint32_t j = 0; j < dims; ++j, rest /= g) {
    const std::uint64_t digit = rest % g;
    u[j] = (static_cast<double>(digit) + r[j]) / static_cast<double>(g);
  }
  if (rest != 0) fail("cube index out of range");
}

namespace gpu {

/// One iteration on the GPU for a host grid.  bin_axes: 0 frozen, 1 axis0, d all.
struct SampleResult {
  double est = 0, var = 0;
  std::uint64_t samples = 0;  ///< finite samples taken, counted on the device
  std::uint64_t writes = 0;   ///< contribution deposits (samples * bin_axes; 0 when frozen)
  std::vector<double> contrib;
};

inline SampleResult sample_once(Context& ctx, const IntegrandOps& ops, const Grid& grid, std::uint64_t m,
                                std::uint64_t s, std::uint64_t p, std::uint64_t seed, std::uint64_t iteration,
                                std::uint32_t bin_axes) {
  ctx.activate();
  const Shape sh = make_shape(grid.dims(), grid.n_bins(), m, s, p);
  const std::size_t n = std::size_t{grid.dims()} * grid.n_bins();
  upload(ctx, ctx.edges, grid.raw_edges().data(), n);
  upload(ctx, ctx.lower, grid.lowers().data(), grid.dims());
  ctx.grid_edges = ctx.edges.get();
  ctx.grid_lower = ctx.lower.get();
  unsigned long long* err = ctx.err_key.ensure(1);
  MCB_CUDA(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), ctx.stream()));
  const std::uint64_t root = iteration_key(seed, iteration);
  // exchange buffer: the sample and non-finite count words, then the accumulator words
  const std::size_t nwords = kXHeader + static_cast<std::size_t>(exchange_accs(bin_axes, sh.nb)) * kXWords;
  unsigned long long* xbuf = ctx.words.ensure(nwords);
  MCB_CUDA(cudaMemsetAsync(xbuf, 0, sizeof(unsigned long long) * nwords, ctx.stream()));
  unsigned long long* words = xbuf + kXHeader;
  (void)ops.k1(ctx, sh, bin_axes, root, 0, m, nullptr, err, words);  // K1 flushes straight into the words
  double* sc = ctx.scalars.ensure(6);  // est, var, then the {samples, writes, overflowed, non-finite} counts
  auto* counts = reinterpret_cast<unsigned long long*>(sc + 2);
  double* contrib = bin_axes ? ctx.contrib.ensure(n) : nullptr;
  launch_finish(ctx, sh, bin_axes, words, sc, sc + 1, contrib, nullptr, nullptr, false, counts);
  // results back through pinned staging
  auto* pin = reinterpret_cast<double*>(ctx.pinned());
  const std::size_t nd = 5 + (bin_axes ? n : 0);
  if ((nd + 1) * sizeof(double) > Context::kPinnedBytes) throw std::invalid_argument("grid too large");
  MCB_CUDA(cudaMemcpyAsync(pin, sc, sizeof(double) * 5, cudaMemcpyDeviceToHost, ctx.stream()));
  if (bin_axes) MCB_CUDA(cudaMemcpyAsync(pin + 5, contrib, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx.stream()));
  MCB_CUDA(cudaMemcpyAsync(pin + nd, err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx.stream()));
  ctx.sync();
  unsigned long long key;
  std::memcpy(&key, pin + nd, sizeof key);
  if (key != ~0ull) throw_nonfinite(ctx, ops, sh, root, key);
  unsigned long long overflow;
  std::memcpy(&overflow, pin + 4, 8);
  if (overflow) throw_overflow();
  SampleResult r;
  r.est = pin[0];
  r.var = pin[1];
  std::memcpy(&r.samples, pin + 2, 8);
  std::memcpy(&r.writes, pin + 3, 8);
  if (bin_axes) r.contrib.assign(pin + 5, pin + 5 + n);
  return r;
}

}  // namespace gpu

/// One adjusting iteration (sampler.hpp:312-333), on the GPU.  s and
/// max_threads are validated/ignored exactly as the reference's outputs are
/// invariant to them.
template <gpu::DeviceIntegrand F>
SampleOutcome v_sample(const F& f, const Grid& grid, std::uint64_t m, std::uint64_t s, std::uint64_t p,
                       std::uint64_t seed, std::uint64_t iteration, BinUpdate mode = BinUpdate::all_axes,
                       unsigned max_threads = 0) {
  (void)max_threads;
  const std::uint32_t bin_axes = mode == BinUpdate::all_axes ? grid.dims() : 1;
  auto r = gpu::sample_once(gpu::default_context(), gpu::make_ops(f), grid, m, s, p, seed, iteration, bin_axes);
  return {r.est, r.var, BinAccumulator(grid.dims(), grid.n_bins(), std::move(r.contrib), r.writes)};
}

/// Frozen-grid iteration (sampler.hpp:339-349), on the GPU.
template <gpu::DeviceIntegrand F>
EstimateVariance v_sample_no_adjust(const F& f, const Grid& grid, std::uint64_t m, std::uint64_t s, std::uint64_t p,
                                    std::uint64_t seed, std::uint64_t iteration, unsigned max_threads = 0) {
  (void)max_threads;
  auto r = gpu::sample_once(gpu::default_context(), gpu::make_ops(f), grid, m, s, p, seed, iteration, 0);
  return {r.est, r.var};
}

// ==================================================================== driver
enum class Variant : std::uint8_t { mcubes, mcubes1d };

[[nodiscard]] inline std::string_view variant_name(Variant v) { return v == Variant::mcubes ? "mcubes" : "mcubes1d"; }
[[nodiscard]] inline std::optional<Variant> parse_variant(std::string_view s) {
  if (s == "mcubes") return Variant::mcubes;
  if (s == "mcubes1d") return Variant::mcubes1d;
  return std::nullopt;
}

/// driver.hpp:37-71, plus B200 fields at the end (aggregate order preserved).
struct RunConfig {
  std::uint32_t dims = 0;
  std::uint32_t n_bins = 50;
  std::uint64_t maxcalls = 0;
  std::uint32_t itmax = 15;
  std::uint32_t ita = 10;
  double tau_rel = 1e-3;
  double alpha = 1.5;
  double chi2_dof_max = 1.5;
  std::uint64_t seed = 0;
  Variant variant = Variant::mcubes;
  std::vector<double> lower;
  std::vector<double> upper;
  unsigned workers = 0;  ///< accepted for source compatibility; the GPU path ignores it
  gpu::RngKind rng = gpu::RngKind::compat;

  /// driver.hpp:52-70: the same checks, in the same order, with the same
  /// messages (the first failing one is reported).
  void validate() const {
    const auto need = [](bool ok, const char* what) {
      if (!ok) throw std::invalid_argument(std::string("RunConfig: ") + what);
    };
    need(dims >= 1, "dims must be >= 1");
    need(n_bins >= 2, "n_bins must be >= 2");
    need(dims < 63 && maxcalls >= (std::uint64_t{2} << dims), "maxcalls must be >= 2*2^dims");
    need(tau_rel > 0.0 && tau_rel < 1.0, "tau_rel must lie in (0, 1)");  // NaN fails both
    need(itmax >= 1, "itmax must be >= 1");
    need(ita <= itmax, "ita must not exceed itmax");
    need(alpha >= 0.0 && std::isfinite(alpha), "alpha must be finite and >= 0");
    need(chi2_dof_max > 0.0, "chi2_dof_max must be positive");
    need(lower.size() == dims && upper.size() == dims, "bounds must have one entry per axis");
    bool box_ok = true;
    for (std::uint32_t j = 0; j < dims && box_ok; ++j)
      box_ok = std::isfinite(lower[j]) && std::isfinite(upper[j]) && lower[j] < upper[j];
    need(box_ok, "requires finite lower < upper on every axis");
  }
};

struct SetupParams {
  std::uint64_t g;
  std::uint64_t m;
  std::uint64_t p;
  std::uint64_t s;
};

/// driver.hpp:82-87: about 32 batches per worker, at least one cube each.
[[nodiscard]] inline std::uint64_t set_batch_size(std::uint64_t m, unsigned workers) {
  if (m == 0) throw std::invalid_argument("set_batch_size: m must be >= 1");
  if (workers == 0) throw std::invalid_argument("set_batch_size: workers must be >= 1");
  const std::uint64_t batches = std::uint64_t{workers} * 32;
  return (m - 1) / batches + 1;  // ceil(m / batches) >= 1
}

namespace detail {
/// The largest g >= 1 with 2 g^d <= maxcalls (1 if there is none), the value
/// of driver.hpp:93-108, found by an exact integer bisection.
inline std::uint64_t intervals_per_axis(std::uint64_t maxcalls, std::uint32_t d) {
  const auto fits = [&](std::uint64_t g) {  // 2 g^d <= maxcalls without overflow
    unsigned __int128 v = 2;
    for (std::uint32_t i = 0; i < d && v <= maxcalls; ++i) v *= g;
    return v <= maxcalls;
  };
  std::uint64_t good = 1, bad = 2;  // fits(good) unless good == 1; !fits(bad) once found
  while (fits(bad)) {
    good = bad;
    bad *= 2;
  }
  while (bad - good > 1) {
    const std::uint64_t mid = good + (bad - good) / 2;
    (fits(mid) ? good : bad) = mid;
  }
  return good;
}
}  // namespace detail

/// driver.hpp:114-123: g intervals per axis, m = g^d sub-cubes, p = maxcalls / m
/// samples per cube (at least 2, so each cube has a variance), batch size.
[[nodiscard]] inline SetupParams setup(const RunConfig& cfg) {
  cfg.validate();
  SetupParams sp{};
  sp.g = detail::intervals_per_axis(cfg.maxcalls, cfg.dims);
  sp.m = 1;
  for (std::uint32_t j = 0; j < cfg.dims; ++j) sp.m *= sp.g;
  sp.p = std::max<std::uint64_t>(2, cfg.maxcalls / sp.m);
  unsigned workers = cfg.workers;
  if (workers == 0) workers = std::max(1u, std::thread::hardware_concurrency());
  sp.s = set_batch_size(sp.m, workers);
  return sp;
}

struct IterationResult {
  double estimate;
  double variance;
  std::uint32_t index;
};

struct Combined {
  double estimate;
  double sigma;
  double chi2_dof;
};

/// driver.hpp:146-169 (host form; the device form is gpu::weighted_estimate_dev).
[[nodiscard]] inline Combined weighted_estimate(std::span<const IterationResult> history) {
  if (history.empty()) throw std::invalid_argument("weighted_estimate: history must be non-empty");
  for (const IterationResult& it : history)
    if (!(it.variance >= 0.0)) throw std::invalid_argument("weighted_estimate: negative variance");
  std::vector<double> e, v;
  for (const IterationResult& it : history) {
    e.push_back(it.estimate);
    v.push_back(it.variance);
  }
  Combined c{};
  gpu::weighted_estimate_dev(e.data(), v.data(), static_cast<std::uint32_t>(e.size()), c.estimate, c.sigma, c.chi2_dof);
  return c;
}

/// driver.hpp:173-178
[[nodiscard]] inline bool check_convergence(const Combined& c, const RunConfig& cfg) {
  return gpu::converged_dev(c.estimate, c.sigma, c.chi2_dof, cfg.tau_rel, cfg.chi2_dof_max);
}

struct IntegrationResult {
  double estimate = 0.0;
  double sigma = 0.0;
  double chi2_dof = 0.0;
  std::uint32_t iterations_used = 0;
  bool converged = false;
  std::uint64_t total_samples = 0;
  std::uint64_t bin_writes = 0;
  SetupParams params{};
  std::vector<IterationResult> history;
};

struct IterationView {
  std::uint32_t iteration;
  bool adjusting;
  const IterationResult& result;
  const Combined& running;
  const Grid& grid;
  std::uint64_t bin_writes;
};

using IterationObserver = std::function<void(const IterationView&)>;

namespace gpu {

/// A device-resident integrate() run that can be stepped one iteration at a
/// time -- the multi-GPU driver inserts its all-reduce of exchange_words()
/// between sample() and finish().  integrate() below is the single-GPU loop.
class Run {
 public:
  Run(Context& ctx, IntegrandOps ops, const RunConfig& cfg)
      : ctx_(ctx), bufs_(ctx.acquire_run_bufs()), b_(*bufs_), ops_(std::move(ops)), cfg_(cfg) {
    sp_ = setup(cfg_);
    sh_ = make_shape(cfg_.dims, cfg_.n_bins, sp_.m, sp_.s, sp_.p);
    ctx_.activate();
    const Grid g0(cfg_.dims, cfg_.n_bins, cfg_.lower, cfg_.upper);
    const std::size_t n = std::size_t{cfg_.dims} * cfg_.n_bins;
    b_.contrib.ensure(n);
    b_.hist_est.ensure(cfg_.itmax);
    b_.hist_var.ensure(cfg_.itmax);
    b_.state.ensure(1);
    b_.err_key.ensure(1);
    xbuf_ = b_.words.ensure(exchange_words(cfg_.dims));
    words_ = xbuf_ + kXHeader;
    if (sizeof(double) * (n + 2 * cfg_.dims) <= Context::kPinnedBytes) {
      // one launch: the kernel reads the staged grid from pinned host memory
      // and zeroes the state and the exchange words
      ctx_.staging_wait();  // an earlier Run's setup may still read the buffer
      auto* pin = reinterpret_cast<double*>(ctx_.pinned());
      std::memcpy(pin, g0.raw_edges().data(), sizeof(double) * n);
      std::memcpy(pin + n, cfg_.lower.data(), sizeof(double) * cfg_.dims);
      std::memcpy(pin + n + cfg_.dims, cfg_.upper.data(), sizeof(double) * cfg_.dims);
      const auto nw = static_cast<std::uint32_t>(exchange_words(cfg_.dims));
      launch_pdl(run_init_kernel<0>, std::max<std::uint32_t>(1, (nw + 255) / 256), 256, 0, ctx_.stream(),
                 static_cast<const double*>(pin), static_cast<std::uint32_t>(n), cfg_.dims, b_.edges.ensure(n),
                 b_.lower.ensure(cfg_.dims), b_.upper.ensure(cfg_.dims), b_.state.get(), b_.err_key.get(),
                 xbuf_, nw);
      ++ctx_.launches;
      ctx_.staging_recorded();
      words_clean_ = true;
    } else {
      upload(ctx_, b_.edges, g0.raw_edges().data(), n);
      upload(ctx_, b_.lower, cfg_.lower.data(), cfg_.dims);
      upload(ctx_, b_.upper, cfg_.upper.data(), cfg_.dims);
      MCB_CUDA(cudaMemsetAsync(b_.state.get(), 0, sizeof(RunState), ctx_.stream()));
      MCB_CUDA(cudaMemsetAsync(b_.err_key.get(), 0xff, sizeof(unsigned long long), ctx_.stream()));
      zero_exchange();
    }
  }

  ~Run() {
    if (!ctx_alive_.expired()) ctx_.release_run_bufs(std::move(bufs_));  // else bufs_ just frees its memory
  }
  Run(const Run&) = delete;
  Run& operator=(const Run&) = delete;

  /// Resume from a checkpoint: the grid in force after `history.size()`
  /// completed iterations and their results.  The stream is keyed by
  /// (seed, iteration), so continuing at iteration history.size() + 1 gives
  /// bit for bit the run that was never interrupted (grid.hpp:148-174 text
  /// I/O carries the grid).  Returns that next iteration.
  std::uint32_t resume(const Grid& grid, std::span<const IterationResult> history) {
    if (grid.dims() != cfg_.dims || grid.n_bins() != cfg_.n_bins)
      throw std::invalid_argument("resume: grid shape does not match the RunConfig");
    for (std::uint32_t j = 0; j < cfg_.dims; ++j)
      if (grid.lowers()[j] != cfg_.lower[j] || grid.uppers()[j] != cfg_.upper[j])
        throw std::invalid_argument("resume: grid bounds do not match the RunConfig");
    const std::uint32_t n = static_cast<std::uint32_t>(history.size());
    if (n > cfg_.itmax) throw std::invalid_argument("resume: more completed iterations than itmax");
    for (std::uint32_t i = 0; i < n; ++i)
      if (history[i].index != i + 1) throw std::invalid_argument("resume: history indices must be 1..n");
    upload(ctx_, b_.edges, grid.raw_edges().data(), std::size_t{cfg_.dims} * cfg_.n_bins);
    RunState st{};
    if (n) {
      std::vector<double> e(n), v(n);
      for (std::uint32_t i = 0; i < n; ++i) {
        e[i] = history[i].estimate;
        v[i] = history[i].variance;
      }
      upload(ctx_, b_.hist_est, e.data(), n);
      upload(ctx_, b_.hist_var, v.data(), n);
      const Combined c = weighted_estimate(history);  // driver.hpp:246-252, as the device epilogue does
      st.iterations_used = n;
      // a checkpoint carries no counts: the completed iterations are credited
      // with the samples and deposits a full iteration takes
      for (std::uint32_t i = 1; i <= n; ++i) {
        st.samples += sp_.m * sp_.p;
        st.bin_writes += sp_.m * sp_.p * bin_axes(i);
      }
      st.estimate = c.estimate;
      st.sigma = c.sigma;
      st.chi2_dof = c.chi2_dof;
      if (check_convergence(c, cfg_)) st.converged = st.stop = 1;
    }
    MCB_CUDA(cudaMemcpyAsync(b_.state.get(), &st, sizeof st, cudaMemcpyHostToDevice, ctx_.stream()));
    ctx_.sync();  // the host-side state copy above must land before it goes out of scope
    return n + 1;
  }

  const SetupParams& params() const { return sp_; }
  const Shape& shape() const { return sh_; }
  std::uint32_t bin_axes(std::uint32_t it) const {
    if (it > cfg_.ita) return 0;
    return cfg_.variant == Variant::mcubes1d ? 1u : cfg_.dims;
  }
  /// Exchange buffer length (u64 words): the kXHeader count words -- finite
  /// samples taken (device-counted: the write count) and non-finite samples
  /// (so every rank learns of a failure in any rank's slice) -- then the
  /// accumulators.  An all-reduce of the first exchange_words_for(it) words
  /// covers iteration it.
  std::size_t exchange_words(std::uint32_t) const {
    return kXHeader + static_cast<std::size_t>(exchange_accs(cfg_.variant == Variant::mcubes1d ? 1u : cfg_.dims,
                                                      cfg_.n_bins)) * kXWords;
  }
  std::size_t exchange_words_for(std::uint32_t it) const {
    return kXHeader + static_cast<std::size_t>(exchange_accs(bin_axes(it), cfg_.n_bins)) * kXWords;
  }
  unsigned long long* exchange() const { return xbuf_; }
  void zero_exchange() {
    MCB_CUDA(cudaMemsetAsync(xbuf_, 0, sizeof(unsigned long long) * exchange_words(cfg_.dims), ctx_.stream()));
    words_clean_ = true;
  }
  /// Have finish() report per-iteration progress into host-mapped flags
  /// (Context::host_flags layout); nullptr turns it off.
  void set_host_flags(int* f) { host_flags_ = f; }
  /// Use a caller-owned exchange buffer of exchange_words() u64 (e.g. a torch
  /// tensor the caller all-reduces).  It is zeroed here; finish() leaves it
  /// zeroed for the next iteration.
  void set_exchange(unsigned long long* p) {
    xbuf_ = p ? p : b_.words.get();
    words_ = xbuf_ + kXHeader;
    zero_exchange();
  }
  const int* stop_flag() const { return &b_.state.get()->stop; }

  /// K1 over the work slice [n0, n1) of the linear work index (default: all
  /// cubes).  Its blocks flush straight into exchange(): after sample() the
  /// exchange words hold this slice's sums (the words are zeroed first unless
  /// finish() already left them zero).
  void sample(std::uint32_t it, std::uint64_t n0 = 0, std::uint64_t n1 = ~0ull) {
    if (n1 > sh_.m) n1 = sh_.m;
    if (npeers_) {
      // peer-memory exchange: never zero here -- other ranks may already be
      // adding this iteration's words into our buffer; finish() leaves each
      // buffer zeroed after reading it, and the two alternate by parity
      use_peers(it);
      bind_grid();
      last_ = ops_.k1(ctx_, sh_, bin_axes(it), iteration_key(cfg_.seed, it), n0, n1, stop_flag(),
                      b_.err_key.get(), words_);
      ctx_.peer.npeers = 0;
      last_it_ = it;
      return;
    }
    if (!words_clean_) zero_exchange();
    bind_grid();
    last_ = ops_.k1(ctx_, sh_, bin_axes(it), iteration_key(cfg_.seed, it), n0, n1, stop_flag(), b_.err_key.get(),
                    words_);
    words_clean_ = false;
    last_it_ = it;
  }

  /// Multi-GPU exchange over peer memory instead of a collective: rank
  /// `rank` of `npeers`; bufs[0] / bufs[1] hold every rank's exchange buffer
  /// (exchange_words() u64 each, zeroed) for odd / even iterations, flags
  /// every rank's flag array (npeers u64, zeroed), counter this rank's K1
  /// block counter (u32, zeroed).  Device pointers, already mapped into this
  /// process (CUDA IPC).  npeers = 0 turns it off.
  void set_peers(int rank, int npeers, unsigned long long* const* bufs_odd, unsigned long long* const* bufs_even,
                 unsigned long long* const* flags, unsigned int* counter) {
    if (npeers < 0 || npeers > kMaxPeers || (npeers && (rank < 0 || rank >= npeers)))
      throw std::invalid_argument("set_peers: need 0 <= rank < npeers <= 8");
    npeers_ = npeers;
    rank_ = rank;
    for (int q = 0; q < npeers; ++q) {
      peer_bufs_[1][q] = bufs_odd[q];
      peer_bufs_[0][q] = bufs_even[q];
      peer_flags_[q] = flags[q];
    }
    peer_counter_ = counter;
  }

  /// The cross-block reduction (the reference's in-process exact merge,
  /// sampler.hpp:272-276).  K1's blocks already added their words into the
  /// exchange buffer, so this only checks the call order; the entry point
  /// stays for the stepped API (mcb_run_reduce).
  void reduce(std::uint32_t it) {
    if (it != last_it_) throw std::invalid_argument("reduce: iteration was not sampled");
  }

  /// K3b + K4 (one fused kernel) for iteration it, after the optional
  /// all-reduce of exchange().
  void finish(std::uint32_t it) {
    if (npeers_) use_peers(it);
    const std::uint32_t ba = bin_axes(it);
    EpilogueArgs e = epilogue_args(it);
    launch_finish(ctx_, sh_, ba, words_, b_.hist_est.get() + (it - 1), b_.hist_var.get() + (it - 1),
                  ba ? b_.contrib.get() : nullptr, stop_flag(), &e, /*zero_words=*/true);
    ctx_.peer.npeers = 0;
    words_clean_ = true;  // (or the run is stopped, and reduce() is a no-op)
  }

  EpilogueArgs epilogue_args(std::uint32_t it) {
    const std::uint32_t ba = bin_axes(it);
    EpilogueArgs e{};
    e.st = b_.state.get();
    e.hist_est = b_.hist_est.get();
    e.hist_var = b_.hist_var.get();
    e.err_key = b_.err_key.get();
    e.it = it;
    e.adjusting = ba ? 1 : 0;
    e.tau = cfg_.tau_rel;
    e.chi2max = cfg_.chi2_dof_max;
    e.adj = AdjustArgs{cfg_.dims,       cfg_.n_bins,
                       b_.lower.get(), b_.upper.get(),
                       b_.edges.get(), b_.contrib.get(),
                       cfg_.alpha,       cfg_.variant == Variant::mcubes1d ? 1 : 0,
                       b_.contrib.get()};
    e.host_flags = host_flags_;
    return e;
  }

  // ---- compact exchange (dist.integrate(transport="compact")):
  // every rank rounds its own slice (round_local), the ranks all-gather the
  // d x n_bins + 6 doubles, every rank sums them in rank order (combine) and
  // runs the epilogue on the result (finish_rounded).  3.2 KB per rank at 8D
  // instead of the exact exchange's 216 KB, at the price of G-dependent last
  // bits (each rank's partial sum is rounded before the cross-rank sum);
  // G = 1 is bitwise the exact path.

  /// Doubles per rank in the compact exchange.
  std::size_t compact_len() const { return kCompactHead + std::size_t{cfg_.dims} * cfg_.n_bins; }
  /// Round this rank's exchange words into `out` (device, compact_len()
  /// doubles, layout of kCompactHead) and leave the words zeroed.
  void round_local(std::uint32_t it, double* out) {
    if (npeers_) throw std::invalid_argument("round_local: the run uses the peer-memory exchange");
    const std::uint32_t ba = bin_axes(it);
    launch_finish(ctx_, sh_, ba, words_, out, out + 1, ba ? out + kCompactHead : nullptr, stop_flag(), nullptr,
                  /*zero_words=*/true, reinterpret_cast<unsigned long long*>(out + 2));
    words_clean_ = true;
  }
  /// Sum `nranks` ranks' round_local outputs (device, nranks x compact_len()
  /// doubles, rank-major) in rank order into this run's iteration state.
  void combine(std::uint32_t it, const double* gathered, int nranks) {
    if (nranks < 1) throw std::invalid_argument("combine: nranks must be >= 1");
    const std::uint32_t ba = bin_axes(it);
    const int len = static_cast<int>(compact_len());
    launch_pdl(combine_kernel<0>, std::max(1, (len + 255) / 256), 256, 0, ctx_.stream(), gathered, nranks, len,
               static_cast<int>(ba ? cfg_.dims * cfg_.n_bins : 0u), b_.hist_est.get() + (it - 1), b_.hist_var.get() + (it - 1),
               b_.contrib.get(), xbuf_, stop_flag());
    ++ctx_.launches;
    words_clean_ = false;  // the header holds the combined counts until finish_rounded()
  }
  /// The epilogue of iteration it (grid adaptation, weighted estimate,
  /// convergence gate) on the combined values.
  void finish_rounded(std::uint32_t it) {
    const std::uint32_t ba = bin_axes(it);
    EpilogueArgs e = epilogue_args(it);
    launch_finish(ctx_, sh_, ba, words_, b_.hist_est.get() + (it - 1), b_.hist_var.get() + (it - 1),
                  ba ? b_.contrib.get() : nullptr, stop_flag(), &e, /*zero_words=*/true, nullptr,
                  /*prerounded=*/true);
    words_clean_ = true;
  }

  RunState state() {
    RunState st;
    MCB_CUDA(cudaMemcpyAsync(&st, b_.state.get(), sizeof st, cudaMemcpyDeviceToHost, ctx_.stream()));
    ctx_.sync();
    return st;
  }

  /// Whether the run stopped on a non-finite sample, and this rank's first
  /// failing sample key (t * p + k; all-ones when the failure was in another
  /// rank's slice).  Multi-rank drivers take the minimum over ranks and hand
  /// it back with set_failure_key() so that every rank reports the same
  /// NonFiniteSample (the reference reports the first in serial order).
  bool failure_key(unsigned long long& key) {
    const RunState st = state();
    MCB_CUDA(cudaMemcpyAsync(&key, b_.err_key.get(), sizeof key, cudaMemcpyDeviceToHost, ctx_.stream()));
    ctx_.sync();
    return st.failed != 0;
  }
  void set_failure_key(unsigned long long key) {
    MCB_CUDA(cudaMemcpyAsync(b_.err_key.get(), &key, sizeof key, cudaMemcpyHostToDevice, ctx_.stream()));
    ctx_.sync();
  }

  /// Replace the device grid with host edges (dims*n_bins), stream-ordered.
  void set_grid(const double* host_edges) {
    upload(ctx_, b_.edges, host_edges, std::size_t{cfg_.dims} * cfg_.n_bins);
  }

  Grid grid() {
    const std::size_t n = std::size_t{cfg_.dims} * cfg_.n_bins;
    std::vector<double> e(n);
    download(ctx_, e.data(), b_.edges.get(), n);
    ctx_.sync();
    return Grid::from_edges(cfg_.dims, cfg_.n_bins, cfg_.lower, cfg_.upper, std::move(e));
  }

  /// Collect the result (one synchronisation); throws NonFiniteSample.
  IntegrationResult result() {
    // one synchronisation: state, error key and the whole history land in
    // the context's pinned staging buffer together
    unsigned char* pin = ctx_.pinned();
    const std::size_t hbytes = sizeof(double) * cfg_.itmax;
    const bool staged = sizeof(RunState) + 8 + 2 * hbytes <= Context::kPinnedBytes;
    RunState st;
    unsigned long long key = ~0ull;
    std::vector<double> e, v;
    if (staged) {
      ctx_.staging_wait();
      launch_pdl(run_collect_kernel<0>, std::max<std::uint32_t>(1, (cfg_.itmax + 255) / 256), 256, 0, ctx_.stream(),
                 static_cast<const RunState*>(b_.state.get()), static_cast<const unsigned long long*>(b_.err_key.get()),
                 static_cast<const double*>(b_.hist_est.get()), static_cast<const double*>(b_.hist_var.get()),
                 cfg_.itmax, pin);
      ++ctx_.launches;
      ctx_.sync();
      std::memcpy(&st, pin, sizeof st);
      std::memcpy(&key, pin + sizeof(RunState), 8);
      const auto* he = reinterpret_cast<const double*>(pin + sizeof(RunState) + 8);
      const auto* hv = reinterpret_cast<const double*>(pin + sizeof(RunState) + 8 + hbytes);
      e.assign(he, he + st.iterations_used);
      v.assign(hv, hv + st.iterations_used);
    } else {
      st = state();
      MCB_CUDA(cudaMemcpyAsync(&key, b_.err_key.get(), sizeof key, cudaMemcpyDeviceToHost, ctx_.stream()));
      e.resize(st.iterations_used);
      v.resize(st.iterations_used);
      if (st.iterations_used) {
        download(ctx_, e.data(), b_.hist_est.get(), st.iterations_used);
        download(ctx_, v.data(), b_.hist_var.get(), st.iterations_used);
      }
      ctx_.sync();
    }
    IntegrationResult res;
    res.params = sp_;
    if (st.failed == 2) throw_overflow();
    if (st.failed) {
      bind_grid();  // the failed iteration's grid (the epilogue aborted before adapting it)
      throw_nonfinite(ctx_, ops_, sh_, iteration_key(cfg_.seed, st.failed_iteration), key);
    }
    const std::uint32_t n = st.iterations_used;
    for (std::uint32_t i = 0; i < n; ++i) res.history.push_back({e[i], v[i], i + 1});
    // device-counted: every finite sample K1 took, and the deposits it made
    // (a resumed run counts only the iterations it ran itself)
    res.total_samples = st.samples;
    res.bin_writes = st.bin_writes;
    res.iterations_used = n;
    res.converged = st.converged != 0;
    res.estimate = st.estimate;
    res.sigma = st.sigma;
    res.chi2_dof = st.chi2_dof;
    return res;
  }

 private:
  Context& ctx_;
  /// The run's own device buffers: nothing else enqueued on the context
  /// (a standalone v_sample, Grid::adjusted, another Run, e.g. from an
  /// observer) can replace this run's grid, state or exchange words.  They
  /// come from the context's pool and go back to it when the run ends.
  std::unique_ptr<RunBufs> bufs_;
  RunBufs& b_;
  std::weak_ptr<const int> ctx_alive_ = ctx_.alive();
  IntegrandOps ops_;
  RunConfig cfg_;
  SetupParams sp_{};
  Shape sh_{};
  /// K1 / the point kernel read this run's grid.
  void bind_grid() {
    ctx_.grid_edges = b_.edges.get();
    ctx_.grid_lower = b_.lower.get();
  }
  /// Point the launch at iteration it's buffers: parity it & 1, flag = it.
  void use_peers(std::uint32_t it) {
    PeerArgs& p = ctx_.peer;
    p = PeerArgs{};
    const int par = static_cast<int>(it & 1u);
    for (int q = 0; q < npeers_; ++q) {
      p.words[q] = peer_bufs_[par][q] + kXHeader;
      p.flags[q] = peer_flags_[q] + rank_;
    }
    p.my_flags = peer_flags_[rank_];
    p.counter = peer_counter_;
    p.flag = it;
    p.npeers = npeers_;
    xbuf_ = peer_bufs_[par][rank_];
    words_ = xbuf_ + kXHeader;
  }

  int npeers_ = 0, rank_ = 0;
  unsigned long long* peer_bufs_[2][kMaxPeers] = {};
  unsigned long long* peer_flags_[kMaxPeers] = {};
  unsigned int* peer_counter_ = nullptr;
  unsigned long long* xbuf_ = nullptr;   ///< exchange buffer: [sample count][non-finite count][accumulator words]
  unsigned long long* words_ = nullptr;  ///< xbuf_ + kXHeader
  Launch last_{};
  std::uint32_t last_it_ = 0;
  int* host_flags_ = nullptr;
  bool words_clean_ = false;  ///< exchange words are zero in stream order
};

/// integrate() for type-erased integrands: the whole schedule is enqueued
/// without host synchronisation unless an observer wants per-iteration views.
inline IntegrationResult integrate_ops(Context& ctx, const IntegrandOps& ops, const RunConfig& cfg,
                                       const IterationObserver& observe = {}, const Grid* resume_grid = nullptr,
                                       std::span<const IterationResult> resume_history = {}) {
  const NvtxRange whole("mcubes::integrate");
  Run run(ctx, ops, cfg);
  const std::uint32_t first = resume_grid ? run.resume(*resume_grid, resume_history) : 1u;
  if (first > 1 && run.state().stop) return run.result();  // the checkpoint had already converged
  // Bounded lookahead: keep at most kAhead iterations in flight and stop
  // enqueuing once the finish kernel has reported convergence through the
  // host-mapped flags, so a run that converges early does not pay for the
  // launches of its remaining (no-op) iterations.  Results are unaffected:
  // iterations after `stop` are no-ops on the device either way.
  constexpr std::uint32_t kAhead = 2;
  const bool lookahead = !observe && cfg.itmax <= Context::kMaxFlagIterations;
  int* flags = ctx.host_flags();
  if (lookahead) {
    std::memset(flags, 0, sizeof(int) * cfg.itmax);
    run.set_host_flags(flags);
  }
  unsigned long long writes_before = 0;  // device-counted deposits before this iteration (observer views)
  for (std::uint32_t it = first; it <= cfg.itmax; ++it) {
    if (lookahead && it >= first + kAhead) {
      const std::uint32_t back = it - kAhead;
      MCB_CUDA(cudaEventSynchronize(ctx.event(back % (kAhead + 1))));
      if (reinterpret_cast<volatile int*>(flags)[back - 1] != 1) break;  // stopped (or never ran: stopped earlier)
    }
    {
      const NvtxRange r(it <= cfg.ita ? "mcubes::iteration (adjusting)" : "mcubes::iteration (frozen)");
      run.sample(it);
      run.reduce(it);
      run.finish(it);
    }
    if (lookahead) MCB_CUDA(cudaEventRecord(ctx.event(it % (kAhead + 1)), ctx.stream()));
    if (observe) {
      const RunState st = run.state();
      if (st.failed || st.iterations_used != it) break;
      const IterationResult r = run.result().history.back();
      const Combined c{st.estimate, st.sigma, st.chi2_dof};
      const Grid g = run.grid();
      observe(IterationView{it, it <= cfg.ita, r, c, g, st.bin_writes - writes_before});
      writes_before = st.bin_writes;
      if (st.stop) break;
    }
  }
  return run.result();
}

}  // namespace gpu

/// integrate() continued from a checkpoint (Run::resume): `grid` is the grid
/// after the completed iterations `history` (1..n).  Bitwise equal to the
/// uninterrupted run.
template <gpu::DeviceIntegrand F>
IntegrationResult integrate_resume(const F& f, const RunConfig& cfg, const Grid& grid,
                                   std::span<const IterationResult> history, const IterationObserver& observe = {}) {
  gpu::Context& ctx = gpu::default_context();
  return gpu::integrate_ops(ctx, gpu::make_ops_for(f, cfg.rng), cfg, observe, &grid, history);
}

/// The full integration loop (driver.hpp:215-258), on the GPU.
template <gpu::DeviceIntegrand F>
IntegrationResult integrate(const F& f, const RunConfig& cfg, const IterationObserver& observe = {}) {
  gpu::Context& ctx = gpu::default_context();
  return gpu::integrate_ops(ctx, gpu::make_ops_for(f, cfg.rng), cfg, observe);
}

}  // namespace mcubes
