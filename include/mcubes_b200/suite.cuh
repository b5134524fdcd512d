// SPDX-License-Identifier: Apache-2.0
//
// The reference's integrand catalogue (integrands.hpp:23-235) for the B200
// C++ API: IntegrandSpec, reference_value, make_suite_integrand, make_fA,
// make_fB, make_integrand -- same names, fields, closed forms and errors.
//
// The one change is the callable.  The reference's IntegrandSpec::evaluate is
// a std::function, which device code cannot call; here it is gpu::fn::Suite,
// a trivially copyable functor that dispatches on the family to the suite
// functors of integrands.cuh (the reference's operation order).  A spec is
// still callable on the host (spec(x)), and mcubes::integrate / v_sample /
// v_sample_no_adjust accept it directly, sampling spec.evaluate on the GPU.
#pragma once

#include <algorithm>
#include <bit>
#include <cmath>
#include <complex>
#include <cstdint>
#include <numbers>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "integrands.cuh"

namespace mcubes {

namespace gpu::fn {

/// Every catalogue integrand behind one device-callable functor: family 1..6
/// (the Genz suite), 7 = fA, 8 = fB (norm = (2 pi 0.01)^-4.5).
struct Suite {
  int family = 0;
  double norm = 0.0;
  ExpConsts ec;  ///< exp's constants, carried in the kernel parameters (integrands.cuh)
  MCB_HD double operator()(std::span<const double> x) const {
    switch (family) {
      case 1: return F1{}(x);
      case 2: return F2{}(x);
      case 3: return F3{}(x);
      case 4: return F4{ec}(x);
      case 5: return F5{ec}(x);
      case 6: return F6{ec}(x);
      case 7: return FA{}(x);
      default: return FB{norm, ec}(x);
    }
  }
};

}  // namespace gpu::fn

/// integrands.hpp:23-32, with a device-callable `evaluate` (see above).
struct IntegrandSpec {
  std::string name;
  std::uint32_t dims = 0;
  std::vector<double> lower;
  std::vector<double> upper;
  gpu::fn::Suite evaluate;
  std::optional<double> reference;  ///< exact integral over the box, when known

  double operator()(std::span<const double> x) const { return evaluate(x); }
};

namespace detail {
/// integral_0^1 e^(i a x) dx = (e^(i a) - 1) / (i a)
inline std::complex<double> unit_phase_integral(double a) {
  return (std::polar(1.0, a) - 1.0) / std::complex<double>(0.0, a);
}

/// Corner peak (1 + sum_i i x_i)^-(d+1) over [0,1]^d: the d-fold
/// antiderivative is an alternating sum over the axis subsets S of
/// 1 / (1 + sum_{i in S} i), divided by d! * prod_i i = (d!)^2.
inline double corner_peak_integral(std::uint32_t d) {
  double alternating = 0.0;
  const std::uint64_t subsets = std::uint64_t{1} << d;
  for (std::uint64_t s = 0; s < subsets; ++s) {
    double denom = 1.0;
    for (std::uint32_t i = 0; i < d; ++i)
      if ((s >> i) & 1u) denom += static_cast<double>(i + 1);
    alternating += (std::popcount(s) & 1 ? -1.0 : 1.0) / denom;
  }
  double factorial_sq = 1.0;
  for (std::uint32_t i = 1; i <= d; ++i) factorial_sq *= static_cast<double>(i) * static_cast<double>(i);
  return alternating / factorial_sq;
}
}  // namespace detail

/// Exact integral of suite family `family` over [0,1]^d -- the closed forms of
/// integrands.hpp:53-104 (oscillatory: complex exponentials; product
/// families: per-axis antiderivatives; corner peak: inclusion-exclusion).
inline double reference_value(int family, std::uint32_t d) {
  if (d < 1) throw std::invalid_argument("reference_value: d must be >= 1");
  const double dd = static_cast<double>(d);
  if (family == 1) {
    std::complex<double> prod = 1.0;
    for (std::uint32_t i = 1; i <= d; ++i) prod *= detail::unit_phase_integral(static_cast<double>(i));
    return prod.real();
  }
  if (family == 2) return std::pow(100.0 * std::atan(25.0), dd);  // per axis (2/a) atan(1/(2a)), a = 1/50
  if (family == 3) return detail::corner_peak_integral(d);
  if (family == 4) return std::pow(std::sqrt(std::numbers::pi) / 25.0 * std::erf(12.5), dd);
  if (family == 5) return std::pow((1.0 - std::exp(-5.0)) / 5.0, dd);
  if (family == 6) {  // axis i (1-based): (e^((i+4) u_i) - 1)/(i+4), u_i = min(1, (3+i)/10)
    double prod = 1.0;
    for (std::uint32_t i = 1; i <= d; ++i) {
      const double rate = static_cast<double>(i) + 4.0;
      const double cut = std::min(1.0, (3.0 + static_cast<double>(i)) / 10.0);
      prod *= (std::exp(rate * cut) - 1.0) / rate;
    }
    return prod;
  }
  throw std::invalid_argument("reference_value: unknown family " + std::to_string(family));
}

/// Suite integrand `family` on the unit hyper-cube with its reference value
/// (integrands.hpp:107-175).
namespace detail {
/// One catalogue entry: `name` on the box [lo, hi]^dims, evaluated on the
/// device by fn::Suite{family, norm}.
inline IntegrandSpec catalogue_entry(std::string name, std::uint32_t dims, double lo, double hi,
                                     std::optional<double> reference, int family, double norm = 0.0) {
  IntegrandSpec spec;
  spec.name = std::move(name);
  spec.dims = dims;
  spec.lower = std::vector<double>(dims, lo);
  spec.upper = std::vector<double>(dims, hi);
  spec.reference = reference;
  spec.evaluate = gpu::fn::Suite{family, norm};
  return spec;
}
}  // namespace detail

/// Genz family 1..6 on the unit cube (integrands.hpp:107-175).
inline IntegrandSpec make_suite_integrand(int family, std::uint32_t d) {
  if (family < 1 || family > 6) throw std::invalid_argument("make_suite_integrand: family must be in 1..6");
  if (d < 1) throw std::invalid_argument("make_suite_integrand: d must be >= 1");
  return detail::catalogue_entry("f" + std::to_string(family), d, 0.0, 1.0, reference_value(family, d), family);
}

/// sin of the coordinate sum over (0,10)^6 (integrands.hpp:181-196); reference
/// Im[((e^(10i) - 1)/i)^6].
inline IntegrandSpec make_fA() {
  const std::complex<double> one_axis = (std::exp(std::complex<double>(0.0, 10.0)) - 1.0) / std::complex<double>(0.0, 1.0);
  return detail::catalogue_entry("fA", 6, 0.0, 10.0, std::pow(one_axis, 6).imag(), 7);
}

/// Normalised Gaussian (variance 0.01 per axis) on (-1,1)^9 (integrands.hpp:200-215):
/// mass erf(1/sqrt(2 sigma^2))^9 inside the box.
inline IntegrandSpec make_fB() {
  constexpr double kSigma2 = 0.01;
  return detail::catalogue_entry("fB", 9, -1.0, 1.0, std::pow(std::erf(1.0 / std::sqrt(2.0 * kSigma2)), 9.0), 8,
                                 std::pow(2.0 * std::numbers::pi * kSigma2, -4.5));
}

/// Look up an integrand by CLI name (integrands.hpp:221-235): "f1".."f6" need
/// an explicit dimension; "fA" / "fB" take 0 or their own dimension.
inline IntegrandSpec make_integrand(std::string_view id, std::uint32_t dims) {
  const std::string name(id);
  if (name == "fA" || name == "fB") {
    IntegrandSpec fixed = name == "fA" ? make_fA() : make_fB();
    if (dims == 0 || dims == fixed.dims) return fixed;
    throw std::invalid_argument(name + " is fixed at " + std::to_string(fixed.dims) + " dimensions");
  }
  const bool genz = name.size() == 2 && name[0] == 'f' && name[1] >= '1' && name[1] <= '6';
  if (!genz) throw std::invalid_argument("unknown integrand \"" + name + "\"");
  if (dims == 0) throw std::invalid_argument(name + " requires an explicit dimension");
  return make_suite_integrand(name[1] - '0', dims);
}

}  // namespace mcubes
