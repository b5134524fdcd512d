// SPDX-License-Identifier: Apache-2.0
//
// The rest of the reference's public headers through the B200 umbrella
// header: integrands.hpp (IntegrandSpec and its factories), oracle.hpp
// (vegas_serial_iteration), accumulators.hpp (CubeAccumulator,
// update_variance), plus the RAII device table.  Checks that need no
// quadrature run here (CHECK lines); values the Python test compares with the
// compiled reference and with scipy quadrature are printed as KEY lines.
// Port of tests/test_integrands.cpp (point values, lookup validation,
// symmetry, factoring, thresholds) without Catch2.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numbers>
#include <random>
#include <span>
#include <stdexcept>
#include <vector>

#include "mcubes_b200/mcubes.hpp"

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("CHECK FAILED line %d: %s\n", __LINE__, #cond);      \
      ++failures;                                                     \
    }                                                                 \
  } while (0)
#define CHECK_THROWS(expr)                                            \
  do {                                                                \
    bool thrown = false;                                              \
    try {                                                             \
      (void)(expr);                                                   \
    } catch (const std::invalid_argument&) {                          \
      thrown = true;                                                  \
    }                                                                 \
    if (!thrown) {                                                    \
      std::printf("CHECK_THROWS FAILED line %d: %s\n", __LINE__, #expr); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static bool rel(double a, double b, double tol) { return std::abs(a - b) <= tol * std::abs(b); }

static double eval(const mcubes::IntegrandSpec& s, std::initializer_list<double> pt) {
  const std::vector<double> x(pt);
  return s(std::span<const double>(x));
}

int main() {
  using namespace mcubes;
  // --- test_integrands.cpp: point values
  CHECK(eval(make_suite_integrand(1, 3), {0.0, 0.0, 0.0}) == 1.0);
  CHECK(eval(make_suite_integrand(4, 2), {0.5, 0.5}) == 1.0);
  CHECK(eval(make_suite_integrand(5, 4), {0.5, 0.5, 0.5, 0.5}) == 1.0);
  CHECK(rel(eval(make_suite_integrand(2, 2), {0.5, 0.5}), 2500.0 * 2500.0, 1e-12));
  CHECK(rel(eval(make_suite_integrand(3, 2), {1.0, 1.0}), 1.0 / 64.0, 1e-12));
  CHECK(reference_value(1, 1) == std::sin(1.0));
  CHECK(reference_value(3, 1) == 0.5);
  // fA / fB
  const auto fa = make_fA();
  CHECK(fa.dims == 6 && fa.lower == std::vector<double>(6, 0.0) && fa.upper == std::vector<double>(6, 10.0));
  CHECK(fa.reference.has_value() && std::abs(*fa.reference - -49.165073) < 1e-6);
  CHECK(eval(fa, {0, 0, 0, 0, 0, 0}) == 0.0);
  CHECK(std::abs(eval(fa, {2.0 * std::numbers::pi, 0, 0, 0, 0, 0})) < 1e-14);
  const auto fb = make_fB();
  CHECK(fb.dims == 9 && fb.lower == std::vector<double>(9, -1.0) && *fb.reference == 1.0);
  const double norm = std::pow(2.0 * std::numbers::pi * 0.01, -4.5);
  CHECK(rel(eval(fb, {0, 0, 0, 0, 0, 0, 0, 0, 0}), norm, 1e-14));
  CHECK(rel(norm, 255970.89820277557, 1e-12));
  // symmetric families are permutation invariant; product families factor
  std::mt19937_64 rng(77);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  for (int family : {2, 4, 5}) {
    const auto s5 = make_suite_integrand(family, 5), s3 = make_suite_integrand(family, 3),
               s1 = make_suite_integrand(family, 1);
    for (int trial = 0; trial < 20; ++trial) {
      std::vector<double> x(5);
      for (auto& v : x) v = unit(rng);
      std::vector<double> y = x;
      std::shuffle(y.begin(), y.end(), rng);
      CHECK(rel(s5(std::span<const double>(y)), s5(std::span<const double>(x)), 1e-12));
      const double joint = s3(std::span<const double>(x.data(), 3));
      CHECK(rel(joint, eval(s1, {x[0]}) * eval(s1, {x[1]}) * eval(s1, {x[2]}), 1e-12));
    }
  }
  // the discontinuous family's thresholds
  const auto f6 = make_suite_integrand(6, 2);
  CHECK(eval(f6, {0.5, 0.1}) == 0.0 && eval(f6, {0.1, 0.6}) == 0.0);
  CHECK(eval(f6, {0.4, 0.1}) == 0.0 && eval(f6, {0.1, 0.5}) == 0.0);
  CHECK(rel(eval(f6, {0.39, 0.49}), std::exp(5.0 * 0.39 + 6.0 * 0.49), 1e-12));
  std::vector<double> near_one(8, 0.01);
  near_one[6] = near_one[7] = 0.99;
  CHECK(make_suite_integrand(6, 8)(std::span<const double>(near_one)) > 0.0);
  // lookup validation
  CHECK(make_integrand("f3", 4).dims == 4 && make_integrand("fA", 0).dims == 6 && make_integrand("fB", 9).name == "fB");
  CHECK_THROWS(make_integrand("f1", 0));
  CHECK_THROWS(make_integrand("fA", 3));
  CHECK_THROWS(make_integrand("fB", 2));
  CHECK_THROWS(make_integrand("f7", 2));
  CHECK_THROWS(make_integrand("g1", 2));
  CHECK_THROWS(make_integrand("", 2));
  CHECK_THROWS(make_suite_integrand(0, 1));
  CHECK_THROWS(make_suite_integrand(7, 1));
  CHECK_THROWS(make_suite_integrand(1, 0));
  CHECK_THROWS(reference_value(9, 1));
  CHECK_THROWS(reference_value(1, 0));
  // reference values for the Python side (vs the compiled reference and quadrature)
  for (int family = 1; family <= 6; ++family)
    for (std::uint32_t d : {1u, 2u, 3u, 6u, 8u})
      std::printf("REFVAL %d %u %.17g\n", family, d, reference_value(family, d));

  // --- accumulators.hpp
  CubeAccumulator ca;
  for (double v : {1.0, 2.0, 4.0}) ca.add(v);
  CHECK(ca.count == 3 && ca.sum_v == 7.0 && ca.sum_v2 == 21.0);
  CHECK(rel(update_variance(ca), (21.0 / 3.0 - (7.0 / 3.0) * (7.0 / 3.0)) / 2.0, 1e-15));
  CubeAccumulator one;
  one.add(1.0);
  CHECK_THROWS(update_variance(one));

  // --- the catalogue on the GPU: integrate(spec), v_sample(spec), vegas_serial_iteration
  {
    const auto spec = make_suite_integrand(4, 8);
    RunConfig cfg;
    cfg.dims = spec.dims;
    cfg.maxcalls = 10'000'000;
    cfg.itmax = 10;
    cfg.ita = 5;
    cfg.tau_rel = 1e-3;
    cfg.seed = 3;
    cfg.lower = spec.lower;
    cfg.upper = spec.upper;
    const IntegrationResult r = integrate(spec, cfg);
    std::printf("SUITE f4 8 estimate %.17g sigma %.17g iterations %u converged %d reference %.17g\n", r.estimate,
                r.sigma, r.iterations_used, r.converged ? 1 : 0, *spec.reference);
    const auto fa_r = integrate(make_fA(), [&] {
      RunConfig c;
      c.dims = 6;
      c.maxcalls = 1'000'000;
      c.lower = fa.lower;
      c.upper = fa.upper;
      c.seed = 1;
      return c;
    }());
    std::printf("SUITE fA 6 estimate %.17g sigma %.17g iterations %u converged %d reference %.17g\n",
                fa_r.estimate, fa_r.sigma, fa_r.iterations_used, fa_r.converged ? 1 : 0, *fa.reference);
    const auto f2 = make_suite_integrand(2, 3);
    const Grid g(3, 8, std::vector<double>(3, 0.0), std::vector<double>(3, 1.0));
    const auto a = v_sample(f2, g, 1000, 7, 3, 5, 1);
    const auto b = vegas_serial_iteration(f2, g, 1000, 3, 5, 1);
    CHECK(a.raw_estimate == b.raw_estimate && a.raw_variance == b.raw_variance);
    CHECK(a.contributions.values() == b.contributions.values() && a.contributions.writes() == b.contributions.writes());
    std::printf("SERIAL est %.17g var %.17g writes %llu\n", b.raw_estimate, b.raw_variance,
                static_cast<unsigned long long>(b.contributions.writes()));
    const auto fr = v_sample_no_adjust(f2, g, 1000, 1, 3, 5, 1);
    CHECK(fr.raw_estimate == a.raw_estimate && fr.raw_variance == a.raw_variance);
  }
  // --- a stateful integrand with an RAII device table: f = prod_j (1 + x_j) on [0,2]^4
  {
    const std::uint32_t d = 4, n = 3;
    std::vector<double> tab(d * n);
    for (std::uint32_t j = 0; j < d; ++j)
      for (std::uint32_t k = 0; k < n; ++k) tab[j * n + k] = 1.0 + static_cast<double>(k);  // x = 0, 1, 2
    const std::vector<double> lo(d, 0.0), hi(d, 2.0);
    gpu::DeviceTable table(d, n, tab, lo, hi);
    RunConfig cfg;
    cfg.dims = d;
    cfg.maxcalls = 1'000'000;
    cfg.itmax = 5;
    cfg.ita = 3;
    cfg.tau_rel = 1e-9;
    cfg.lower = lo;
    cfg.upper = hi;
    const auto r = integrate(table.view(), cfg);
    std::printf("TABLE estimate %.17g sigma %.17g truth %.17g\n", r.estimate, r.sigma, std::pow(4.0, 4.0));
  }
  std::printf("FAILURES %d\n", failures);
  return failures ? 1 : 0;
}
