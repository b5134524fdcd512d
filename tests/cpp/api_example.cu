// Drop-in check of the C++ header API (include/mcubes_b200/mcubes.cuh): code
// written against the reference's mcubes:: API (driver.hpp / sampler.hpp /
// grid.hpp) compiles unchanged except for the include line and the
// __host__ __device__ marker on the functor, and runs on the GPU.
// Prints machine-readable lines checked by tests/test_gpu_cpp_api.py.
#include <cmath>
#include <cstdio>
#include <span>

#include "mcubes_b200/mcubes.cuh"

// A user integrand in the reference's style (README.md quickstart):
// exp(-50 sum (x-1/2)^2), plus a stateful member.
struct Bump {
  double width;
  __host__ __device__ double operator()(std::span<const double> x) const {
    double s = 0.0;
    for (const double xi : x) s += (xi - 0.5) * (xi - 0.5);
    return std::exp(-s / width);
  }
};

// Functors used as kernel template arguments must be namespace-scope types
// (a CUDA rule); state travels by value.
struct Seven {
  __host__ __device__ double operator()(std::span<const double>) const { return 7.0; }
};
struct Bad {
  __host__ __device__ double operator()(std::span<const double> x) const { return x[0] > 0.5 ? INFINITY : 1.0; }
};

int main() {
  mcubes::RunConfig cfg;
  cfg.dims = 3;
  cfg.maxcalls = 200000;
  cfg.lower.assign(3, 0.0);
  cfg.upper.assign(3, 1.0);
  cfg.tau_rel = 1e-4;
  int observed = 0;
  const auto res = mcubes::integrate(Bump{1.0 / 50.0}, cfg, [&](const mcubes::IterationView& v) {
    ++observed;
    std::printf("iter %u adjusting %d estimate %.17g writes %llu\n", v.iteration, v.adjusting ? 1 : 0,
                v.result.estimate, static_cast<unsigned long long>(v.bin_writes));
  });
  const double truth = std::pow(std::sqrt(M_PI / 50.0) * std::erf(std::sqrt(50.0) / 2.0), 3.0);
  std::printf("RESULT estimate %.17g sigma %.17g chi2 %.17g iterations %u converged %d truth %.17g observed %d\n",
              res.estimate, res.sigma, res.chi2_dof, res.iterations_used, res.converged ? 1 : 0, truth, observed);

  // v_sample + Grid::adjusted through the same API
  const mcubes::Grid g(2, 8, std::vector<double>{0.0, 0.0}, std::vector<double>{2.0, 2.0});
  const auto out = mcubes::v_sample(Seven{}, g, 16, 1, 4, 9, 1);
  const auto g2 = g.adjusted(out.contributions, 1.5);
  std::printf("VSAMPLE estimate %.17g variance %.17g writes %llu edge %.17g\n", out.raw_estimate, out.raw_variance,
              static_cast<unsigned long long>(out.contributions.writes()), g2.edges(0)[7]);
  try {
    (void)mcubes::v_sample(Bad{}, g, 16, 1, 4, 9, 1);
    std::printf("NONFINITE none\n");
  } catch (const mcubes::NonFiniteSample& e) {
    std::printf("NONFINITE x0 %.17g value %g\n", e.point()[0], e.value());
  }
  return 0;
}
