// Drop-in check of the C++ header API (include/mcubes_b200/mcubes.cuh): code
// written against the reference's mcubes:: API (driver.hpp / sampler.hpp /
// grid.hpp) compiles unchanged except for the include line and the
// __host__ __device__ marker on the functor, and runs on the GPU.
// Prints machine-readable lines checked by tests/test_gpu_cpp_api.py.
#include <chrono>
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
// BASELINE config 3's optional variant: a sharply peaked normalised Gaussian,
// sigma = 0.01 per axis, centred at 1/2 (a user functor, not a built-in).
struct SharpGauss {
  double inv2s2, norm;  // 1 / (2 sigma^2), (2 pi sigma^2)^(-d/2)
  __host__ __device__ double operator()(std::span<const double> x) const {
    double s = 0.0;
    for (const double xi : x) s += (xi - 0.5) * (xi - 0.5);
    return norm * std::exp(-s * inv2s2);
  }
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
  // BASELINE config 3 (sigma 0.01 variant) on the Philox path: 6D at 1e9 calls per iteration
  {
    const double sg = 0.01;
    mcubes::RunConfig c3;
    c3.dims = 6;
    c3.maxcalls = 1000000000ull;
    c3.itmax = 4;
    c3.ita = 3;
    c3.tau_rel = 1e-12;
    c3.lower.assign(6, 0.0);
    c3.upper.assign(6, 1.0);
    c3.rng = mcubes::gpu::RngKind::philox;
    const SharpGauss fg{1.0 / (2.0 * sg * sg), std::pow(2.0 * M_PI * sg * sg, -3.0)};
    (void)mcubes::integrate(fg, c3);  // warm-up (module load)
    const auto t0 = std::chrono::steady_clock::now();
    const auto r3 = mcubes::integrate(fg, c3);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const double truth = std::pow(std::erf(0.5 / (sg * std::sqrt(2.0))), 6.0);
    std::printf("C3SHARP estimate %.17g sigma %.17g truth %.17g iterations %u evals_per_s %.6g\n", r3.estimate, r3.sigma,
                truth, r3.iterations_used, static_cast<double>(r3.total_samples) / secs);
  }

  // checkpoint / resume through the C++ API: 2 iterations, then the rest
  {
    mcubes::RunConfig rc = cfg;
    rc.tau_rel = 1e-12;
    rc.itmax = 6;
    rc.ita = 4;
    std::vector<mcubes::Grid> grids;
    const auto full = mcubes::integrate(Bump{1.0 / 50.0}, rc, [&](const mcubes::IterationView& v) { grids.push_back(v.grid); });
    mcubes::RunConfig first = rc;
    first.itmax = 2;
    first.ita = 2;
    const auto part = mcubes::integrate(Bump{1.0 / 50.0}, first);
    const auto res2 = mcubes::integrate_resume(Bump{1.0 / 50.0}, rc, grids[1], part.history);
    std::printf("RESUME same %d\n", res2.estimate == full.estimate && res2.sigma == full.sigma ? 1 : 0);
  }
  return 0;
}
