// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY -- never linked into or called by the product.
//
// A C-ABI shim over the UNMODIFIED reference headers (compiled from where they
// lie, -I/root/reference/proj/include; nothing is copied into this repo).
// Built by oracle/Makefile into oracle/_ref/libmcubes_ref.so.  Used by:
//   * tests/golden/gen_golden.py to produce the committed golden fixtures,
//   * tests/ to pin oracle/mcubes_oracle.c (the C restatement) to the
//     reference bit for bit,
//   * bench.py --impl reference (the reference CPU arm) and bench.py's
//     cpu_baseline leg (kind "reference").
//
// Integrand ids match include/mcubes_b200.h (mcb_integrand_id).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "mcubes/mcubes.hpp"

using namespace mcubes;

namespace {

// CPU twin of the table integrand (BASELINE config 4, no reference
// implementation exists: PAPER.md:332-338).  Layout of params:
//   [n, lo_0..lo_{d-1}, inv_h_0..inv_h_{d-1}, T_0[0..n), ..., T_{d-1}[0..n)]
// f(x) = prod_j lerp(T_j, (x_j - lo_j) * inv_h_j), evaluated in axis order.
struct TableFn {
  std::uint32_t d;
  const double* params;
  double operator()(std::span<const double> x) const {
    const auto n = static_cast<std::uint32_t>(params[0]);
    const double* lo = params + 1;
    const double* inv_h = params + 1 + d;
    const double* tab = params + 1 + 2 * d;
    double prod = 1.0;
    for (std::uint32_t j = 0; j < d; ++j) {
      const double t = (x[j] - lo[j]) * inv_h[j];
      std::uint32_t k = 0;
      if (t >= static_cast<double>(n - 1)) k = n - 2;
      else if (t > 0.0) k = static_cast<std::uint32_t>(t);
      if (k > n - 2) k = n - 2;
      const double* row = tab + static_cast<std::size_t>(j) * n;
      const double frac = t - static_cast<double>(k);
      const double v = row[k] + frac * (row[k + 1] - row[k]);
      prod *= v;
    }
    return prod;
  }
};

std::function<double(std::span<const double>)> make_fn(int id, const double* params,
                                                        std::uint32_t nparams, std::uint32_t d) {
  switch (id) {
    case 1: case 2: case 3: case 4: case 5: case 6:
      return make_suite_integrand(id, d).evaluate;
    case 7: return make_fA().evaluate;
    case 8: return make_fB().evaluate;
    case 9: {
      if (nparams < 1) throw std::invalid_argument("table integrand needs params");
      const auto n = static_cast<std::uint32_t>(params[0]);
      if (n < 2 || nparams != 1 + 2 * d + static_cast<std::size_t>(n) * d)
        throw std::invalid_argument("table integrand: bad params");
      return TableFn{d, params};
    }
    case 32: return [](std::span<const double> x) { return x[0]; };
    case 33: {
      const double c = nparams ? params[0] : 0.0;
      return [c](std::span<const double>) { return c; };
    }
    case 34: return [](std::span<const double> x) { return x[0] * x[0] + 0.5; };
    case 35:
      return [](std::span<const double> x) {
        return x[0] > 0.0 ? std::numeric_limits<double>::infinity() : 1.0;
      };
    case 36: return [](std::span<const double>) { return std::numeric_limits<double>::infinity(); };
    case 37: return [](std::span<const double>) { return 0.0; };
    default: throw std::invalid_argument("unknown integrand id " + std::to_string(id));
  }
}

Grid make_grid(std::uint32_t d, std::uint32_t nb, const double* lower, const double* upper,
               const double* edges) {
  if (!edges) {
    return Grid(d, nb, std::span<const double>(lower, d), std::span<const double>(upper, d));
  }
  std::ostringstream os;
  os.precision(17);
  os << d << ' ' << nb << '\n';
  for (std::uint32_t j = 0; j < d; ++j) {
    os << lower[j] << ' ' << upper[j];
    for (std::uint32_t i = 0; i < nb; ++i) os << ' ' << edges[std::size_t{j} * nb + i];
    os << '\n';
  }
  std::istringstream is(os.str());
  return Grid::read(is);
}

void copy_edges(const Grid& g, double* out) {
  for (std::uint32_t j = 0; j < g.dims(); ++j) {
    const auto row = g.edges(j);
    std::memcpy(out + std::size_t{j} * g.n_bins(), row.data(), sizeof(double) * g.n_bins());
  }
}

thread_local std::string g_err;

template <class Fn>
int guarded(Fn&& fn, double* err_x, double* err_fx) {
  try {
    fn();
    return 0;
  } catch (const NonFiniteSample& e) {
    g_err = e.what();
    if (err_x) std::memcpy(err_x, e.point().data(), sizeof(double) * e.point().size());
    if (err_fx) *err_fx = e.value();
    return -2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -9;
  }
}

RunConfig make_cfg(std::uint32_t d, std::uint32_t nb, std::uint64_t maxcalls, std::uint32_t itmax,
                   std::uint32_t ita, double tau, double alpha, double chi2max, std::uint64_t seed,
                   int variant, const double* lower, const double* upper, unsigned workers) {
  RunConfig cfg;
  cfg.dims = d;
  cfg.n_bins = nb;
  cfg.maxcalls = maxcalls;
  cfg.itmax = itmax;
  cfg.ita = ita;
  cfg.tau_rel = tau;
  cfg.alpha = alpha;
  cfg.chi2_dof_max = chi2max;
  cfg.seed = seed;
  cfg.variant = variant ? Variant::mcubes1d : Variant::mcubes;
  cfg.lower.assign(lower, lower + d);
  cfg.upper.assign(upper, upper + d);
  cfg.workers = workers;
  return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

double ref_uniform01(std::uint64_t seed, std::uint64_t iter, std::uint64_t cube,
                     std::uint64_t sample, std::uint64_t axis) {
  return uniform01(SampleKey{seed, iter, cube, sample, axis});
}

std::uint64_t ref_iteration_root(std::uint64_t seed, std::uint64_t iter) {
  return detail::iteration_root(seed, iter);
}

double ref_exact_sum(const double* v, std::uint64_t n) {
  ExactSum s;
  for (std::uint64_t i = 0; i < n; ++i) s.add(v[i]);
  return s.value();
}

double ref_reference_value(int family, std::uint32_t d) {
  switch (family) {
    case 7: return *make_fA().reference;
    case 8: return *make_fB().reference;
    default: return reference_value(family, d);
  }
}

int ref_eval(int id, const double* params, std::uint32_t nparams, std::uint32_t d,
             const double* x, double* out) {
  return guarded([&] { *out = make_fn(id, params, nparams, d)(std::span<const double>(x, d)); },
                 nullptr, nullptr);
}

int ref_transform(std::uint32_t d, std::uint32_t nb, const double* lower, const double* upper,
                  const double* edges, const double* u, double* x, std::uint32_t* bins,
                  double* jac) {
  return guarded(
      [&] {
        const Grid g = make_grid(d, nb, lower, upper, edges);
        *jac = g.transform(std::span<const double>(u, d), std::span<double>(x, d),
                           std::span<std::uint32_t>(bins, d));
      },
      nullptr, nullptr);
}

// mode: 0 = v_sample all_axes, 1 = v_sample axis0_only, 2 = v_sample_no_adjust,
//       3 = vegas_serial_iteration all_axes, 4 = vegas_serial_iteration axis0_only
int ref_v_sample(int id, const double* params, std::uint32_t nparams, std::uint32_t d,
                 std::uint32_t nb, const double* lower, const double* upper, const double* edges,
                 std::uint64_t m, std::uint64_t s, std::uint64_t p, std::uint64_t seed,
                 std::uint64_t iteration, int mode, unsigned max_threads, double* est, double* var,
                 double* contrib, std::uint64_t* writes, double* err_x, double* err_fx) {
  return guarded(
      [&] {
        const auto f = make_fn(id, params, nparams, d);
        const Grid g = make_grid(d, nb, lower, upper, edges);
        if (mode == 2) {
          const EstimateVariance ev = v_sample_no_adjust(f, g, m, s, p, seed, iteration, max_threads);
          *est = ev.raw_estimate;
          *var = ev.raw_variance;
          return;
        }
        const BinUpdate bu = (mode == 1 || mode == 4) ? BinUpdate::axis0_only : BinUpdate::all_axes;
        const SampleOutcome out = mode >= 3
                                      ? vegas_serial_iteration(f, g, m, p, seed, iteration, bu)
                                      : v_sample(f, g, m, s, p, seed, iteration, bu, max_threads);
        *est = out.raw_estimate;
        *var = out.raw_variance;
        if (writes) *writes = out.contributions.writes();
        if (contrib)
          for (std::uint32_t j = 0; j < d; ++j)
            for (std::uint32_t i = 0; i < nb; ++i)
              contrib[std::size_t{j} * nb + i] = out.contributions.at(j, i);
      },
      err_x, err_fx);
}

int ref_grid_adjust(std::uint32_t d, std::uint32_t nb, const double* lower, const double* upper,
                    const double* edges, const double* contrib, double alpha, int symmetric,
                    double* out) {
  return guarded(
      [&] {
        const Grid g = make_grid(d, nb, lower, upper, edges);
        if (symmetric) {
          copy_edges(g.adjusted_symmetric(std::span<const double>(contrib, nb), alpha), out);
        } else {
          BinAccumulator acc(d, nb, std::vector<double>(contrib, contrib + std::size_t{d} * nb), 0);
          copy_edges(g.adjusted(acc, alpha), out);
        }
      },
      nullptr, nullptr);
}

int ref_setup(std::uint32_t d, std::uint32_t nb, std::uint64_t maxcalls, std::uint32_t itmax,
              std::uint32_t ita, double tau, double alpha, double chi2max, const double* lower,
              const double* upper, unsigned workers, std::uint64_t* out4) {
  return guarded(
      [&] {
        const SetupParams sp =
            setup(make_cfg(d, nb, maxcalls, itmax, ita, tau, alpha, chi2max, 0, 0, lower, upper, workers));
        out4[0] = sp.g;
        out4[1] = sp.m;
        out4[2] = sp.p;
        out4[3] = sp.s;
      },
      nullptr, nullptr);
}

int ref_set_batch_size(std::uint64_t m, unsigned workers, std::uint64_t* out) {
  return guarded([&] { *out = set_batch_size(m, workers); }, nullptr, nullptr);
}

int ref_weighted_estimate(std::uint32_t n, const double* est, const double* var, double* out3) {
  return guarded(
      [&] {
        std::vector<IterationResult> h;
        for (std::uint32_t i = 0; i < n; ++i) h.push_back({est[i], var[i], i + 1});
        const Combined c = weighted_estimate(h);
        out3[0] = c.estimate;
        out3[1] = c.sigma;
        out3[2] = c.chi2_dof;
      },
      nullptr, nullptr);
}

int ref_check_convergence(double estimate, double sigma, double chi2, double tau, double chi2max) {
  RunConfig cfg;
  cfg.tau_rel = tau;
  cfg.chi2_dof_max = chi2max;
  return check_convergence(Combined{estimate, sigma, chi2}, cfg) ? 1 : 0;
}

// Full integrate().  res8 = {estimate, sigma, chi2_dof, iterations_used, converged,
// total_samples, bin_writes, unused}; sp4 = {g, m, p, s}.  hist_est/var hold
// `cap` entries.  If grids_out is non-null it receives, per iteration, the grid
// edges seen by the observer (d*nb doubles each, itmax slots).
int ref_integrate(int id, const double* params, std::uint32_t nparams, std::uint32_t d,
                  std::uint32_t nb, std::uint64_t maxcalls, std::uint32_t itmax, std::uint32_t ita,
                  double tau, double alpha, double chi2max, std::uint64_t seed, int variant,
                  const double* lower, const double* upper, unsigned workers, double* res8,
                  std::uint64_t* sp4, double* hist_est, double* hist_var, std::uint32_t cap,
                  double* grids_out, std::uint64_t* writes_out, double* err_x, double* err_fx) {
  return guarded(
      [&] {
        const auto f = make_fn(id, params, nparams, d);
        const RunConfig cfg =
            make_cfg(d, nb, maxcalls, itmax, ita, tau, alpha, chi2max, seed, variant, lower, upper, workers);
        std::uint32_t k = 0;
        const IntegrationResult r = integrate(f, cfg, [&](const IterationView& v) {
          if (grids_out && k < itmax) copy_edges(v.grid, grids_out + std::size_t{k} * d * nb);
          if (writes_out && k < itmax) writes_out[k] = v.bin_writes;
          ++k;
        });
        res8[0] = r.estimate;
        res8[1] = r.sigma;
        res8[2] = r.chi2_dof;
        res8[3] = r.iterations_used;
        res8[4] = r.converged ? 1.0 : 0.0;
        res8[5] = static_cast<double>(r.total_samples);
        res8[6] = static_cast<double>(r.bin_writes);
        res8[7] = 0.0;
        sp4[0] = r.params.g;
        sp4[1] = r.params.m;
        sp4[2] = r.params.p;
        sp4[3] = r.params.s;
        for (std::uint32_t i = 0; i < r.history.size() && i < cap; ++i) {
          hist_est[i] = r.history[i].estimate;
          hist_var[i] = r.history[i].variance;
        }
      },
      err_x, err_fx);
}

}  // extern "C"
