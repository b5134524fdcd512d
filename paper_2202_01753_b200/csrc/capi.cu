// SPDX-License-Identifier: Apache-2.0
//
// The C ABI of include/mcubes_b200.h over the C++ engine
// (include/mcubes_b200/mcubes.cuh).  Exceptions map to status codes the way
// the reference's error types split: std::invalid_argument ->
// MCB_EINVAL, NonFiniteSample -> MCB_ENONFINITE (+ mcb_last_nonfinite),
// CUDA failures -> MCB_ECUDA.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "mcubes_b200.h"
#include "registry.cuh"

using mcubes::gpu::Context;
using mcubes::gpu::DevBuf;
using mcubes::gpu::IntegrandOps;
using mcubes::gpu::RngKind;

struct mcb_ctx {
  std::unique_ptr<Context> ctx;
  std::string err;
  std::vector<double> nf_x;
  double nf_fx = 0.0;
  DevBuf<double> params;  // device copy of the last integrand's params
};

struct mcb_run {
  mcb_ctx* owner = nullptr;
  DevBuf<double> params;
  std::unique_ptr<mcubes::gpu::Run> run;
  mcubes::RunConfig cfg;
};

namespace {

template <class Fn>
int guarded(mcb_ctx* c, Fn&& fn) {
  try {
    fn();
    return MCB_OK;
  } catch (const mcubes::NonFiniteSample& e) {
    if (c) {
      c->err = e.what();
      c->nf_x = e.point();
      c->nf_fx = e.value();
    }
    return MCB_ENONFINITE;
  } catch (const std::invalid_argument& e) {
    if (c) c->err = e.what();
    return MCB_EINVAL;
  } catch (const mcubes::gpu::CudaError& e) {
    if (c) c->err = e.what();
    return MCB_ECUDA;
  } catch (const std::exception& e) {
    if (c) c->err = e.what();
    return MCB_EINTERNAL;
  }
}

IntegrandOps builtin_ops(Context& ctx, DevBuf<double>& pbuf, const mcb_integrand* f, std::uint32_t dims,
                         RngKind rng) {
  namespace abi = mcubes::gpu::abi;
  if (!f) throw std::invalid_argument("integrand must not be null");
  abi::BuiltinArgs a{dims, nullptr, f->params, f->n_params};
  if (f->n_params && !f->params) throw std::invalid_argument("integrand params pointer is null");
  switch (f->id) {
    case MCB_F1: return abi::ops_F1(f->id, rng, a);
    case MCB_F2: return abi::ops_F2(f->id, rng, a);
    case MCB_F3: return abi::ops_F3(f->id, rng, a);
    case MCB_F4: return abi::ops_F4(f->id, rng, a);
    case MCB_F5: return abi::ops_F5(f->id, rng, a);
    case MCB_F6: return abi::ops_F6(f->id, rng, a);
    case MCB_FA: return abi::ops_FA(f->id, rng, a);
    case MCB_FB: return abi::ops_FB(f->id, rng, a);
    case MCB_TABLE: {
      if (f->n_params < 1) throw std::invalid_argument("table integrand needs params");
      const auto n = static_cast<std::uint32_t>(f->params[0]);
      if (n < 2 || f->n_params != 1 + 2 * dims + static_cast<std::size_t>(n) * dims)
        throw std::invalid_argument("table integrand: bad params");
      double* d = pbuf.ensure(f->n_params);
      MCB_CUDA(cudaMemcpyAsync(d, f->params, sizeof(double) * f->n_params, cudaMemcpyHostToDevice, ctx.stream()));
      a.dev_params = d;
      return abi::ops_Table(f->id, rng, a);
    }
    case MCB_T_X0: case MCB_T_CONST: case MCB_T_X0SQ_HALF: case MCB_T_INF_X0POS: case MCB_T_INF: case MCB_T_ZERO:
    case MCB_T_INF_NEAR_ORIGIN:
      if (rng != RngKind::compat) throw std::invalid_argument("test integrands support the compat stream only");
      if (dims > 10) throw std::invalid_argument("test integrands are compiled for dims <= 10");
      return abi::ops_Tests(f->id, rng, a);
    default:
      throw std::invalid_argument("unknown integrand id " + std::to_string(f->id));
  }
}

mcubes::Grid host_grid(std::uint32_t dims, std::uint32_t nb, const double* lower, const double* upper,
                       const double* edges) {
  if (!lower || !upper) throw std::invalid_argument("Grid: bounds must have one entry per axis");
  if (dims == 0) throw std::invalid_argument("Grid: dims must be >= 1");
  std::vector<double> lo(lower, lower + dims), hi(upper, upper + dims);
  mcubes::Grid uniform(dims, nb, lo, hi);
  if (!edges) return uniform;
  return mcubes::Grid::from_edges(dims, nb, lo, hi, std::vector<double>(edges, edges + std::size_t{dims} * nb));
}

mcubes::RunConfig to_cfg(const mcb_config* c) {
  if (!c) throw std::invalid_argument("config must not be null");
  mcubes::RunConfig cfg;
  cfg.dims = c->dims;
  cfg.n_bins = c->n_bins;
  cfg.maxcalls = c->maxcalls;
  cfg.itmax = c->itmax;
  cfg.ita = c->ita;
  cfg.tau_rel = c->tau_rel;
  cfg.alpha = c->alpha;
  cfg.chi2_dof_max = c->chi2_dof_max;
  cfg.seed = c->seed;
  cfg.variant = c->variant == MCB_VARIANT_MCUBES1D ? mcubes::Variant::mcubes1d : mcubes::Variant::mcubes;
  if (c->dims && (!c->lower || !c->upper)) throw std::invalid_argument("RunConfig: bounds must have one entry per axis");
  if (c->lower) cfg.lower.assign(c->lower, c->lower + c->dims);
  if (c->upper) cfg.upper.assign(c->upper, c->upper + c->dims);
  cfg.workers = c->workers;
  if (c->rng != MCB_RNG_COMPAT && c->rng != MCB_RNG_PHILOX && c->rng != MCB_RNG_PHILOX_EXACT)
    throw std::invalid_argument("RunConfig: unknown rng " + std::to_string(c->rng));
  cfg.rng = static_cast<RngKind>(c->rng);
  return cfg;
}

void fill_result(const mcubes::IntegrationResult& r, mcb_result* out, mcb_iteration* hist, std::uint32_t cap) {
  if (out) {
    out->estimate = r.estimate;
    out->sigma = r.sigma;
    out->chi2_dof = r.chi2_dof;
    out->iterations_used = r.iterations_used;
    out->converged = r.converged ? 1 : 0;
    out->total_samples = r.total_samples;
    out->bin_writes = r.bin_writes;
    out->g = r.params.g;
    out->m = r.params.m;
    out->p = r.params.p;
    out->s = r.params.s;
  }
  if (hist)
    for (std::uint32_t i = 0; i < r.history.size() && i < cap; ++i)
      hist[i] = mcb_iteration{r.history[i].estimate, r.history[i].variance, r.history[i].index, 0};
}

int v_sample_impl(mcb_ctx* c, const mcb_integrand* f, uint32_t dims, uint32_t n_bins, const double* lower,
                  const double* upper, const double* edges, uint64_t m, uint64_t s, uint64_t p, uint64_t seed,
                  uint64_t iteration, int32_t bin_axes_mode, RngKind rng, double* est, double* var,
                  double* contrib, uint64_t* writes) {
  if (!c) return MCB_EINVAL;
  return guarded(c, [&] {
    Context& ctx = *c->ctx;
    ctx.activate();
    const mcubes::Grid grid = host_grid(dims, n_bins, lower, upper, edges);
    const IntegrandOps ops = builtin_ops(ctx, c->params, f, dims, rng);
    std::uint32_t bin_axes = 0;
    if (bin_axes_mode >= 0) bin_axes = bin_axes_mode == MCB_BIN_AXIS0_ONLY ? 1u : dims;
    auto r = mcubes::gpu::sample_once(ctx, ops, grid, m, s, p, seed, iteration, bin_axes);
    if (est) *est = r.est;
    if (var) *var = r.var;
    if (contrib && bin_axes) std::memcpy(contrib, r.contrib.data(), sizeof(double) * r.contrib.size());
    if (writes) *writes = r.writes;  // device-counted deposits (sampler.hpp:116-119)
  });
}

}  // namespace

extern "C" {

int mcb_abi_version(void) { return MCB_ABI_VERSION; }

int mcb_ctx_create(int device, mcb_ctx** out) {
  if (!out) return MCB_EINVAL;
  *out = nullptr;
  auto c = std::make_unique<mcb_ctx>();
  const int rc = guarded(c.get(), [&] { c->ctx = std::make_unique<Context>(device); });
  if (rc == MCB_OK) *out = c.release();
  return rc;
}

int mcb_ctx_destroy(mcb_ctx* c) {
  delete c;
  return MCB_OK;
}

int mcb_ctx_set_stream(mcb_ctx* c, void* stream) {
  if (!c) return MCB_EINVAL;
  c->ctx->set_stream(static_cast<cudaStream_t>(stream));
  return MCB_OK;
}

int mcb_ctx_synchronize(mcb_ctx* c) {
  if (!c) return MCB_EINVAL;
  return guarded(c, [&] { c->ctx->sync(); });
}

uint64_t mcb_ctx_launches(const mcb_ctx* c) { return c ? c->ctx->launches : 0; }

const char* mcb_last_error(const mcb_ctx* c) { return c ? c->err.c_str() : "null context"; }

int mcb_last_nonfinite(const mcb_ctx* c, double* x, uint32_t cap, double* fx) {
  if (!c) return MCB_EINVAL;
  if (x)
    for (std::uint32_t i = 0; i < cap && i < c->nf_x.size(); ++i) x[i] = c->nf_x[i];
  if (fx) *fx = c->nf_fx;
  return MCB_OK;
}

int mcb_v_sample(mcb_ctx* c, const mcb_integrand* f, uint32_t dims, uint32_t n_bins, const double* lower,
                 const double* upper, const double* edges, uint64_t m, uint64_t s, uint64_t p, uint64_t seed,
                 uint64_t iteration, int32_t bin_update, double* est, double* var, double* contrib,
                 uint64_t* writes) {
  return v_sample_impl(c, f, dims, n_bins, lower, upper, edges, m, s, p, seed, iteration,
                       bin_update == MCB_BIN_AXIS0_ONLY ? MCB_BIN_AXIS0_ONLY : MCB_BIN_ALL_AXES, RngKind::compat,
                       est, var, contrib, writes);
}

int mcb_v_sample_philox(mcb_ctx* c, const mcb_integrand* f, uint32_t dims, uint32_t n_bins, const double* lower,
                        const double* upper, const double* edges, uint64_t m, uint64_t s, uint64_t p,
                        uint64_t seed, uint64_t iteration, int32_t bin_update, double* est, double* var,
                        double* contrib, uint64_t* writes) {
  const int32_t mode = bin_update == MCB_BIN_NONE ? -1
                       : bin_update == MCB_BIN_AXIS0_ONLY ? MCB_BIN_AXIS0_ONLY : MCB_BIN_ALL_AXES;
  return v_sample_impl(c, f, dims, n_bins, lower, upper, edges, m, s, p, seed, iteration, mode, RngKind::philox,
                       est, var, mode < 0 ? nullptr : contrib, mode < 0 ? nullptr : writes);
}

int mcb_v_sample_rng(mcb_ctx* c, const mcb_integrand* f, int32_t rng, uint32_t dims, uint32_t n_bins,
                     const double* lower, const double* upper, const double* edges, uint64_t m, uint64_t s,
                     uint64_t p, uint64_t seed, uint64_t iteration, int32_t bin_update, double* est, double* var,
                     double* contrib, uint64_t* writes) {
  if (rng != MCB_RNG_COMPAT && rng != MCB_RNG_PHILOX && rng != MCB_RNG_PHILOX_EXACT) {
    if (c) c->err = "unknown rng " + std::to_string(rng);
    return MCB_EINVAL;
  }
  const int32_t mode = bin_update == MCB_BIN_NONE ? -1
                       : bin_update == MCB_BIN_AXIS0_ONLY ? MCB_BIN_AXIS0_ONLY : MCB_BIN_ALL_AXES;
  return v_sample_impl(c, f, dims, n_bins, lower, upper, edges, m, s, p, seed, iteration, mode,
                       static_cast<RngKind>(rng), est, var, mode < 0 ? nullptr : contrib, mode < 0 ? nullptr : writes);
}

int mcb_v_sample_no_adjust(mcb_ctx* c, const mcb_integrand* f, uint32_t dims, uint32_t n_bins,
                           const double* lower, const double* upper, const double* edges, uint64_t m, uint64_t s,
                           uint64_t p, uint64_t seed, uint64_t iteration, double* est, double* var) {
  return v_sample_impl(c, f, dims, n_bins, lower, upper, edges, m, s, p, seed, iteration, -1, RngKind::compat, est,
                       var, nullptr, nullptr);
}

int mcb_grid_adjust(mcb_ctx* c, uint32_t dims, uint32_t n_bins, const double* lower, const double* upper,
                    const double* edges, const double* contrib, double alpha, int32_t symmetric, double* out) {
  if (!c) return MCB_EINVAL;
  return guarded(c, [&] {
    c->ctx->activate();
    const mcubes::Grid g = host_grid(dims, n_bins, lower, upper, edges);
    if (!contrib || !out) throw std::invalid_argument("contributions and output must not be null");
    mcubes::Grid r = symmetric ? g.adjusted_symmetric(std::span<const double>(contrib, n_bins), alpha)
                               : g.adjusted(mcubes::BinAccumulator(dims, n_bins,
                                                                   std::vector<double>(contrib, contrib + std::size_t{dims} * n_bins), 0),
                                            alpha);
    std::memcpy(out, r.raw_edges().data(), sizeof(double) * r.raw_edges().size());
  });
}

int mcb_setup(const mcb_config* cfg, uint64_t* g, uint64_t* m, uint64_t* p, uint64_t* s) {
  return guarded(nullptr, [&] {
    const auto sp = mcubes::setup(to_cfg(cfg));
    if (g) *g = sp.g;
    if (m) *m = sp.m;
    if (p) *p = sp.p;
    if (s) *s = sp.s;
  });
}

int mcb_set_batch_size(uint64_t m, uint32_t workers, uint64_t* s) {
  return guarded(nullptr, [&] { *s = mcubes::set_batch_size(m, workers); });
}

int mcb_weighted_estimate(uint32_t n, const double* e, const double* v, double* est, double* sigma, double* chi2) {
  return guarded(nullptr, [&] {
    std::vector<mcubes::IterationResult> h;
    for (std::uint32_t i = 0; i < n; ++i) h.push_back({e[i], v[i], i + 1});
    const auto cmb = mcubes::weighted_estimate(h);
    *est = cmb.estimate;
    *sigma = cmb.sigma;
    *chi2 = cmb.chi2_dof;
  });
}

int mcb_check_convergence(double est, double sigma, double chi2, double tau, double chi2max) {
  return mcubes::gpu::converged_dev(est, sigma, chi2, tau, chi2max) ? 1 : 0;
}

int mcb_grid_uniform(uint32_t dims, uint32_t n_bins, const double* lower, const double* upper, double* edges) {
  return guarded(nullptr, [&] {
    const mcubes::Grid g = host_grid(dims, n_bins, lower, upper, nullptr);
    std::memcpy(edges, g.raw_edges().data(), sizeof(double) * g.raw_edges().size());
  });
}

int mcb_integrate(mcb_ctx* c, const mcb_integrand* f, const mcb_config* cfgp, mcb_result* result,
                  mcb_iteration* history, uint32_t cap, mcb_observer observer, void* user) {
  return mcb_integrate_resume(c, f, cfgp, nullptr, nullptr, 0, result, history, cap, observer, user);
}

int mcb_integrate_resume(mcb_ctx* c, const mcb_integrand* f, const mcb_config* cfgp, const double* edges,
                         const mcb_iteration* done, uint32_t n_done, mcb_result* result, mcb_iteration* history,
                         uint32_t cap, mcb_observer observer, void* user) {
  if (!c) return MCB_EINVAL;
  return guarded(c, [&] {
    Context& ctx = *c->ctx;
    ctx.activate();
    const mcubes::RunConfig cfg = to_cfg(cfgp);
    cfg.validate();
    const IntegrandOps ops = builtin_ops(ctx, c->params, f, cfg.dims, cfg.rng);
    mcubes::IterationObserver obs;
    if (observer)
      obs = [&](const mcubes::IterationView& v) {
        mcb_iteration_view cv{};
        cv.iteration = v.iteration;
        cv.adjusting = v.adjusting ? 1 : 0;
        cv.result = mcb_iteration{v.result.estimate, v.result.variance, v.result.index, 0};
        cv.running_estimate = v.running.estimate;
        cv.running_sigma = v.running.sigma;
        cv.running_chi2_dof = v.running.chi2_dof;
        cv.grid_edges = v.grid.raw_edges().data();
        cv.bin_writes = v.bin_writes;
        observer(&cv, user);
      };
    if (!edges) {
      if (n_done) throw std::invalid_argument("resume: completed iterations need the grid they produced");
      fill_result(mcubes::gpu::integrate_ops(ctx, ops, cfg, obs), result, history, cap);
      return;
    }
    if (n_done && !done) throw std::invalid_argument("resume: null history");
    const mcubes::Grid grid = host_grid(cfg.dims, cfg.n_bins, cfg.lower.data(), cfg.upper.data(), edges);
    std::vector<mcubes::IterationResult> h(n_done);
    for (std::uint32_t i = 0; i < n_done; ++i) h[i] = {done[i].estimate, done[i].variance, done[i].index};
    fill_result(mcubes::gpu::integrate_ops(ctx, ops, cfg, obs, &grid, h), result, history, cap);
  });
}

int mcb_run_create(mcb_ctx* c, const mcb_integrand* f, const mcb_config* cfgp, mcb_run** out) {
  if (!c || !out) return MCB_EINVAL;
  *out = nullptr;
  auto r = std::make_unique<mcb_run>();
  r->owner = c;
  const int rc = guarded(c, [&] {
    Context& ctx = *c->ctx;
    ctx.activate();
    r->cfg = to_cfg(cfgp);
    r->cfg.validate();
    const IntegrandOps ops = builtin_ops(ctx, r->params, f, r->cfg.dims, r->cfg.rng);
    r->run = std::make_unique<mcubes::gpu::Run>(ctx, ops, r->cfg);
  });
  if (rc == MCB_OK) *out = r.release();
  return rc;
}

int mcb_run_destroy(mcb_run* r) {
  delete r;
  return MCB_OK;
}

uint64_t mcb_run_exchange_words(const mcb_run* r, uint32_t it) {
  if (!r) return 0;
  return it ? r->run->exchange_words_for(it) : r->run->exchange_words(0);
}

int mcb_run_set_exchange(mcb_run* r, void* p) {
  if (!r) return MCB_EINVAL;
  r->run->set_exchange(static_cast<unsigned long long*>(p));
  return MCB_OK;
}

void* mcb_run_exchange_ptr(const mcb_run* r) { return r ? r->run->exchange() : nullptr; }

int mcb_run_resume(mcb_run* r, const double* edges, const mcb_iteration* done, uint32_t n_done,
                   uint32_t* next_iteration) {
  if (!r || !edges || (n_done && !done)) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    r->owner->ctx->activate();
    const mcubes::Grid grid = host_grid(r->cfg.dims, r->cfg.n_bins, r->cfg.lower.data(), r->cfg.upper.data(), edges);
    std::vector<mcubes::IterationResult> h(n_done);
    for (std::uint32_t i = 0; i < n_done; ++i) h[i] = {done[i].estimate, done[i].variance, done[i].index};
    const std::uint32_t next = r->run->resume(grid, h);
    if (next_iteration) *next_iteration = next;
  });
}

int mcb_run_set_progress(mcb_run* r, int* host_flags) {
  if (!r) return MCB_EINVAL;
  r->run->set_host_flags(host_flags);
  return MCB_OK;
}

int mcb_run_set_peers(mcb_run* r, int rank, int npeers, void* const* bufs_odd, void* const* bufs_even,
                      void* const* flags, void* counter) {
  if (!r || (npeers && (!bufs_odd || !bufs_even || !flags || !counter))) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    r->run->set_peers(rank, npeers, reinterpret_cast<unsigned long long* const*>(bufs_odd),
                      reinterpret_cast<unsigned long long* const*>(bufs_even),
                      reinterpret_cast<unsigned long long* const*>(flags), static_cast<unsigned int*>(counter));
  });
}

int mcb_dev_alloc(mcb_ctx* c, uint64_t bytes, void** ptr) {
  if (!c || !ptr || !bytes) return MCB_EINVAL;
  return guarded(c, [&] {
    c->ctx->activate();
    void* p = nullptr;
    MCB_CUDA(cudaMalloc(&p, bytes));
    MCB_CUDA(cudaMemset(p, 0, bytes));
    MCB_CUDA(cudaDeviceSynchronize());
    *ptr = p;
  });
}

int mcb_dev_free(mcb_ctx* c, void* ptr) {
  if (!c) return MCB_EINVAL;
  return guarded(c, [&] {
    c->ctx->activate();
    MCB_CUDA(cudaFree(ptr));
  });
}

int mcb_ipc_handle(mcb_ctx* c, void* ptr, unsigned char* handle) {
  if (!c || !ptr || !handle) return MCB_EINVAL;
  return guarded(c, [&] {
    c->ctx->activate();
    cudaIpcMemHandle_t h;
    MCB_CUDA(cudaIpcGetMemHandle(&h, ptr));
    static_assert(sizeof h == MCB_IPC_HANDLE_BYTES);
    std::memcpy(handle, &h, sizeof h);
  });
}

int mcb_ipc_open(mcb_ctx* c, const unsigned char* handle, void** ptr) {
  if (!c || !handle || !ptr) return MCB_EINVAL;
  return guarded(c, [&] {
    c->ctx->activate();
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    MCB_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int mcb_ipc_close(mcb_ctx* c, void* ptr) {
  if (!c || !ptr) return MCB_EINVAL;
  return guarded(c, [&] {
    c->ctx->activate();
    MCB_CUDA(cudaIpcCloseMemHandle(ptr));
  });
}

int mcb_run_failure_key(mcb_run* r, int* failed, uint64_t* key) {
  if (!r || !failed || !key) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    r->owner->ctx->activate();
    unsigned long long k = ~0ull;
    *failed = r->run->failure_key(k) ? 1 : 0;
    *key = k;
  });
}

int mcb_run_set_failure_key(mcb_run* r, uint64_t key) {
  if (!r) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    r->owner->ctx->activate();
    r->run->set_failure_key(key);
  });
}

uint64_t mcb_run_work_items(const mcb_run* r) { return r ? r->run->params().m : 0; }

int mcb_run_sample(mcb_run* r, uint32_t it, uint64_t n0, uint64_t n1) {
  if (!r) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    if (it < 1 || it > r->cfg.itmax) throw std::invalid_argument("iteration out of range");
    r->run->sample(it, n0, n1);
  });
}

int mcb_run_reduce(mcb_run* r, uint32_t it) {
  if (!r) return MCB_EINVAL;
  return guarded(r->owner, [&] { r->run->reduce(it); });
}

int mcb_run_finish(mcb_run* r, uint32_t it) {
  if (!r) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    if (it < 1 || it > r->cfg.itmax) throw std::invalid_argument("iteration out of range");
    r->run->finish(it);
  });
}

uint64_t mcb_run_compact_len(const mcb_run* r) { return r ? r->run->compact_len() : 0; }

int mcb_run_round_local(mcb_run* r, uint32_t it, double* out) {
  if (!r || !out) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    if (it < 1 || it > r->cfg.itmax) throw std::invalid_argument("iteration out of range");
    r->run->round_local(it, out);
  });
}

int mcb_run_combine(mcb_run* r, uint32_t it, const double* gathered, int nranks) {
  if (!r || !gathered) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    if (it < 1 || it > r->cfg.itmax) throw std::invalid_argument("iteration out of range");
    r->run->combine(it, gathered, nranks);
  });
}

int mcb_run_finish_rounded(mcb_run* r, uint32_t it) {
  if (!r) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    if (it < 1 || it > r->cfg.itmax) throw std::invalid_argument("iteration out of range");
    r->run->finish_rounded(it);
  });
}

int mcb_run_result(mcb_run* r, mcb_result* result, mcb_iteration* history, uint32_t cap) {
  if (!r) return MCB_EINVAL;
  return guarded(r->owner, [&] { fill_result(r->run->result(), result, history, cap); });
}

int mcb_run_set_grid(mcb_run* r, const double* edges) {
  if (!r || !edges) return MCB_EINVAL;
  return guarded(r->owner, [&] { r->run->set_grid(edges); });
}

int mcb_run_grid(mcb_run* r, double* edges) {
  if (!r) return MCB_EINVAL;
  return guarded(r->owner, [&] {
    const auto g = r->run->grid();
    std::memcpy(edges, g.raw_edges().data(), sizeof(double) * g.raw_edges().size());
  });
}

}  // extern "C"
