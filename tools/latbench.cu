// Per-phase device time of one small-ncall iteration (BASELINE C1: 5D f4,
// 1e6 calls) through gpu::Run, CUDA events between the phases.
//   ./latbench [rng 0|1] [maxcalls] [dims]
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "mcubes_b200/mcubes.cuh"

using namespace mcubes;

static int fixed_cost() {
  gpu::Context ctx(0);
  const gpu::fn::F4 f{};
  const gpu::IntegrandOps ops = gpu::make_ops<gpu::fn::F4, gpu::RngKind::philox>(f);
  for (std::uint32_t its : {1u, 2u, 20u}) {
    RunConfig cfg;
    cfg.dims = 5;
    cfg.maxcalls = 1000000;
    cfg.lower.assign(5, 0.0);
    cfg.upper.assign(5, 1.0);
    cfg.itmax = its;
    cfg.ita = its;
    cfg.tau_rel = 1e-15;
    cfg.rng = gpu::RngKind::philox;
    const IntegrationResult res0 = gpu::integrate_ops(ctx, ops, cfg);
    double best = 1e30;
    for (int r = 0; r < 7; ++r) {
      ctx.sync();
      const auto t0 = std::chrono::steady_clock::now();
      (void)gpu::integrate_ops(ctx, ops, cfg);
      best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::uint64_t eb;
    std::memcpy(&eb, &res0.estimate, 8);
    std::printf("C++ integrate_ops itmax=%u: %.1f us  (estimate bits %016llx)\n", its, best * 1e6, (unsigned long long)eb);
  }
  return 0;
}

// Upper bound on what a CUDA graph could save: the C1 loop (10 adjusting
// iterations) enqueued on the stream vs the same launches captured once into
// a graph and replayed (state reset inside; device time with events).
static int graph_gain() {
  gpu::Context ctx(0);
  const gpu::fn::F4 f{};
  const gpu::IntegrandOps ops = gpu::make_ops<gpu::fn::F4, gpu::RngKind::philox>(f);
  RunConfig cfg;
  cfg.dims = 5;
  cfg.maxcalls = 1000000;
  cfg.lower.assign(5, 0.0);
  cfg.upper.assign(5, 1.0);
  cfg.itmax = 10;
  cfg.ita = 10;
  cfg.tau_rel = 1e-15;
  cfg.rng = gpu::RngKind::philox;
  gpu::Run run(ctx, ops, cfg);
  cudaStream_t s = ctx.stream();
  auto body = [&] {
    cudaMemsetAsync(const_cast<int*>(run.stop_flag()) - offsetof(gpu::RunState, stop) / sizeof(int), 0, sizeof(gpu::RunState), s);
    for (std::uint32_t it = 1; it <= cfg.itmax; ++it) {
      run.sample(it);
      run.finish(it);
    }
  };
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed = [&](auto&& fn) {
    float best = 1e30f;
    for (int r = 0; r < 20; ++r) {
      ctx.sync();
      cudaEventRecord(e0, s);
      fn();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    return best * 1e3f;
  };
  const float t_stream = timed(body);
  cudaGraph_t g;
  MCB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  body();
  MCB_CUDA(cudaStreamEndCapture(s, &g));
  cudaGraphExec_t ge;
  const auto t0 = std::chrono::steady_clock::now();
  MCB_CUDA(cudaGraphInstantiate(&ge, g, 0));
  const double inst_us = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e6;
  const float t_graph = timed([&] { MCB_CUDA(cudaGraphLaunch(ge, s)); });
  std::printf("C1 loop (10 iterations, device time): stream %.1f us  graph %.1f us  (instantiate %.1f us host)\n",
              t_stream, t_graph, inst_us);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "fixed") return fixed_cost();
  if (argc > 1 && std::string(argv[1]) == "graph") return graph_gain();
  const int rngk = argc > 1 ? std::atoi(argv[1]) : 1;
  const std::uint64_t maxcalls = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1000000ull;
  const int D = argc > 3 ? std::atoi(argv[3]) : 5;
  RunConfig cfg;
  cfg.dims = D;
  cfg.maxcalls = maxcalls;
  cfg.lower.assign(D, 0.0);
  cfg.upper.assign(D, 1.0);
  cfg.itmax = 40;
  cfg.ita = 40;
  cfg.tau_rel = 1e-15;
  gpu::Context ctx(0);
  const gpu::fn::F4 f{};
  const gpu::IntegrandOps ops = rngk ? gpu::make_ops<gpu::fn::F4, gpu::RngKind::philox>(f)
                                     : gpu::make_ops<gpu::fn::F4, gpu::RngKind::compat>(f);
  gpu::Run run(ctx, ops, cfg);
  cudaEvent_t ev[4];
  for (auto& e : ev) cudaEventCreate(&e);
  double t[3] = {0, 0, 0};
  int n = 0;
  for (int it = 1; it <= 40; ++it) {
    cudaEventRecord(ev[0], ctx.stream());
    run.sample(it);
    cudaEventRecord(ev[1], ctx.stream());
    run.reduce(it);
    cudaEventRecord(ev[2], ctx.stream());
    run.finish(it);
    cudaEventRecord(ev[3], ctx.stream());
    cudaEventSynchronize(ev[3]);
#ifdef MCB_FINISH_TIMING
    if (it == 20) {
      unsigned long long tt[16];
      cudaMemcpyFromSymbol(tt, gpu::g_fin_times, sizeof tt);
      std::printf("finish phases (us from start): blocks done %.2f  last block in %.2f  staged %.2f  adjusted %.2f  end %.2f\n",
                  (tt[1] - tt[0]) * 1e-3, (tt[2] - tt[0]) * 1e-3, (tt[3] - tt[0]) * 1e-3, (tt[4] - tt[0]) * 1e-3,
                  (tt[5] - tt[0]) * 1e-3);
      std::printf("adjust (us from start): staged %.2f smoothed %.2f total %.2f importance %.2f sums %.2f walk %.2f [6] %.2f\n",
                  (tt[8] - tt[0]) * 1e-3, (tt[9] - tt[0]) * 1e-3, (tt[10] - tt[0]) * 1e-3, (tt[11] - tt[0]) * 1e-3,
                  (tt[12] - tt[0]) * 1e-3, (tt[13] - tt[0]) * 1e-3, (tt[14] - tt[0]) * 1e-3);
    }
    {
      unsigned long long z[16] = {};
      cudaMemcpyToSymbol(gpu::g_fin_times, z, sizeof z);
    }
#endif
#ifdef MCB_K1_TIMING
    if (it == 20) {
      unsigned long long tt[8];
      cudaMemcpyFromSymbol(tt, gpu::g_k1_times, sizeof tt);
      auto us = [&](int i) { return (double)(tt[i] - tt[0]) * 1e-3; };
      std::printf("K1 phases (us from first block start): last block start %.2f  prologue done %.2f  first thread done %.2f  "
                  "last block loop done %.2f  flushed %.2f\n", us(1), us(2), us(3), us(4), us(5));
    }
    {
      unsigned long long z[8] = {~0ull, 0, 0, ~0ull, 0, 0, 0, 0};
      cudaMemcpyToSymbol(gpu::g_k1_times, z, sizeof z);
    }
#endif
    if (it > 10) {
      for (int k = 0; k < 3; ++k) {
        float ms;
        cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
        t[k] += ms;
      }
      ++n;
    }
  }
  const IntegrationResult res = run.result();
  std::uint64_t eb;
  std::memcpy(&eb, &res.estimate, 8);
  std::printf("rng=%d D=%d maxcalls=%llu m=%llu p=%llu  per iteration (us): sample %.1f  reduce %.1f  finish %.1f"
              "  estimate bits %016llx\n",
              rngk, D, (unsigned long long)maxcalls, (unsigned long long)run.params().m,
              (unsigned long long)run.params().p, 1e3 * t[0] / n, 1e3 * t[1] / n, 1e3 * t[2] / n,
              (unsigned long long)eb);
  return 0;
}
