// K1 micro-benchmark used to choose build-time variants (threads per block,
// deposit/transform forms).  Runs the 8D Genz f4 m-Cubes loop through
// gpu::Run (so the grid is ADAPTED, as in bench.py), then times the sampling
// kernel alone with CUDA events over `reps` further adjusting iterations and
// prints evals/s plus the run's final estimate bits (identical across
// variants: the sums are exact).
//   nvcc ... -DMCB_SAMPLE_THREADS_PHILOX=768 tools/k1bench.cu
//   ./k1bench [maxcalls] [reps] [rng: 0 compat, 1 philox, 2 philox with exact bins] [frozen: 0|1] [warm iterations]
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <unistd.h>

#include "mcubes_b200/mcubes.cuh"

using namespace mcubes;

int main(int argc, char** argv) {
  const std::uint64_t maxcalls = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000000ull;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
  const int rngk = argc > 3 ? std::atoi(argv[3]) : 1;
  const bool frozen = argc > 4 && std::atoi(argv[4]);
  const int warm = argc > 5 ? std::atoi(argv[5]) : 4;
  const long long direct_key = argc > 6 ? std::atoll(argv[6]) : -1;  // >= 0: time launch_k1 directly with this key
  constexpr int D = 8;
  RunConfig cfg;
  cfg.dims = D;
  cfg.maxcalls = maxcalls;
  cfg.lower.assign(D, 0.0);
  cfg.upper.assign(D, 1.0);
  cfg.itmax = static_cast<std::uint32_t>(warm + reps);
  cfg.ita = frozen ? static_cast<std::uint32_t>(warm) : cfg.itmax;
  cfg.tau_rel = 1e-15;
  gpu::Context ctx(0);
  const gpu::fn::F4 f{};
  const gpu::IntegrandOps ops = rngk == 2 ? gpu::make_ops<gpu::fn::F4, gpu::RngKind::philox_exact>(f)
                                : rngk ? gpu::make_ops<gpu::fn::F4, gpu::RngKind::philox>(f)
                                       : gpu::make_ops<gpu::fn::F4, gpu::RngKind::compat>(f);
  if (direct_key >= 0) {  // uniform grid, fixed iteration key, no Run
    const SetupParams sp = setup(cfg);
    const gpu::Shape sh = gpu::make_shape(D, 50, sp.m, 1, sp.p);
    const Grid g(D, 50, cfg.lower, cfg.upper);
    gpu::upload(ctx, ctx.edges, g.raw_edges().data(), D * 50);
    gpu::upload(ctx, ctx.lower, cfg.lower.data(), D);
    ctx.grid_edges = ctx.edges.get();
    ctx.grid_lower = ctx.lower.get();
    unsigned long long* err = ctx.err_key.ensure(1);
    MCB_CUDA(cudaMemsetAsync(err, 0xff, 8, ctx.stream()));
    const std::uint64_t key = direct_key == 0 ? gpu::iteration_key(cfg.seed, 1) : static_cast<std::uint64_t>(direct_key);
    cudaEvent_t a0, a1;
    cudaEventCreate(&a0);
    cudaEventCreate(&a1);
    float best = 1e30f;
    const int between = std::getenv("K1_BETWEEN") ? std::atoi(std::getenv("K1_BETWEEN")) : 0;
    const std::size_t nwords = gpu::kXHeader + static_cast<std::size_t>(gpu::exchange_accs(D, 50)) * gpu::kXWords;
    unsigned long long* words = ctx.words.ensure(nwords) + gpu::kXHeader;  // [counts][accumulators]
    for (int r = 0; r < reps + 1; ++r) {
      cudaEventRecord(a0, ctx.stream());
      (void)ops.k1(ctx, sh, frozen ? 0u : D, key, 0, sh.m, nullptr, err, words);
      cudaEventRecord(a1, ctx.stream());
      if (between == 1) cudaMemsetAsync(words - gpu::kXHeader, 0, sizeof(unsigned long long) * nwords, ctx.stream());
      cudaEventSynchronize(a1);
      if (between == 2) usleep(200000);
      float ms;
      cudaEventElapsedTime(&ms, a0, a1);
      std::printf("  r=%d k1_ms=%.3f\n", r, ms);
      if (r) best = ms < best ? ms : best;
    }
    std::printf("direct key=%llx rng=%d best_ms=%.3f evals/s=%.4e\n", (unsigned long long)key, rngk, best,
                static_cast<double>(sp.m) * sp.p / (best * 1e-3));
    return 0;
  }
  gpu::Run run(ctx, ops, cfg);
  for (int it = 1; it <= warm; ++it) {
    run.sample(it);
    run.reduce(it);
    run.finish(it);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f, total = 0;
  for (int r = 0; r < reps; ++r) {
    const int it = warm + 1 + r;
    cudaEventRecord(e0, ctx.stream());
    run.sample(it);
    cudaEventRecord(e1, ctx.stream());
    run.reduce(it);
    run.finish(it);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("  it=%d k1_ms=%.3f\n", it, ms);
    best = ms < best ? ms : best;
    total += ms;
  }
  {  // the same kernel launched directly (no stop flag) on the run's current grid
    unsigned long long* err = ctx.err_key.ensure(1);
    cudaEventRecord(e0, ctx.stream());
    ops.k1(ctx, run.shape(), frozen ? 0u : D, gpu::iteration_key(cfg.seed, 1), 0, run.shape().m, nullptr, err, run.exchange() + 1);
    cudaEventRecord(e1, ctx.stream());
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("  direct-after-run k1_ms=%.3f\n", ms);
    cudaEventRecord(e0, ctx.stream());
    ops.k1(ctx, run.shape(), frozen ? 0u : D, gpu::iteration_key(cfg.seed, 1), 0, run.shape().m, run.stop_flag(), err, run.exchange() + 1);
    cudaEventRecord(e1, ctx.stream());
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("  direct-after-run with stop flag k1_ms=%.3f\n", ms);
  }
  const IntegrationResult res = run.result();
  std::uint64_t eb;
  std::memcpy(&eb, &res.estimate, 8);
  const double evals = static_cast<double>(run.params().m) * run.params().p;
  const int threads = rngk ? gpu::sample_threads(gpu::RngKind::philox, D) : gpu::sample_threads(gpu::RngKind::compat, D);
  std::printf("rng=%d frozen=%d threads=%d m=%llu p=%llu warm=%d best_ms=%.3f avg_ms=%.3f evals/s=%.4e est=%016llx\n",
              rngk, int(frozen), threads, (unsigned long long)run.params().m, (unsigned long long)run.params().p, warm,
              best, total / reps, evals / (best * 1e-3), (unsigned long long)eb);
  return 0;
}
