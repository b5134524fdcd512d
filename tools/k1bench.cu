// K1 micro-benchmark used to choose build-time variants (threads per block,
// to_unit form).  Times vsample_kernel<F4, 8, rng> alone with CUDA events
// and prints evals/s plus the estimate bits (identical across variants).
//   nvcc ... -DMCB_SAMPLE_THREADS=640 tools/k1bench.cu
//   ./k1bench [maxcalls] [reps] [rng: 0 compat, 1 philox] [frozen: 0|1]
#include <cstdio>
#include <cstring>

#include "mcubes_b200/mcubes.cuh"

using namespace mcubes;

int main(int argc, char** argv) {
  const std::uint64_t maxcalls = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000000ull;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
  const int rngk = argc > 3 ? std::atoi(argv[3]) : 0;
  const std::uint32_t bin_axes = (argc > 4 && std::atoi(argv[4])) ? 0u : 8u;
  constexpr int D = 8;
  RunConfig cfg;
  cfg.dims = D;
  cfg.maxcalls = maxcalls;
  cfg.lower.assign(D, 0.0);
  cfg.upper.assign(D, 1.0);
  const SetupParams sp = setup(cfg);
  gpu::Context ctx(0);
  const gpu::Shape sh = gpu::make_shape(D, 50, sp.m, 1, sp.p);
  const Grid g(D, 50, cfg.lower, cfg.upper);
  gpu::upload(ctx, ctx.edges, g.raw_edges().data(), D * 50);
  gpu::upload(ctx, ctx.lower, cfg.lower.data(), D);
  unsigned long long* err = ctx.err_key.ensure(1);
  MCB_CUDA(cudaMemsetAsync(err, 0xff, 8, ctx.stream()));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const gpu::fn::F4 f{};
  gpu::Launch L{};
  for (int w = 0; w < 2; ++w) L = (rngk ? gpu::launch_k1<gpu::fn::F4, D, gpu::RngKind::philox, 50>(ctx, f, sh, bin_axes, 123, 0, sh.m, nullptr, err)
             : gpu::launch_k1<gpu::fn::F4, D, gpu::RngKind::compat, 50>(ctx, f, sh, bin_axes, 123, 0, sh.m, nullptr, err));
  float best = 1e30f, total = 0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0, ctx.stream());
    L = (rngk ? gpu::launch_k1<gpu::fn::F4, D, gpu::RngKind::philox, 50>(ctx, f, sh, bin_axes, 123, 0, sh.m, nullptr, err)
             : gpu::launch_k1<gpu::fn::F4, D, gpu::RngKind::compat, 50>(ctx, f, sh, bin_axes, 123, 0, sh.m, nullptr, err));
    cudaEventRecord(e1, ctx.stream());
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
    total += ms;
  }
  unsigned long long* words = ctx.words.ensure(static_cast<std::size_t>(gpu::exchange_accs(D, 50)) * gpu::kXWords);
  gpu::launch_reduce(ctx, L, bin_axes, 50, words, nullptr);
  double* sc = ctx.scalars.ensure(2);
  double* contrib = ctx.contrib.ensure(D * 50);
  gpu::launch_finish(ctx, sh, bin_axes, words, sc, sc + 1, contrib, nullptr, nullptr);
  double h[2];
  gpu::download(ctx, h, sc, 2);
  ctx.sync();
  std::uint64_t eb, vb;
  std::memcpy(&eb, &h[0], 8);
  std::memcpy(&vb, &h[1], 8);
  const double evals = static_cast<double>(sp.m) * sp.p;
  std::printf("rng=%d frozen=%d threads=%d blocks=%d smem=%zu m=%llu p=%llu best_ms=%.3f avg_ms=%.3f evals/s=%.4e est=%016llx var=%016llx\n",
              rngk, int(bin_axes == 0), rngk ? gpu::sample_threads(gpu::RngKind::philox, 8) : gpu::kSampleThreads, L.blocks, L.smem, (unsigned long long)sp.m, (unsigned long long)sp.p, best,
              total / reps, evals / (best * 1e-3), (unsigned long long)eb, (unsigned long long)vb);
  return 0;
}
