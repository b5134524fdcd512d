// SPDX-License-Identifier: Apache-2.0
//
// Host engine: device context, buffers and the launch sequence of one m-Cubes
// iteration (K1 sample + exact cross-block sum into the exchange words ->
// [all-reduce] -> K3b round -> K4 adapt/combine).  Everything here is
// stream-ordered; a whole
// integrate() run is enqueued without a host synchronisation (the device
// `stop` flag turns iterations after convergence into no-ops).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "config.cuh"
#include "epilogue.cuh"
#include "exact.cuh"
#include "integrands.cuh"
#include "rng.cuh"
#include "sampler.cuh"

namespace mcubes::gpu {

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " + file +
                    ":" + std::to_string(line));
}
#define MCB_CUDA(x) ::mcubes::gpu::cuda_check((x), #x, __FILE__, __LINE__)

/// Programmatic dependent launch for the run's kernels (config.cuh
/// pdl_wait/pdl_trigger); MCB_PDL=0 in the environment turns it off.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("MCB_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

/// MCB_K1_CLUSTER=1: K1 in 2-CTA clusters (each CTA flushes half of both CTAs' words over DSMEM).
inline bool k1_cluster_enabled() {  // off by default since round 2 (DESIGN.md section 4 table)
  static const bool on = [] {
    const char* v = std::getenv("MCB_K1_CLUSTER");
    return v && v[0] == '1';
  }();
  return on;
}

/// MCB_FULL_BLOCKS=1: K1 always launches full blocks (A/B timing of the
/// small-problem block sizing; same bits either way).
inline bool full_blocks_forced() {
  static const bool on = [] {
    const char* v = std::getenv("MCB_FULL_BLOCKS");
    return v && v[0] == '1';
  }();
  return on;
}

/// Block-wide grid adaptation in the finish kernel (adjust_grid_par);
/// MCB_ADJ_PAR=0 selects the warp-per-axis form (same bits, for A/B timing).
inline bool adjust_par_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("MCB_ADJ_PAR");
    return !(v && v[0] == '0');
  }();
  return on;
}

/// kern<<<grid, block, smem, stream>>>(args...) with programmatic stream
/// serialisation (the kernel must pdl_wait() before reading its
/// predecessor's output).
/// launch_pdl with thread-block clusters of `cluster` CTAs along x (1: none).
template <class... KArgs, class... Args>
void launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t stream,
                        unsigned cluster, Args&&... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  lc.attrs = at;
  lc.numAttrs = 1;
  if (cluster > 1) {
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cluster;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    lc.numAttrs = 2;
  }
  MCB_CUDA(cudaLaunchKernelEx(&lc, kern, std::forward<Args>(args)...));
}

template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t stream,
                Args&&... args) {
  launch_pdl_cluster(kern, grid, block, smem, stream, 1, std::forward<Args>(args)...);
}



template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  T* ensure(std::size_t n) {
    if (n > cap_) {
      release();
      MCB_CUDA(cudaMalloc(&p_, sizeof(T) * std::max<std::size_t>(n, 1)));
      cap_ = n;
    }
    return p_;
  }
  T* get() const { return p_; }
  std::size_t capacity() const { return cap_; }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    cap_ = 0;
  }

 private:
  T* p_ = nullptr;
  std::size_t cap_ = 0;
};

/// Sampling shape of one iteration (checked like check_sample_args,
/// sampler.hpp:285-295).
struct Shape {
  std::uint32_t dims = 0, nb = 0;
  std::uint64_t m = 0, p = 0, g = 0;
  std::uint64_t A = 0;  ///< 1 + g + ... + g^(d-1) mod m
  double scale = 0, rcp_g = 0, pp1 = 0, rcp_pp1 = 0;
};

/// d-th integer root of m, or 0 (sampler.hpp:184-197).
inline std::uint64_t exact_root(std::uint64_t m, std::uint32_t d) {
  const auto guess = static_cast<std::uint64_t>(
      std::llround(std::pow(static_cast<double>(m), 1.0 / static_cast<double>(d))));
  for (std::uint64_t g = guess > 2 ? guess - 2 : 1; g <= guess + 2; ++g) {
    std::uint64_t acc = 1;
    bool overflow = false;
    for (std::uint32_t i = 0; i < d && !overflow; ++i) {
      if (acc > m / g) overflow = true;
      else acc *= g;
    }
    if (!overflow && acc == m) return g;
  }
  return 0;
}

inline Shape make_shape(std::uint32_t dims, std::uint32_t nb, std::uint64_t m, std::uint64_t s,
                        std::uint64_t p) {
  if (m == 0) throw std::invalid_argument("v_sample: m must be >= 1");
  if (p < 2) throw std::invalid_argument("v_sample: p must be >= 2");
  if (s == 0) throw std::invalid_argument("v_sample: batch size must be >= 1");
  const std::uint64_t g = exact_root(m, dims);
  if (g == 0) throw std::invalid_argument("v_sample: m must be a perfect d-th power of the cube count");
  if (p >= (std::uint64_t{1} << 32))  // K1 keys samples by a 32-bit index (Philox counter word, Welford count)
    throw std::invalid_argument("B200 path: p must be < 2^32 samples per cube");
  if (dims > static_cast<std::uint32_t>(kMaxDims))
    throw std::invalid_argument("B200 path: dims must be <= " + std::to_string(kMaxDims));
  Shape sh;
  sh.dims = dims;
  sh.nb = nb;
  sh.m = m;
  sh.p = p;
  sh.g = g;
  unsigned __int128 A = 0, pw = 1;
  for (std::uint32_t j = 0; j < dims; ++j) {
    A += pw;
    pw *= g;
  }
  sh.A = static_cast<std::uint64_t>(A % m);
  sh.scale = 1.0 / (static_cast<double>(m) * static_cast<double>(p));  // sampler.hpp:293
  sh.rcp_g = 1.0 / static_cast<double>(g);
  sh.pp1 = static_cast<double>(p) * static_cast<double>(p - 1);  // sampler.hpp:178
  sh.rcp_pp1 = 1.0 / sh.pp1;
  return sh;
}

/// Device buffers of one Run (mcubes.cuh): its grid, bounds, contributions,
/// history, state, error key and exchange words -- exclusively its own while
/// it lives, recycled through the Context's pool afterwards (cudaMalloc and
/// the device-synchronising cudaFree cost ~50 us per integrate() call
/// otherwise).
struct RunBufs {
  DevBuf<double> edges, lower, upper, contrib, hist_est, hist_var;
  DevBuf<unsigned long long> words, err_key;
  DevBuf<RunState> state;
  cudaEvent_t released = nullptr;  ///< recorded on the releasing run's stream
  bool pending = false;            ///< `released` marks work a reuser must wait for
  RunBufs() = default;
  RunBufs(const RunBufs&) = delete;
  RunBufs& operator=(const RunBufs&) = delete;
  ~RunBufs() {
    if (released) cudaEventDestroy(released);
  }
};

/// A device context: one CUDA device, one stream, reusable scratch.
/// Use from one host thread at a time; separate contexts may run concurrently.
class Context {
 public:
  explicit Context(int device = -1) {
    if (device < 0) MCB_CUDA(cudaGetDevice(&device));
    device_ = device;
    MCB_CUDA(cudaSetDevice(device_));
    MCB_CUDA(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device_));
    MCB_CUDA(cudaDeviceGetAttribute(&max_smem_, cudaDevAttrMaxSharedMemoryPerBlockOptin, device_));
    MCB_CUDA(cudaStreamCreateWithFlags(&own_stream_, cudaStreamNonBlocking));
    stream_ = own_stream_;
    MCB_CUDA(cudaMallocHost(&pinned_, kPinnedBytes));
    MCB_CUDA(cudaMallocHost(&flags_, sizeof(int) * kMaxFlagIterations));
  }
  ~Context() {
    cudaSetDevice(device_);
    if (own_stream_) cudaStreamDestroy(own_stream_);
    if (pinned_) cudaFreeHost(pinned_);
    if (flags_) cudaFreeHost(flags_);
    if (staging_ev_) cudaEventDestroy(staging_ev_);
    for (cudaEvent_t e : events_) cudaEventDestroy(e);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  int device() const { return device_; }
  int sms() const { return sms_; }
  int max_smem() const { return max_smem_; }
  cudaStream_t stream() const { return stream_; }
  /// Run on a caller-owned stream (e.g. torch's current stream) instead.
  void set_stream(cudaStream_t s) { stream_ = s ? s : own_stream_; }
  void activate() const { MCB_CUDA(cudaSetDevice(device_)); }
  void sync() const { MCB_CUDA(cudaStreamSynchronize(stream_)); }

  /// Number of kernels this context enqueued (our own kernels only).
  std::uint64_t launches = 0;

  /// Scratch of the standalone calls (v_sample, v_sample_no_adjust,
  /// Grid::adjusted); a Run owns its own buffers (mcubes.cuh Run::Bufs).
  DevBuf<double> edges, lower, upper, contrib, scalars, point;
  DevBuf<unsigned long long> words, err_key;
  /// The grid the next K1 / point-kernel launch reads (device edges, lower
  /// bounds), bound by the caller right before it enqueues the launch.
  const double* grid_edges = nullptr;
  const double* grid_lower = nullptr;
  DevBuf<unsigned int> counter;  ///< finish-kernel last-block counter (self-resetting)
  DevBuf<unsigned int> peer_counter;  ///< K1 last-block counter of the peer-memory exchange (self-resetting)
  /// Peer-memory exchange of the launch being enqueued (npeers == 0: off);
  /// set by Run around its K1 / finish launches.
  PeerArgs peer{};
  DevBuf<double> table;  ///< parameters of a stateful integrand (owned copy)

  static constexpr std::size_t kPinnedBytes = 1 << 20;
  unsigned char* pinned() const { return pinned_; }
  /// Host writes into pinned() must not overtake asynchronous copies that
  /// still read it: writers call staging_wait() first and staging_recorded()
  /// after enqueuing their copies.
  void staging_wait() {
    if (staging_live_) MCB_CUDA(cudaEventSynchronize(staging_ev_));
    staging_live_ = false;
  }
  void staging_recorded() {
    if (!staging_ev_) MCB_CUDA(cudaEventCreateWithFlags(&staging_ev_, cudaEventDisableTiming));
    MCB_CUDA(cudaEventRecord(staging_ev_, stream_));
    staging_live_ = true;
  }

  /// Host-mapped per-iteration progress flags written by the finish kernel
  /// (0 = not run, 1 = continue, 2 = stop), for integrate()'s bounded lookahead.
  static constexpr std::uint32_t kMaxFlagIterations = 16384;
  int* host_flags() const { return flags_; }
  /// A Run's buffer set: a recycled one when available (stream-ordered after
  /// the work of the run that released it), else a new one.
  std::unique_ptr<RunBufs> acquire_run_bufs() {
    if (run_pool_.empty()) return std::make_unique<RunBufs>();
    std::unique_ptr<RunBufs> b = std::move(run_pool_.back());
    run_pool_.pop_back();
    if (b->pending) {  // the releasing run's kernels may still be in flight on another stream
      MCB_CUDA(cudaStreamWaitEvent(stream_, b->released, 0));
      b->pending = false;
    }
    return b;
  }
  /// Liveness token: a Run that outlives its context frees its buffers
  /// instead of returning them to the (destroyed) pool.
  std::weak_ptr<const int> alive() const { return alive_; }
  /// Return a Run's buffers after its last enqueued work (stream order).
  void release_run_bufs(std::unique_ptr<RunBufs> b) noexcept {
    if (!b) return;
    if (!b->released && cudaEventCreateWithFlags(&b->released, cudaEventDisableTiming) != cudaSuccess) return;
    if (cudaEventRecord(b->released, stream_) != cudaSuccess) return;  // dropped: freed instead of pooled
    b->pending = true;
    if (run_pool_.size() < kRunPool) run_pool_.push_back(std::move(b));
  }
  static constexpr std::size_t kRunPool = 8;

  /// The i-th event of a reusable pool (created on first use).
  cudaEvent_t event(std::size_t i) {
    while (events_.size() <= i) {
      cudaEvent_t e;
      MCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      events_.push_back(e);
    }
    return events_[i];
  }

 private:
  int device_ = 0;
  int sms_ = 0;
  int max_smem_ = 0;
  cudaStream_t own_stream_ = nullptr;
  cudaStream_t stream_ = nullptr;
  unsigned char* pinned_ = nullptr;
  cudaEvent_t staging_ev_ = nullptr;
  bool staging_live_ = false;
  int* flags_ = nullptr;
  std::vector<cudaEvent_t> events_;
  std::vector<std::unique_ptr<RunBufs>> run_pool_;
  std::shared_ptr<const int> alive_ = std::make_shared<const int>(1);
};

/// Geometry of one K1 launch (results do not depend on it).
struct Launch {
  int blocks = 0;
  std::size_t smem = 0;
  std::uint32_t pnb = 0;  ///< histogram cells per axis (n_bins, +1 padding cell on the Philox path)
  std::uint32_t passes = 1;  ///< bin passes (> 1 when the histograms exceed one CTA's shared memory)
  std::uint32_t copies = 1;  ///< grid-table copies in shared memory (stage_grid)
};

/// Cells per axis in K1's shared histogram for a stream kind.
constexpr std::uint32_t partial_bins(RngKind r, std::uint32_t nb) { return nb + (philox_stream(r) ? 1u : 0u); }

/// The work-index -> cube map of K1 (see vsample_kernel): whole rows along
/// axis 0 once there are enough of them.
inline bool row_mode(const Shape& sh) { return sh.dims >= 2 && sh.m / sh.g >= (std::uint64_t{1} << 20); }

/// Philox4x32-10 key schedule of the iteration key (uniform per launch).
inline void set_round_keys(SampleArgs& a, std::uint64_t key) {
  std::uint32_t k0 = static_cast<std::uint32_t>(key), k1 = static_cast<std::uint32_t>(key >> 32);
  for (int r = 0; r < 10; ++r) {
    a.round_keys[2 * r] = k0;
    a.round_keys[2 * r + 1] = k1;
    k0 += rng::kPhiloxW0;
    k1 += rng::kPhiloxW1;
  }
}

/// Constants of the Philox path: z = u32 * cs + digit * nbg, J = nb^D * prod(width).
inline void set_fast_constants(SampleArgs& a, const Shape& sh, int D) {
  a.nbg = static_cast<double>(sh.nb) / static_cast<double>(sh.g);
  a.cs = a.nbg * 0x1.0p-32;
  double pw = 1.0;
  for (int j = 0; j < D; ++j) pw *= static_cast<double>(sh.nb);
  a.nbpow = pw;
}

template <class F, int D, RngKind R, int NB = 0>
Launch launch_k1(Context& ctx, const F& f, const Shape& sh, std::uint32_t bin_axes,
                 std::uint64_t iter_root, std::uint64_t n0, std::uint64_t n1, const int* stop,
                 unsigned long long* err_key, unsigned long long* words) {
  auto kern = vsample_kernel<F, D, R, NB>;
  constexpr int kThreads = sample_threads(R, D);
  Launch L;
  L.pnb = partial_bins(R, sh.nb);
  // Bin passes: when bin_axes x (n_bins + 1) exact accumulators do not fit one
  // CTA's shared memory, the axes are split over passes that re-sample the
  // same keyed points (SampleArgs::bin_lo/bin_n); results are bitwise those of
  // one pass.
  const std::size_t budget = std::min<std::size_t>(kK1SmemBudget, static_cast<std::size_t>(ctx.max_smem()));
  const auto fits = [&](std::uint32_t na) { return sample_smem_bytes(D, L.pnb, na) <= budget; };
  std::uint32_t passes = 1, per_pass = bin_axes;
  if (!fits(bin_axes)) {
    std::uint32_t most = bin_axes;
    while (most > 1 && !fits(most)) --most;
    if (!fits(most))
      throw std::invalid_argument("B200 path: n_bins too large for one axis' shared-memory histogram (" +
                                  std::to_string(sample_smem_bytes(D, L.pnb, 1)) + " B > " +
                                  std::to_string(ctx.max_smem()) + " B)");
    passes = (bin_axes + most - 1) / most;
    per_pass = (bin_axes + passes - 1) / passes;  // balanced
    if constexpr (NB != 0)  // the compile-time-n_bins kernels run one pass (see vsample_kernel)
      return launch_k1<F, D, R, 0>(ctx, f, sh, bin_axes, iter_root, n0, n1, stop, err_key, words);
  }
  L.passes = passes;
  // grid-table copies: fixed per instantiation for the compile-time-n_bins
  // kernels (they fit by construction), else the most that fit this pass
  if constexpr (NB != 0) {
    L.copies = fixed_tab_copies(D, L.pnb);
    if (sample_smem_bytes(D, L.pnb, per_pass, L.copies) > budget)
      return launch_k1<F, D, R, 0>(ctx, f, sh, bin_axes, iter_root, n0, n1, stop, err_key, words);
  } else {
    L.copies = MCB_K1_TAB_COPIES_MAX;
    while (L.copies > 1 && sample_smem_bytes(D, L.pnb, per_pass, L.copies) > budget) L.copies >>= 1;
  }
  L.smem = sample_smem_bytes(D, L.pnb, per_pass, L.copies);
  // attribute + occupancy queries are cached per instantiation (host latency
  // matters for small-ncall iterations)
  thread_local std::size_t cached_smem = 0;
  thread_local int cached_occ = 0, cached_dev = -1;
  if (cached_smem != L.smem || cached_dev != ctx.device()) {
    MCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(L.smem)));
    MCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cached_occ, kern, kThreads, L.smem));
    cached_smem = L.smem;
    cached_dev = ctx.device();
  }
  const int occ = std::max(cached_occ, 1);
  const std::uint64_t work = n1 > n0 ? n1 - n0 : 0;
  // Blocks: every SM once the work fills a warp per SM.  Small problems
  // (fewer work items than one full block per SM, e.g. 10D at 1e6 calls:
  // 59,049 cubes of 16 samples) then spread over all SMs with fewer threads
  // each instead of filling a few SMs with full blocks.
  const std::uint64_t want = (work + 31) / 32;
  L.blocks = static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(want, std::uint64_t(ctx.sms()) * occ)));
  // Threads per block: the fewest (whole warps) that keep the per-thread cube
  // count of a full block.  Small problems then run every thread over the
  // same number of cubes instead of a last wave of partly idle warps (C1:
  // 2.45 cubes per thread at 1024 -> 3 each at 864 threads).  Row mode
  // (large problems) keeps full blocks.
  int threads = kThreads;
  if (!row_mode(sh) && work > 0 && !full_blocks_forced()) {
    const std::uint64_t full = static_cast<std::uint64_t>(L.blocks) * kThreads;
    const std::uint64_t per = (work + full - 1) / full;
    const std::uint64_t need = (work + static_cast<std::uint64_t>(L.blocks) * per - 1) /
                               (static_cast<std::uint64_t>(L.blocks) * per);
    threads = static_cast<int>(std::min<std::uint64_t>(kThreads, (need + 31) / 32 * 32));
  }
  const int walkers = threads;  // threads that walk cubes

  SampleArgs a{};
  if (!ctx.grid_edges || !ctx.grid_lower) throw std::invalid_argument("K1: no grid bound to the context");
  a.edges = ctx.grid_edges;
  a.lower = ctx.grid_lower;
  a.dims = sh.dims;
  a.nb = sh.nb;
  a.bin_axes = bin_axes;
  a.m = sh.m;
  a.p = sh.p;
  a.g = sh.g;
  a.nbd = static_cast<double>(sh.nb);
  a.gd = static_cast<double>(sh.g);
  a.rcp_g = sh.rcp_g;
  set_fast_constants(a, sh, D);
  a.scale = sh.scale;
  a.pp1 = sh.pp1;
  a.rcp_pp1 = sh.rcp_pp1;
  a.iter_root = iter_root;
  set_round_keys(a, iter_root);
  a.n0 = n0;
  a.n1 = n1;
  a.A = sh.A;
  const std::uint64_t T = static_cast<std::uint64_t>(L.blocks) * walkers;
  // Row mode when there are >= 2^20 rows (of g cubes along axis 0).  The
  // n -> cube map must depend on the problem only (m, g, d), never on the
  // slice [n0, n1) or the launch, so that slices sampled by different ranks
  // or calls partition the same cube set.
  const std::uint64_t nrows = D >= 2 ? sh.m / sh.g : 1;
  a.row_mode = row_mode(sh) ? 1u : 0u;
  a.R = nrows;
  if (a.row_mode) {
    unsigned __int128 Ap = 0, pw = 1;  // A' = 1 + g + ... + g^(D-2) mod R
    for (int j = 0; j + 1 < D; ++j) {
      Ap += pw;
      pw *= sh.g;
    }
    a.A = static_cast<std::uint64_t>(Ap % nrows);
    a.stepR = static_cast<std::uint64_t>((static_cast<unsigned __int128>(T % nrows) * a.A) % nrows);
    std::uint64_t st = a.stepR;
    a.step_digits[0] = 0;
    for (int j = 1; j < kMaxDims; ++j) {
      a.step_digits[j] = j < D ? st % sh.g : 0;
      if (j < D) st /= sh.g;
    }
  } else {
    a.stepT = static_cast<std::uint64_t>((static_cast<unsigned __int128>(T % sh.m) * sh.A) % sh.m);
    std::uint64_t st = a.stepT;
    for (int j = 0; j < kMaxDims; ++j) {
      a.step_digits[j] = j < static_cast<int>(sh.dims) ? st % sh.g : 0;
      if (j < static_cast<int>(sh.dims)) st /= sh.g;
    }
  }
  if (!words) throw std::invalid_argument("K1: the exchange buffer must be provided");
  a.words = words;
  a.nb_out = sh.nb;
  a.tab_copies = L.copies;
  a.err_key = err_key;
  a.stop = stop;
  a.peer = ctx.peer;
  // pairs of CTAs in a cluster split the flush (each adds both CTAs' words
  // for half of the accumulators, read over DSMEM): half the global
  // reductions per SM.  Two-CTA clusters keep all 148 SMs usable at one CTA
  // per SM (tools/microbench/clusters.cu).
  const unsigned cluster = (L.blocks % 2 == 0 && k1_cluster_enabled()) ? 2u : 1u;
  for (std::uint32_t q = 0; q < passes; ++q) {
    a.bin_lo = q * per_pass;
    a.bin_n = std::min(per_pass, bin_axes - a.bin_lo);
    a.scalars = q == 0 ? 1u : 0u;
    a.publish = q + 1 == passes ? 1u : 0u;
    const std::size_t smem = sample_smem_bytes(D, L.pnb, a.bin_n, L.copies);
    launch_pdl_cluster(kern, L.blocks, threads, smem, ctx.stream(), cluster, a, f);
    ++ctx.launches;
  }
  return L;
}

template <class F, int D, RngKind R>
void launch_point(Context& ctx, const F& f, const Shape& sh, std::uint64_t iter_root, std::uint64_t t,
                  std::uint64_t k, double* out_x, double* out_fx) {
  SampleArgs a{};
  if (!ctx.grid_edges || !ctx.grid_lower) throw std::invalid_argument("K1: no grid bound to the context");
  a.edges = ctx.grid_edges;
  a.lower = ctx.grid_lower;
  a.dims = sh.dims;
  a.nb = sh.nb;
  a.m = sh.m;
  a.p = sh.p;
  a.g = sh.g;
  a.nbd = static_cast<double>(sh.nb);
  a.gd = static_cast<double>(sh.g);
  a.rcp_g = sh.rcp_g;
  set_fast_constants(a, sh, D);
  a.iter_root = iter_root;
  set_round_keys(a, iter_root);
  const std::size_t smem = 2 * sizeof(double) * D * partial_bins(R, sh.nb);
  auto kern = sample_point_kernel<F, D, R>;
  MCB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<1, 128, smem, ctx.stream()>>>(a, f, t, k, out_x, out_fx);
  MCB_CUDA(cudaGetLastError());
  ++ctx.launches;
}

/// Compile-time dimension dispatch.  The set of instantiated dimensions can
/// be narrowed with MCB_DIMS_MAX to trade compile time for coverage.
#ifndef MCB_DIMS_MAX
#define MCB_DIMS_MAX 20
#endif

template <class F, RngKind R>
Launch dispatch_k1(Context& ctx, const F& f, const Shape& sh, std::uint32_t bin_axes, std::uint64_t iter_root,
                   std::uint64_t n0, std::uint64_t n1, const int* stop, unsigned long long* err_key,
                   unsigned long long* words) {
  switch (sh.dims) {
#define MCB_CASE(D) \
  case D:           \
    if constexpr (D <= MCB_DIMS_MAX) {                                                                                  \
      if (sh.nb == 50 && D <= 16) /* the compile-time n_bins fast path up to 16 axes */                              \
        return launch_k1<F, D, R, (D <= 16 ? 50 : 0)>(ctx, f, sh, bin_axes, iter_root, n0, n1, stop, err_key, words); \
      return launch_k1<F, D, R, 0>(ctx, f, sh, bin_axes, iter_root, n0, n1, stop, err_key, words);                  \
    }                                                                                                                   \
    break;
    MCB_CASE(1) MCB_CASE(2) MCB_CASE(3) MCB_CASE(4) MCB_CASE(5) MCB_CASE(6) MCB_CASE(7) MCB_CASE(8)
    MCB_CASE(9) MCB_CASE(10) MCB_CASE(11) MCB_CASE(12) MCB_CASE(13) MCB_CASE(14) MCB_CASE(15) MCB_CASE(16) \
    MCB_CASE(17) MCB_CASE(18) MCB_CASE(19) MCB_CASE(20)
#undef MCB_CASE
    default:
      break;
  }
  throw std::invalid_argument("B200 path: no kernel compiled for dims=" + std::to_string(sh.dims));
}

template <class F, RngKind R>
void dispatch_point(Context& ctx, const F& f, const Shape& sh, std::uint64_t iter_root, std::uint64_t t,
                    std::uint64_t k, double* out_x, double* out_fx) {
  switch (sh.dims) {
#define MCB_CASE(D) \
  case D:           \
    if constexpr (D <= MCB_DIMS_MAX) { launch_point<F, D, R>(ctx, f, sh, iter_root, t, k, out_x, out_fx); return; } \
    break;
    MCB_CASE(1) MCB_CASE(2) MCB_CASE(3) MCB_CASE(4) MCB_CASE(5) MCB_CASE(6) MCB_CASE(7) MCB_CASE(8)
    MCB_CASE(9) MCB_CASE(10) MCB_CASE(11) MCB_CASE(12) MCB_CASE(13) MCB_CASE(14) MCB_CASE(15) MCB_CASE(16) \
    MCB_CASE(17) MCB_CASE(18) MCB_CASE(19) MCB_CASE(20)
#undef MCB_CASE
    default:
      break;
  }
  throw std::invalid_argument("B200 path: no kernel compiled for dims=" + std::to_string(sh.dims));
}

/// Warps of a finish/adjust block that adapt axes (one axis each); their
/// scratch bounds the block's shared memory.
inline int adjust_warps(std::uint32_t dims, std::uint32_t nb, int max_smem) {
  int w = std::max(1, std::min<int>(static_cast<int>(dims), kFinishThreads / 32));
  const std::size_t fixed = 2 * sizeof(double) * static_cast<std::size_t>(dims) * nb;  // contributions + edges
  while (w > 1 && fixed + sizeof(double) * static_cast<std::size_t>(w) * kAdjustScratch * nb >
                      static_cast<std::size_t>(max_smem))
    --w;
  if (fixed + sizeof(double) * static_cast<std::size_t>(w) * kAdjustScratch * nb > static_cast<std::size_t>(max_smem))
    throw std::invalid_argument("B200 path: n_bins too large for the on-device grid adaptation");
  return w;
}

/// K3b + K4 fused: exchange words -> estimate, variance, contributions; with
/// an epilogue, also grid adaptation + weighted estimate + convergence.
inline void launch_finish(Context& ctx, const Shape& sh, std::uint32_t bin_axes, unsigned long long* words,
                          double* est, double* var, double* contrib, const int* stop, const EpilogueArgs* epi,
                          bool zero_words = false, unsigned long long* counts = nullptr, bool prerounded = false) {
  RoundArgs r{};
  r.words = words;
  r.dims = sh.dims;
  r.nb = sh.nb;
  r.bin_axes = bin_axes;
  r.md2 = static_cast<double>(sh.m) * static_cast<double>(sh.m);
  r.est = est;
  r.var = var;
  r.contrib = contrib;
  r.counts = counts;
  r.stop = stop;
  r.zero_words = zero_words ? 1 : 0;
  r.prerounded = prerounded ? 1 : 0;
  if (epi && ctx.peer.npeers) {
    r.wait_flags = ctx.peer.my_flags;
    r.nwait = ctx.peer.npeers;
    r.wait_value = ctx.peer.flag;
  }
  EpilogueArgs e{};
  std::size_t smem = 0;
  if (epi) {
    e = *epi;
    e.adj_warps = adjust_warps(sh.dims, sh.nb, ctx.max_smem());
    const std::size_t staged = 2 * static_cast<std::size_t>(sh.dims) * sh.nb;  // contributions + edges
    const std::size_t par = sizeof(double) * (staged + adjust_par_scratch(sh.dims, sh.nb));
    e.adj_par = (!e.adj.symmetric && par <= static_cast<std::size_t>(ctx.max_smem()) && adjust_par_enabled()) ? 1 : 0;
    smem = e.adj_par ? par
                     : sizeof(double) * (staged + static_cast<std::size_t>(e.adj_warps) * kAdjustScratch * sh.nb);
  }
  // the raised limit is a per-device function attribute: cache it per device
  thread_local std::map<int, std::size_t> attr_smem;
  if (smem > 48 * 1024 && smem > attr_smem[ctx.device()]) {
    MCB_CUDA(cudaFuncSetAttribute(finish_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr_smem[ctx.device()] = smem;
  }
  unsigned int* counter = ctx.counter.get();
  if (!counter) {
    counter = ctx.counter.ensure(1);
    MCB_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned int), ctx.stream()));
  }
  const int values = static_cast<int>(sh.dims * sh.nb + 2);  // one warp per output value
  const int warps_per_block = kFinishThreads / 32;
  const int blocks = prerounded ? 1 : (values + warps_per_block - 1) / warps_per_block;  // prerounded: epilogue only
  launch_pdl(finish_kernel<0>, blocks, kFinishThreads, smem, ctx.stream(), r, e, epi ? 1 : 0, counter);
  ++ctx.launches;
}

/// Standalone Grid::adjusted on device (edges in ctx.edges, contributions in
/// ctx.contrib).
inline void launch_adjust(Context& ctx, AdjustArgs a) {
  const int w = adjust_warps(a.dims, a.nb, ctx.max_smem());
  const std::size_t smem = sizeof(double) * static_cast<std::size_t>(w) * kAdjustScratch * a.nb;
  if (smem > 48 * 1024)
    MCB_CUDA(cudaFuncSetAttribute(adjust_grid_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  adjust_grid_kernel<0><<<1, 32 * w, smem, ctx.stream()>>>(a);
  MCB_CUDA(cudaGetLastError());
  ++ctx.launches;
}

}  // namespace mcubes::gpu
