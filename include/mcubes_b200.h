/* SPDX-License-Identifier: Apache-2.0
 *
 * mcubes_b200 C ABI -- the FFI boundary of the B200 m-Cubes path
 * (libmcubes_b200.so, built from paper_2202_01753_b200/csrc/).
 *
 * The reference is a header-only C++20 template library with no C ABI
 * (SURVEY.md section 8b); each entry point below is the C-callable form of the
 * reference function it replaces, cited as path:line under
 * /root/reference/proj/include/mcubes/.  C++ users can instead include
 * <mcubes_b200/mcubes.cuh>, the source-compatible template API, and pass their
 * own device functors.  Python binds this header via ctypes
 * (paper_2202_01753_b200/_lib.py); see INTEGRATION.md.
 *
 * Conventions: plain pointers + sizes, caller-owned HOST buffers (never
 * retained), row-major dims x n_bins matrices (grid.hpp:303,
 * accumulators.hpp:26-27).  Every call returns an int status:
 *   MCB_OK, MCB_EINVAL (std::invalid_argument), MCB_ENONFINITE
 *   (NonFiniteSample; query mcb_last_nonfinite), MCB_ECUDA, MCB_EINTERNAL.
 * A context must be used from one host thread at a time; separate contexts
 * may run concurrently.
 */
#ifndef MCUBES_B200_H
#define MCUBES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCB_ABI_VERSION 2
#define MCB_XWORDS 67 /* u64 words per exact accumulator in the exchange buffer */
#define MCB_XHEADER 3 /* u64 count words ahead of the accumulators: overflowed addends, finite
                         samples (device-counted; the write count), non-finite samples */

enum mcb_status {
  MCB_OK = 0,
  MCB_EINVAL = -1,
  MCB_ENONFINITE = -2,
  MCB_ECUDA = -3,
  MCB_EINTERNAL = -9
};

/* Built-in integrands (the reference's suite, integrands.hpp:107-215, plus
 * the stateful table integrand of BASELINE config 4 and the small functors
 * the reference's unit tests use). */
enum mcb_integrand_id {
  MCB_F1 = 1, /* oscillatory        cos(sum (i+1) x_i)                 */
  MCB_F2 = 2, /* product peak       prod 1/(1/2500 + (x_i-1/2)^2)      */
  MCB_F3 = 3, /* corner peak        (1 + sum (i+1) x_i)^(-d-1)         */
  MCB_F4 = 4, /* Gaussian           exp(-625 sum (x_i-1/2)^2)          */
  MCB_F5 = 5, /* C0                 exp(-10 sum |x_i-1/2|)             */
  MCB_F6 = 6, /* discontinuous      exp(sum (i+5) x_i) below cutoffs   */
  MCB_FA = 7, /* sin(sum x) on (0,10)^6                                */
  MCB_FB = 8, /* normalized 9D Gaussian on (-1,1)^9                    */
  MCB_TABLE = 9, /* prod_j lerp(T_j, (x_j-lo_j)*inv_h_j); params =
                    [n, lo[d], inv_h[d], T_0[n] .. T_{d-1}[n]]          */
  MCB_T_X0 = 32,         /* x[0]                                          */
  MCB_T_CONST = 33,      /* params[0]                                     */
  MCB_T_X0SQ_HALF = 34,  /* x[0]*x[0] + 0.5                               */
  MCB_T_INF_X0POS = 35,  /* x[0] > 0 ? inf : 1                            */
  MCB_T_INF = 36,        /* inf                                           */
  MCB_T_ZERO = 37,       /* 0                                             */
  MCB_T_INF_NEAR_ORIGIN = 38 /* inf if every x_j < params[0], else 1 (multi-rank failure tests) */
};

enum mcb_bin_update { MCB_BIN_ALL_AXES = 0, MCB_BIN_AXIS0_ONLY = 1, /* sampler.hpp:51-54 */
                      MCB_BIN_NONE = 2 /* frozen iteration (mcb_v_sample_philox only) */ };
enum mcb_variant { MCB_VARIANT_MCUBES = 0, MCB_VARIANT_MCUBES1D = 1 }; /* driver.hpp:23 */
/* Sample stream and bin precision: COMPAT = the reference's keyed SplitMix
 * stream and arithmetic order with exact bins (bitwise the reference);
 * PHILOX = the north-star Philox4x32-10 stream, bins summed from (f J)^2
 * rounded to 24 significant bits; PHILOX_EXACT = the Philox stream with exact
 * bins (the reference's ExactBins precision). */
enum mcb_rng { MCB_RNG_COMPAT = 0, MCB_RNG_PHILOX = 1, MCB_RNG_PHILOX_EXACT = 2 };

typedef struct mcb_ctx mcb_ctx;
typedef struct mcb_run mcb_run;

typedef struct {
  int32_t id;             /* mcb_integrand_id */
  uint32_t n_params;
  const double* params;   /* host; copied to the device by the call */
} mcb_integrand;

/* RunConfig (driver.hpp:37-71) + B200 fields. */
typedef struct {
  uint32_t dims;
  uint32_t n_bins;        /* reference default 50 */
  uint64_t maxcalls;
  uint32_t itmax;         /* 15 */
  uint32_t ita;           /* 10 */
  double tau_rel;         /* 1e-3 */
  double alpha;           /* 1.5 */
  double chi2_dof_max;    /* 1.5 */
  uint64_t seed;
  int32_t variant;        /* mcb_variant */
  uint32_t workers;       /* accepted, ignored (results are worker-invariant) */
  const double* lower;    /* dims */
  const double* upper;    /* dims */
  int32_t rng;            /* mcb_rng */
  int32_t reserved;
} mcb_config;

/* IntegrationResult (driver.hpp:181-191). */
typedef struct {
  double estimate, sigma, chi2_dof;
  uint32_t iterations_used;
  int32_t converged;
  uint64_t total_samples, bin_writes;
  uint64_t g, m, p, s; /* SetupParams (driver.hpp:74-79) */
} mcb_result;

/* IterationResult (driver.hpp:126-130). */
typedef struct {
  double estimate, variance;
  uint32_t index;
  uint32_t pad;
} mcb_iteration;

/* IterationView (driver.hpp:196-203); grid_edges is dims*n_bins, valid only
 * during the callback. */
typedef struct {
  uint32_t iteration;
  int32_t adjusting;
  mcb_iteration result;
  double running_estimate, running_sigma, running_chi2_dof;
  const double* grid_edges;
  uint64_t bin_writes;
} mcb_iteration_view;
typedef void (*mcb_observer)(const mcb_iteration_view* view, void* user);

/* ---- context ---- */
int mcb_ctx_create(int device, mcb_ctx** out);
int mcb_ctx_destroy(mcb_ctx* ctx);
/* Run on a caller-owned cudaStream_t (NULL = the context's own stream). */
int mcb_ctx_set_stream(mcb_ctx* ctx, void* cuda_stream);
int mcb_ctx_synchronize(mcb_ctx* ctx);
/* Kernels launched through this context so far. */
uint64_t mcb_ctx_launches(const mcb_ctx* ctx);
const char* mcb_last_error(const mcb_ctx* ctx);
/* Point (dims doubles) and f(x) of the last MCB_ENONFINITE (sampler.hpp:35-36). */
int mcb_last_nonfinite(const mcb_ctx* ctx, double* x, uint32_t cap, double* fx);
int mcb_abi_version(void);

/* ---- one iteration: v_sample (sampler.hpp:312-333) ----
 * edges: dims*n_bins right edges (NULL = uniform grid on [lower, upper]).
 * contrib: dims*n_bins out (rows >= bin_axes are zero); writes = m*p*bin_axes. */
int mcb_v_sample(mcb_ctx* ctx, const mcb_integrand* f, uint32_t dims, uint32_t n_bins,
                 const double* lower, const double* upper, const double* edges, uint64_t m,
                 uint64_t s, uint64_t p, uint64_t seed, uint64_t iteration, int32_t bin_update,
                 double* estimate, double* variance, double* contrib, uint64_t* writes);

/* ---- frozen iteration: v_sample_no_adjust (sampler.hpp:339-349) ---- */
int mcb_v_sample_no_adjust(mcb_ctx* ctx, const mcb_integrand* f, uint32_t dims, uint32_t n_bins,
                           const double* lower, const double* upper, const double* edges,
                           uint64_t m, uint64_t s, uint64_t p, uint64_t seed, uint64_t iteration,
                           double* estimate, double* variance);

/* ---- Philox-path variant of v_sample (north-star RNG + FMA-contracted
 * transform; not bitwise comparable with the reference, statistically
 * equivalent).  bin_update = MCB_BIN_NONE runs the frozen iteration
 * (v_sample_no_adjust) and leaves contrib / writes untouched. ---- */
int mcb_v_sample_philox(mcb_ctx* ctx, const mcb_integrand* f, uint32_t dims, uint32_t n_bins,
                        const double* lower, const double* upper, const double* edges, uint64_t m,
                        uint64_t s, uint64_t p, uint64_t seed, uint64_t iteration,
                        int32_t bin_update, double* estimate, double* variance, double* contrib,
                        uint64_t* writes);

/* ---- v_sample on any stream (mcb_rng: COMPAT, PHILOX, PHILOX_EXACT);
 * bin_update as mcb_v_sample_philox.  *writes is the device-counted number of
 * contribution deposits (sampler.hpp:116-119). ---- */
int mcb_v_sample_rng(mcb_ctx* ctx, const mcb_integrand* f, int32_t rng, uint32_t dims, uint32_t n_bins,
                     const double* lower, const double* upper, const double* edges, uint64_t m, uint64_t s,
                     uint64_t p, uint64_t seed, uint64_t iteration, int32_t bin_update, double* estimate,
                     double* variance, double* contrib, uint64_t* writes);

/* ---- grid adaptation on the device: Grid::adjusted / adjusted_symmetric
 * (grid.hpp:104-146, 232-297).  symmetric != 0 reads contrib row 0 only. ---- */
int mcb_grid_adjust(mcb_ctx* ctx, uint32_t dims, uint32_t n_bins, const double* lower,
                    const double* upper, const double* edges, const double* contrib, double alpha,
                    int32_t symmetric, double* out_edges);

/* ---- host utilities (driver.hpp:82-178) ---- */
int mcb_setup(const mcb_config* cfg, uint64_t* g, uint64_t* m, uint64_t* p, uint64_t* s);
int mcb_set_batch_size(uint64_t m, uint32_t workers, uint64_t* s);
int mcb_weighted_estimate(uint32_t n, const double* estimates, const double* variances,
                          double* estimate, double* sigma, double* chi2_dof);
int mcb_check_convergence(double estimate, double sigma, double chi2_dof, double tau_rel,
                          double chi2_dof_max);
int mcb_grid_uniform(uint32_t dims, uint32_t n_bins, const double* lower, const double* upper,
                     double* edges);

/* ---- the full loop: integrate (driver.hpp:215-258) ----
 * history: caller array of history_cap entries (may be NULL).  observer may be
 * NULL (then the run is enqueued with a single synchronisation at the end). */
int mcb_integrate(mcb_ctx* ctx, const mcb_integrand* f, const mcb_config* cfg, mcb_result* result,
                  mcb_iteration* history, uint32_t history_cap, mcb_observer observer, void* user);

/* ---- integrate() resumed from a checkpoint: `edges` (dims x n_bins) is the
 * grid after the n_done completed iterations `done` (indices 1..n_done), e.g.
 * read back with the grid.hpp:148-174 text format.  The stream is keyed by
 * (seed, iteration), so the result is bitwise equal to the uninterrupted run.
 * (The reference has the grid I/O but no resume entry point.) ---- */
int mcb_integrate_resume(mcb_ctx* ctx, const mcb_integrand* f, const mcb_config* cfg, const double* edges,
                         const mcb_iteration* done, uint32_t n_done, mcb_result* result, mcb_iteration* history,
                         uint32_t history_cap, mcb_observer observer, void* user);

/* ---- stepped run: the multi-GPU hook.  Each rank samples its slice of the
 * linear work index, the caller all-reduces (sum, uint64) the exchange buffer
 * across ranks, then every rank finishes the iteration identically. ---- */
int mcb_run_create(mcb_ctx* ctx, const mcb_integrand* f, const mcb_config* cfg, mcb_run** out);
int mcb_run_destroy(mcb_run* run);
/* Exchange buffer length (u64 words) for iteration it (1-based; 0 = the
 * largest).  MCB_XHEADER count words (overflowed exact addends, finite
 * samples, non-finite samples), then MCB_XWORDS words per accumulator (est+,
 * est-, var, bins); all-reducing the first mcb_run_exchange_words(run, it)
 * words covers iteration it. */
uint64_t mcb_run_exchange_words(const mcb_run* run, uint32_t it);
/* Use a caller-owned DEVICE buffer (>= max exchange words) for the exchange. */
int mcb_run_set_exchange(mcb_run* run, void* device_ptr);
/* Progress reporting for early exit without a synchronising read: after
 * iteration it has finished on the device, host_flags[it-1] = 1 (continue) or
 * 2 (the run stopped: converged, failed or done).  host_flags must be pinned,
 * device-accessible host memory of itmax ints, zeroed by the caller; NULL
 * turns reporting off.  (No reference counterpart: the reference's integrate
 * loop is synchronous, driver.hpp:227-256.) */
int mcb_run_set_progress(mcb_run* run, int* host_flags);
/* Multi-rank failure reporting: *failed = 1 if the run stopped on a
 * non-finite sample (in any rank's slice: the count is exchanged with the
 * words), *key = this rank's first failing sample t*p+k (all ones if none was
 * in its slice).  Drivers all-reduce the key with MIN and hand it back with
 * mcb_run_set_failure_key before mcb_run_result, so every rank returns the
 * same MCB_ENONFINITE point. */
int mcb_run_failure_key(mcb_run* run, int* failed, uint64_t* key);

/* ---- multi-GPU exchange over peer memory (NVLink / NVSwitch) instead of a
 * collective.  Every rank allocates two exchange buffers (odd and even
 * iterations, mcb_run_exchange_words(run, 0) u64 each), a flag array
 * (npeers u64) and a block counter (u32) with mcb_dev_alloc (zeroed), shares
 * their CUDA IPC handles (mcb_ipc_handle / mcb_ipc_open) and hands every
 * rank's pointers to mcb_run_set_peers.  Each iteration is then
 * mcb_run_sample + mcb_run_finish with no collective: K1's blocks add their
 * exact words into every rank's buffer with system-scope reductions and
 * release a per-iteration flag; the finish kernel acquires all ranks' flags.
 * Arrays are indexed by rank; npeers <= 8; 0 turns it off. ---- */
#define MCB_IPC_HANDLE_BYTES 64
int mcb_run_set_peers(mcb_run* run, int rank, int npeers, void* const* bufs_odd, void* const* bufs_even,
                      void* const* flags, void* counter);
int mcb_dev_alloc(mcb_ctx* ctx, uint64_t bytes, void** ptr);
int mcb_dev_free(mcb_ctx* ctx, void* ptr);
int mcb_ipc_handle(mcb_ctx* ctx, void* ptr, unsigned char* handle);
int mcb_ipc_open(mcb_ctx* ctx, const unsigned char* handle, void** ptr);
int mcb_ipc_close(mcb_ctx* ctx, void* ptr);
int mcb_run_set_failure_key(mcb_run* run, uint64_t key);
/* Resume a stepped run from a checkpoint (see mcb_integrate_resume); on
 * success *next_iteration is the first iteration to sample. */
int mcb_run_resume(mcb_run* run, const double* edges, const mcb_iteration* done, uint32_t n_done,
                   uint32_t* next_iteration);
void* mcb_run_exchange_ptr(const mcb_run* run);
/* Total linear work items (= m cubes). */
uint64_t mcb_run_work_items(const mcb_run* run);
/* K1: sample work items [n0, n1) of iteration it; its blocks add their exact
 * sums into the exchange buffer (which then holds exactly this slice's sums). */
int mcb_run_sample(mcb_run* run, uint32_t it, uint64_t n0, uint64_t n1);
/* The cross-block reduction step of the reference's merge (sampler.hpp:272-276):
 * already done by K1's flush; kept so stepped callers read sample -> reduce ->
 * all-reduce -> finish.  Checks that `it` was sampled. */
int mcb_run_reduce(mcb_run* run, uint32_t it);
/* K3b + K4: round, adapt the grid, combine, convergence gate. */
int mcb_run_finish(mcb_run* run, uint32_t it);

/* ---- compact exchange: SURVEY.md section 8(e)'s all-gather of each rank's
 * rounded (d*n_bins + 2) doubles, combined in a fixed rank order (replaces
 * the reference's in-process merge of worker partials, sampler.hpp:272-276,
 * across GPUs).  Per iteration: mcb_run_sample on the rank's slice;
 * mcb_run_round_local into a device buffer of mcb_run_compact_len(run)
 * doubles (estimate, variance, 4 u64 counts bit-cast to doubles --
 * samples, writes, overflowed addends, non-finite samples -- then the
 * contributions); all-gather those buffers rank-major; mcb_run_combine sums
 * them in rank order on the device; mcb_run_finish_rounded adapts the grid
 * and updates the weighted estimate (driver.hpp:231-252).  Every rank holds
 * identical state; the last bits depend on the rank count (each rank rounds
 * its partial sums), one rank is bitwise the exact path. */
uint64_t mcb_run_compact_len(const mcb_run* run);
int mcb_run_round_local(mcb_run* run, uint32_t it, double* out);
int mcb_run_combine(mcb_run* run, uint32_t it, const double* gathered, int nranks);
int mcb_run_finish_rounded(mcb_run* run, uint32_t it);
int mcb_run_result(mcb_run* run, mcb_result* result, mcb_iteration* history, uint32_t history_cap);
/* Replace the device grid with host edges (dims*n_bins); stream-ordered. */
int mcb_run_set_grid(mcb_run* run, const double* edges);
/* Current grid edges (dims*n_bins) -- synchronises. */
int mcb_run_grid(mcb_run* run, double* edges);

#ifdef __cplusplus
}
#endif

#endif /* MCUBES_B200_H */
