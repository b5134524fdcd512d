// Microbenchmarks that decide the sampling-kernel design on sm_100a:
// FP64 issue rate, SplitMix64 cost, conversions, division, shared-memory
// 64-bit integer atomics (the exact-histogram primitive), FP64 smem atomics,
// MATCH.ANY.  Each kernel reports (per SM) thread-ops per SM clock measured
// with clock64() inside the kernel.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ unsigned long long g_cycles[4096];
__device__ double g_sink_d[1 << 20];
__device__ unsigned long long g_sink_u[1 << 20];

constexpr int ITERS = 4096;

__global__ void k_dadd(int flag) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double c = 1e-9 * (flag + 1);
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    a0 = __dadd_rn(a0, c); a1 = __dadd_rn(a1, c); a2 = __dadd_rn(a2, c); a3 = __dadd_rn(a3, c);
    a4 = __dadd_rn(a4, c); a5 = __dadd_rn(a5, c); a6 = __dadd_rn(a6, c); a7 = __dadd_rn(a7, c);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_d[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_dfma(int flag) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double c = 1.0 + 1e-9 * (flag + 1);
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    a0 = __fma_rn(a0, c, c); a1 = __fma_rn(a1, c, c); a2 = __fma_rn(a2, c, c); a3 = __fma_rn(a3, c, c);
    a4 = __fma_rn(a4, c, c); a5 = __fma_rn(a5, c, c); a6 = __fma_rn(a6, c, c); a7 = __fma_rn(a7, c, c);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_d[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ uint64_t avalanche(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__global__ void k_splitmix(int flag) {
  uint64_t h0 = threadIdx.x + flag, h1 = h0 * 3, h2 = h0 * 5, h3 = h0 * 7;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < ITERS / 4; ++i) {
    h0 = avalanche(h0 + 0x9e3779b97f4a7c15ull); h1 = avalanche(h1 + 0x9e3779b97f4a7c15ull);
    h2 = avalanche(h2 + 0x9e3779b97f4a7c15ull); h3 = avalanche(h3 + 0x9e3779b97f4a7c15ull);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_u[threadIdx.x] = h0 ^ h1 ^ h2 ^ h3;
}

// u64 -> f64 conversion of a 53-bit integer (to_unit), 4 independent chains
__global__ void k_i2f(int flag) {
  uint64_t h0 = threadIdx.x + flag, h1 = h0 * 3, h2 = h0 * 5, h3 = h0 * 7;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    s0 += (double)(h0 >> 11); s1 += (double)(h1 >> 11); s2 += (double)(h2 >> 11); s3 += (double)(h3 >> 11);
    h0 += 977; h1 += 977; h2 += 977; h3 += 977;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_d[threadIdx.x] = s0 + s1 + s2 + s3;
}

// f64 -> u32 (bin index) conversion
__global__ void k_f2i(int flag) {
  double z0 = threadIdx.x * 0.37 + flag, z1 = z0 + 0.5, z2 = z0 + 0.25, z3 = z0 + 0.125;
  unsigned s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    s0 += (unsigned)z0; s1 += (unsigned)z1; s2 += (unsigned)z2; s3 += (unsigned)z3;
    z0 += 1.0; z1 += 1.0; z2 += 1.0; z3 += 1.0;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_u[threadIdx.x] = s0 + s1 + s2 + s3;
}

__global__ void k_ddiv(int flag) {
  double a0 = threadIdx.x + 0.3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  const double g = 9.0 + flag;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
    s0 += a0 / g; s1 += a1 / g; s2 += a2 / g; s3 += a3 / g;
    a0 += 0.1; a1 += 0.1; a2 += 0.1; a3 += 0.1;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_d[threadIdx.x] = s0 + s1 + s2 + s3;
}

__global__ void k_exp(int flag) {
  double a0 = -(threadIdx.x * 0.01) - flag, a1 = a0 - 0.5, a2 = a0 - 0.25, a3 = a0 - 0.75;
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < ITERS / 16; ++i) {
    s0 += exp(a0); s1 += exp(a1); s2 += exp(a2); s3 += exp(a3);
    a0 -= 0.001; a1 -= 0.001; a2 -= 0.001; a3 -= 0.001;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_d[threadIdx.x] = s0 + s1 + s2 + s3;
}

// shared-memory 64-bit integer atomics: mode 0 = distinct addresses per lane
// (no return), 1 = distinct with return used, 2 = 4 lanes per address,
// 3 = all 32 lanes one address, 4 = random bins over 400 (like histogram)
template <int MODE>
__global__ void k_atoms_u64(int flag) {
  extern __shared__ unsigned long long sm[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long acc = 0;
  uint64_t h = threadIdx.x * 0x9e3779b97f4a7c15ull + flag;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
    int addr;
    if (MODE == 0 || MODE == 1) addr = (warp * 32 + lane) * 2 + (i & 1) * 1024;
    else if (MODE == 2) addr = (warp * 8 + (lane >> 2)) * 4 + (i & 1) * 1024;
    else if (MODE == 3) addr = warp * 64 + (i & 1);
    else { h = h * 6364136223846793005ull + 1442695040888963407ull; addr = (int)((h >> 40) % 400u) * 17; }
    if (MODE == 1) acc += atomicAdd(&sm[addr], (unsigned long long)(i + 1));
    else atomicAdd(&sm[addr], (unsigned long long)(i + 1));
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_u[threadIdx.x] = acc + sm[threadIdx.x];
}

template <int MODE>
__global__ void k_atoms_f64(int flag) {
  extern __shared__ double smd[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) smd[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t h = threadIdx.x * 0x9e3779b97f4a7c15ull + flag;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
    int addr;
    if (MODE == 0) addr = (warp * 32 + lane) * 2 + (i & 1) * 1024;
    else { h = h * 6364136223846793005ull + 1442695040888963407ull; addr = (int)((h >> 40) % 400u); }
    atomicAdd(&smd[addr], 1.0 + i);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_d[threadIdx.x] = smd[threadIdx.x];
}

// plain LDS+DADD+STS to a thread-private slot (private histogram cost)
__global__ void k_lds_private(int flag) {
  extern __shared__ double smd[];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) smd[i] = 0;
  __syncthreads();
  uint64_t h = threadIdx.x * 0x9e3779b97f4a7c15ull + flag;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    int slot = (int)((h >> 40) & 7);
    double* p = &smd[slot * blockDim.x + threadIdx.x];
    *p = *p + 1.0;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_d[threadIdx.x] = smd[threadIdx.x];
}

__global__ void k_match(int flag) {
  uint64_t h = threadIdx.x * 0x9e3779b97f4a7c15ull + flag;
  unsigned acc = 0;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    unsigned b = (unsigned)(h >> 40) % 50u;
    acc += __match_any_sync(0xffffffffu, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_u[threadIdx.x] = acc;
}

// baseline for the LCG overhead used by the random-address tests
__global__ void k_lcg(int flag) {
  uint64_t h = threadIdx.x * 0x9e3779b97f4a7c15ull + flag;
  unsigned acc = 0;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS / 4; ++i) {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    acc += (unsigned)(h >> 40) % 400u;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_u[threadIdx.x] = acc;
}


// exact deposit: u32 words, radix 2^32 digits, carry via returned old value.
__device__ __forceinline__ void exact_add_u32(unsigned* acc, double v) {
  const unsigned long long bits = __double_as_longlong(v);
  if (bits == 0) return;
  const unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
  const unsigned be = hi >> 20;
  const unsigned m1 = (hi & 0xFFFFFu) | (be ? 0x100000u : 0u);
  const unsigned pos = be ? be - 1 : 0;
  const unsigned w = pos >> 5, off = pos & 31;
  const unsigned d0 = lo << off;
  const unsigned d1 = __funnelshift_l(lo, m1, off);
  const unsigned d2 = __funnelshift_l(m1, 0u, off);
  unsigned* p = acc + w;
  unsigned o0 = atomicAdd(p, d0);
  unsigned c = (o0 + d0) < o0;
  unsigned t1 = d1 + c;
  c = (t1 < c);
  unsigned o1 = atomicAdd(p + 1, t1);
  c += (o1 + t1) < o1;
  unsigned t2 = d2 + c;
  unsigned o2 = atomicAdd(p + 2, t2);
  if ((o2 + t2) < o2) {
    unsigned k = 3;
    while (atomicAdd(p + k, 1u) == 0xFFFFFFFFu) ++k;
  }
}

__global__ void k_exact(int flag) {
  extern __shared__ unsigned smu[];
  for (int i = threadIdx.x; i < 400 * 66; i += blockDim.x) smu[i] = 0;
  __syncthreads();
  uint64_t h = threadIdx.x * 0x9e3779b97f4a7c15ull + flag + blockIdx.x;
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < ITERS / 4; ++i) {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    int bin = (int)((h >> 40) % 400u);
    double v = __longlong_as_double((long long)((h >> 12) | 0x3800000000000000ull));
    exact_add_u32(smu + bin * 66, v);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_u[threadIdx.x] = smu[threadIdx.x];
}

__global__ void k_f64cas(int flag) {
  extern __shared__ double smd[];
  for (int i = threadIdx.x; i < 400; i += blockDim.x) smd[i] = 0;
  __syncthreads();
  uint64_t h = threadIdx.x * 0x9e3779b97f4a7c15ull + flag + blockIdx.x;
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < ITERS / 4; ++i) {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    int bin = (int)((h >> 40) % 400u);
    double v = __longlong_as_double((long long)((h >> 12) | 0x3800000000000000ull));
    atomicAdd(smd + bin, v);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (flag == 12345) g_sink_d[threadIdx.x] = smd[threadIdx.x];
}

typedef void (*kfn)(int);

static double run(const char* name, kfn k, int blocks, int threads, size_t smem, double ops_per_thread) {
  if (smem) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<blocks, threads, smem>>>(0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads, smem>>>(0);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc[4096];
  CK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * blocks));
  double mean = 0; for (int i = 0; i < blocks; ++i) mean += cyc[i]; mean /= blocks;
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int per_sm = blocks / nsm;
  // thread-ops per SM-cycle: per_sm blocks resident concurrently
  double ops_per_cyc = per_sm * threads * ops_per_thread / mean;
  double total = (double)blocks * threads * ops_per_thread;
  printf("%-28s blocks=%d thr=%d : %8.2f thread-ops/clk/SM  (%.2f warp-ops/clk/SM)  %.3f ms  %.3e ops/s\n",
         name, blocks, threads, ops_per_cyc, ops_per_cyc / 32, ms, total / (ms * 1e-3));
  return ops_per_cyc;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock=%d kHz\n", nsm, clk);
  for (int occ : {1, 2}) {
    int B = nsm * occ, T = 256;
    printf("--- %d blocks/SM x %d threads\n", occ, T);
    run("dadd (8 chains)", k_dadd, B, T, 0, 8.0 * ITERS);
    run("dfma (8 chains)", k_dfma, B, T, 0, 8.0 * ITERS);
    run("splitmix feed (4 chains)", k_splitmix, B, T, 0, 4.0 * (ITERS / 4));
    run("i2f.f64.u64 + dadd", k_i2f, B, T, 0, 4.0 * ITERS);
    run("f2i.u32.f64 + dadd", k_f2i, B, T, 0, 4.0 * ITERS);
    run("ddiv IEEE (+dadd)", k_ddiv, B, T, 0, 4.0 * (ITERS / 4));
    run("exp f64", k_exp, B, T, 0, 4.0 * (ITERS / 16));
    run("lcg+mod baseline", k_lcg, B, T, 0, 1.0 * (ITERS / 4));
    run("match.any (+lcg)", k_match, B, T, 0, 1.0 * (ITERS / 4));
    run("lds/dadd/sts private (+lcg)", k_lds_private, B, T, 65536, 1.0 * (ITERS / 4));
    run("atoms.u64 distinct noret", k_atoms_u64<0>, B, T, 65536, 1.0 * (ITERS / 4));
    run("atoms.u64 distinct ret", k_atoms_u64<1>, B, T, 65536, 1.0 * (ITERS / 4));
    run("atoms.u64 4-way", k_atoms_u64<2>, B, T, 65536, 1.0 * (ITERS / 4));
    run("atoms.u64 32-way", k_atoms_u64<3>, B, T, 65536, 1.0 * (ITERS / 4));
    run("atoms.u64 random/400 (+lcg)", k_atoms_u64<4>, B, T, 65536, 1.0 * (ITERS / 4));
    run("atoms.f64 distinct", k_atoms_f64<0>, B, T, 65536, 1.0 * (ITERS / 4));
    run("atoms.f64 random/400 (+lcg)", k_atoms_f64<1>, B, T, 65536, 1.0 * (ITERS / 4));
    run("exact u32 deposit (+lcg)", k_exact, B, T, 400 * 66 * 4, 1.0 * (ITERS / 4));
    run("f64 cas deposit (+lcg)", k_f64cas, B, T, 4096, 1.0 * (ITERS / 4));
  }
  return 0;
}
