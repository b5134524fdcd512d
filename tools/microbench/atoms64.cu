// Shared-memory 64-bit vs 32-bit atomic add throughput on sm_100a (random
// addresses in a K1-sized histogram, returned values consumed).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t atoms_add32(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v));
  return old;
}
__device__ __forceinline__ unsigned long long atoms_add64(uint32_t addr, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.shared.add.u64 %0, [%1], %2;" : "=l"(old) : "r"(addr), "l"(v));
  return old;
}
template <int W>
__global__ void k(unsigned long long* out, int iters, uint32_t nbytes) {
  extern __shared__ unsigned long long s[];
  for (int i = threadIdx.x; i < nbytes / 8; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(s);
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
  unsigned long long acc = 0;
  const uint32_t n = nbytes / (W == 64 ? 8 : 4);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x = x * 1664525u + 1013904223u;
      const uint32_t w = (x >> 8) % n;
      if (W == 64) acc += atoms_add64(base + 8 * w, x);
      else acc += atoms_add32(base + 4 * w, x);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0] + acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned long long* out; cudaMalloc(&out, 4096 * 8);
  const uint32_t nbytes = 170 * 1024;
  const int iters = 2000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w : {32, 64})
    for (int thr : {512, 1024}) {
      auto kern = w == 64 ? k<64> : k<32>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, nbytes);
      kern<<<sms, thr, nbytes>>>(out, 10, nbytes);
      cudaEventRecord(a);
      kern<<<sms, thr, nbytes>>>(out, iters, nbytes);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)sms * thr * iters * 8;
      const double clks = ms * 1e-3 * clk * 1e3;
      printf("atom.shared.add.u%d random thr=%4d: %.2f thread-ops/clk/SM\n", w, thr, ops / clks / sms);
    }
  return 0;
}
