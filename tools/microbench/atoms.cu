// Shared-memory 32-bit atomic add throughput on sm_100a: warp-instructions and
// thread-ops per clock per SM for conflict-free, random-within-histogram and
// return-dependent chains (the K1 bin deposit pattern).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t atoms_add(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v));
  return old;
}
__device__ __forceinline__ void reds_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
}
template <int MODE>
__global__ void k(uint32_t* out, int iters, uint32_t nwords) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) s[i] = 0;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(s);
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x, acc = 0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x = x * 1664525u + 1013904223u;
      uint32_t w;
      if (MODE == 0) w = ((x >> 8) % (nwords / 32)) * 32 + lane;       // conflict-free (bank = lane)
      else w = (x >> 8) % nwords;                                      // random
      if (MODE == 2) reds_add(base + 4 * w, x);
      else acc += atoms_add(base + 4 * w, x);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0] + acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* out; cudaMalloc(&out, 4096 * 4);
  const uint32_t nwords = 400 * 67;
  const int iters = 2000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[3] = {"atoms conflict-free (ret)", "atoms random 400x67 (ret)", "reds random 400x67 (noret)"};
  for (int mode = 0; mode < 3; ++mode)
    for (int thr : {256, 512, 1024}) {
      auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, nwords * 4);
      kern<<<sms, thr, nwords * 4>>>(out, 10, nwords);
      cudaEventRecord(a);
      kern<<<sms, thr, nwords * 4>>>(out, iters, nwords);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)sms * thr * iters * 8;
      const double clks = ms * 1e-3 * clk * 1e3;
      printf("%-30s thr=%4d: %.2f thread-ops/clk/SM  %.3f warp-instr/clk/SM\n", names[mode], thr, ops / clks / sms,
             ops / 32 / clks / sms);
    }
  return 0;
}
