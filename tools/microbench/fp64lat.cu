// Dependent-chain latency of FP64 add / fma on sm_100a (one thread, clock64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/fp64lat.cu -o fp64lat
#include <cstdio>
__global__ void chain(double* out, long long* cyc, double a, double b) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x = x + b;
  }
  long long t1 = clock64();
  double y = a;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) y = __fma_rn(y, a, b);
  }
  long long t2 = clock64();
  double z = a;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) z = z / b;
  }
  long long t3 = clock64();
  out[0] = x + y + z;
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
  cyc[2] = t3 - t2;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMallocManaged(&c, 24);
  for (int r = 0; r < 2; ++r) {
    chain<<<1, 1>>>(o, c, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
  }
  std::printf("cycles per dependent op: dadd %.1f  dfma %.1f  ddiv %.1f\n", c[0] / 8000.0, c[1] / 8000.0, c[2] / 8000.0);
  return 0;
}
