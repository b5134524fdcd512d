// How many K1-shaped clusters (1024 threads, ~170 KB shared memory per CTA,
// one CTA per SM) can be co-resident on this GPU: cudaOccupancyMaxActiveClusters
// for cluster sizes 1, 2, 4, 8.
#include <cstdio>
__global__ void __launch_bounds__(1024, 1) k(int* out) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 170 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms / c * c);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    std::printf("cluster %d: max active clusters %d (%d CTAs of %d SMs) %s\n", c, n, n * c, sms,
                e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
