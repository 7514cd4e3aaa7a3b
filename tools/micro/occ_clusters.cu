#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
  int smems[3] = {231680, 166144, 100000};
  for (int cs = 1; cs <= 4; cs *= 2) for (int i = 0; i < 3; ++i) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smems[i]);
    cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(144); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smems[i]; cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %d smem %d: max active clusters %d (%s) -> CTAs %d\n", cs, smems[i], n, cudaGetErrorString(e), n * cs);
  }
}
