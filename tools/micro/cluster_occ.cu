// How many 2-CTA clusters of the pair-bias backward's shape (512 threads, 231680 B smem) can be
// resident at once, vs single CTAs (cudaOccupancyMaxActiveClusters).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_occ cluster_occ.cu
#include <cstdio>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
  const size_t smem = 231680;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs = 1; cs <= 4; cs *= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(144);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster size %d: max active clusters %d (%d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
