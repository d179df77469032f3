// How many thread-block clusters of size 2/4/8 can be co-resident with one
// ~200 KB-smem CTA per SM (cudaOccupancyMaxActiveClusters) -- sizing the grid of
// persistent cluster kernels.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dummy(int* p) { if (p) p[blockIdx.x] = 1; }
int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    printf("{\"cluster\": %d, \"max_active_clusters\": %d, \"ctas\": %d, \"err\": \"%s\"}\n", cs, n, n * cs,
           cudaGetErrorString(e));
  }
  return 0;
}
