// Can the persistent trunk run as a cooperative grid of 2-CTA clusters (148 CTAs, one per SM)?
// And what does a split-K partial exchange cost: each CTA writes half of a 128 x 32 fp32 tile
// (8 KB) into its partner's shared memory with st.shared::cluster, then a cluster barrier.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2603_28708_b200/csrc -o probe_coop_cluster probe_coop_cluster.cu
#include <cstdio>
#include "common.cuh"
using namespace prlab_gpu;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) k(unsigned* gbar, long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* buf = reinterpret_cast<float*>(sm);
  const uint32_t rank = cluster_ctarank();
  // grid barrier once (cooperative co-residency check)
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(gbar, 1u);
    while (atomicAdd(gbar, 0u) < gridDim.x) {}
  }
  __syncthreads();
  cluster_sync_all();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // 8 KB: 256 threads x 2 float4
    const uint32_t peer = mapa_shared(smem_u32(buf + 2048 * (it & 1)), rank ^ 1);
    for (int q = 0; q < 2; ++q)
      st_dsmem_f4(peer + (threadIdx.x * 2 + q) * 16, make_float4(it, rank, threadIdx.x, q));
    cluster_sync_all();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
}

int main() {
  unsigned* gbar;
  long long* out;
  cudaMalloc(&gbar, 4);
  cudaMalloc(&out, 148 * 8);
  cudaMemset(gbar, 0, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int iters = 100;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, gbar, out, iters);
  cudaError_t e2 = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  printf("{\"probe\": \"coop_cluster2\", \"launch\": \"%s\", \"sync\": \"%s\", \"cycles_per_8KB_exchange_plus_cluster_barrier\": %.0f}\n",
         cudaGetErrorString(e), cudaGetErrorString(e2), avg / 148);
  return 0;
}
