// Cost-model probes for a cluster-per-row-block batch-1 trunk:
//  (1) barrier.cluster (arrive.release + wait.acquire) latency for clusters of 2..16 CTAs,
//      every co-resident cluster looping at once;
//  (2) weight streaming when each of C clusters re-reads the same 14 MB layer of weights
//      (L2-resident after the first pass): CTA r of a cluster streams slice r of it with
//      32 KB cp.async.bulk requests, 4 in flight -- per-SM and aggregate bytes/clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_cluster_trunk ubench_cluster_trunk.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void bar_kernel(int iters, long long* out) {
  cluster_sync();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cluster_sync();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

constexpr int kChunk = 32 * 1024, kInflight = 4;

__global__ void stream_kernel(const char* w, long long slice_bytes, int csize, int passes, long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bars[kInflight];
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const char* base = w + static_cast<long long>(rank) * slice_bytes;
  const int nchunks = static_cast<int>(slice_bytes / kChunk);
  if (threadIdx.x == 0)
    for (int i = 0; i < kInflight; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    uint32_t phase[kInflight] = {0, 0, 0, 0};
    long long g = 0;  // chunks issued over all passes
    auto wait_slot = [&](int s) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n\tselp.u32 %0, 1, 0, q;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(&bars[s])), "r"(phase[s])
            : "memory");
      phase[s] ^= 1;
    };
    for (int p = 0; p < passes; ++p) {
      if (p == 1) t0 = clock64();  // pass 0 pulls the layer into L2
      for (int c = 0; c < nchunks; ++c, ++g) {
        const int s = static_cast<int>(g % kInflight);
        if (g >= kInflight) wait_slot(s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(kChunk)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sm + s * kChunk)),
            "l"(base + static_cast<long long>(c) * kChunk), "r"(kChunk), "r"(smem_u32(&bars[s]))
            : "memory");
      }
    }
    for (long long k = (g > kInflight ? g - kInflight : 0); k < g; ++k) wait_slot(static_cast<int>(k % kInflight));
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kChunk * kInflight);
  long long* d_out;
  cudaMalloc(&d_out, 4096 * sizeof(long long));
  long long h[4096];
  const int iters = 2000;
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    int nclusters = 0;
    cudaOccupancyMaxActiveClusters(&nclusters, (void*)bar_kernel, &cfg);
    cfg.gridDim = dim3(cs * nclusters);
    cudaError_t e = cudaLaunchKernelEx(&cfg, bar_kernel, iters, d_out);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d_out, sizeof(long long) * cs * nclusters, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < cs * nclusters; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("{\"probe\": \"cluster_barrier\", \"cluster\": %d, \"clusters\": %d, \"cycles_per_barrier\": %.1f, \"err\": \"%s\"}\n",
           cs, nclusters, static_cast<double>(mx) / iters, cudaGetErrorString(e));
  }
  // weight streaming: a 14 MB layer split into `cs` slices, every cluster reads all of it
  const long long layer = 14ll << 20;
  char* w;
  cudaMalloc(&w, layer);
  cudaMemset(w, 1, layer);
  for (int cs : {8, 16}) {
    for (int nc : {1, 2, 4, 8}) {
      cudaLaunchConfig_t cfg = {};
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = kChunk * kInflight;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cfg.gridDim = dim3(cs);
      int maxc = 0;
      cudaOccupancyMaxActiveClusters(&maxc, (void*)stream_kernel, &cfg);
      if (nc > maxc) continue;
      cfg.gridDim = dim3(cs * nc);
      const long long slice = (layer / cs) / kChunk * kChunk;
      const int passes = 4;
      cudaError_t e = cudaLaunchKernelEx(&cfg, stream_kernel, (const char*)w, slice, cs, passes, d_out);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d_out, sizeof(long long) * cs * nc, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < cs * nc; ++i) mx = h[i] > mx ? h[i] : mx;
      const double per_sm = static_cast<double>(slice) * (passes - 1) / mx;
      printf("{\"probe\": \"weight_stream\", \"cluster\": %d, \"clusters\": %d, \"slice_MB\": %.2f, "
             "\"cycles_per_layer_slice\": %.0f, \"B_per_clk_per_sm\": %.1f, \"B_per_clk_total\": %.0f, \"err\": \"%s\"}\n",
             cs, nc, slice / 1048576.0, static_cast<double>(mx) / (passes - 1), per_sm, per_sm * cs * nc,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
