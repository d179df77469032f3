// Weight-stream rate of the cluster batch-1 kernel's layout (fwd_cluster.cu), no compute:
// 4 clusters x 16 CTAs (one per SM, ~216 KB smem), each CTA streams its own contiguous
// slice of a 12-layer weight stream (layer = 888 units of 16 KB; rank c < 12: 60 units,
// else 42) through a ring of `slots` x `chunk` bytes with cp.async.bulk; a consumer thread
// releases each slot as soon as it lands.  Variants: ring geometry, L2 prefetch one layer
// ahead, and a pass over an L2-warm stream (second launch).  Reports B/clk per SM.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2603_28708_b200/csrc -o ubench_cluster_stream ubench_cluster_stream.cu
#include <cstdio>
#include "common.cuh"
using namespace prlab_gpu;

constexpr int kUnitsHead = 60, kUnitsOther = 42, kUnitsLayer = 12 * 60 + 4 * 42;
constexpr uint32_t kUnit = 16384;

__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(288, 1)
    stream_kernel(const uint8_t* ws, int L, int slots, int chunk, int prefetch, long long* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[8], empty[8];
  const int c = static_cast<int>(cluster_ctarank());
  if (threadIdx.x == 0) {
    for (int i = 0; i < slots; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int units = c < 12 ? kUnitsHead : kUnitsOther;
  const int64_t cbase = c < 12 ? kUnitsHead * c : 12 * kUnitsHead + kUnitsOther * (c - 12);
  const int nch = units * kUnit / chunk;
  const long long t0 = clock64();
  if (threadIdx.x == 256) {  // producer
    uint32_t ch = 0;
    auto pf = [&](int l) {
      const uint8_t* src = ws + (static_cast<int64_t>(l) * kUnitsLayer + cbase) * kUnit;
      for (int i = 0; i < units * kUnit / 32768; ++i)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + static_cast<int64_t>(i) * 32768), "r"(32768)
                     : "memory");
    };
    if (prefetch) pf(0);
    for (int l = 0; l < L; ++l) {
      if (prefetch && l + 1 < L) pf(l + 1);
      const uint8_t* src = ws + (static_cast<int64_t>(l) * kUnitsLayer + cbase) * kUnit;
      for (int i = 0; i < nch; ++i, ++ch) {
        const uint32_t s = ch % slots;
        mbar_wait(&empty[s], ((ch / slots) & 1) ^ 1);
        mbar_expect_tx(&full[s], chunk);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + s * chunk)),
                     "l"(src + static_cast<int64_t>(i) * chunk), "r"(chunk), "r"(smem_u32(&full[s]))
                     : "memory");
      }
    }
  } else if (threadIdx.x == 0) {  // consumer: release on arrival
    uint32_t ch = 0;
    for (int l = 0; l < L; ++l)
      for (int i = 0; i < nch; ++i, ++ch) {
        const uint32_t s = ch % slots;
        mbar_wait(&full[s], (ch / slots) & 1);
        mbar_arrive(&empty[s]);
      }
    out[blockIdx.x] = clock64() - t0;
    out[1024 + blockIdx.x] = static_cast<long long>(L) * units * kUnit;
  }
  __syncthreads();
}

void run(const uint8_t* ws, int L, int slots, int chunk, int prefetch, int clusters, const char* tag) {
  long long* d;
  cudaMalloc(&d, 2048 * 8);
  const int smem = 216 * 1024;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int rep = 0; rep < 3; ++rep) stream_kernel<<<16 * clusters, 288, smem>>>(ws, L, slots, chunk, prefetch, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2048];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0, bytes = 0, sum = 0;
  for (int i = 0; i < 16 * clusters; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    sum += static_cast<double>(h[1024 + i]) / h[i];
    bytes += h[1024 + i];
  }
  printf("{\"probe\": \"cluster_stream\", \"mode\": \"%s\", \"clusters\": %d, \"slots\": %d, \"chunk\": %d, \"prefetch\": %d, "
         "\"us_per_layer\": %.2f, \"B_per_clk_per_sm_avg\": %.1f, \"err\": \"%s\"}\n",
         tag, clusters, slots, chunk, prefetch, mx / L / 1965.0, sum / (16 * clusters), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  const int L = 12;
  uint8_t* ws;
  const size_t bytes = static_cast<size_t>(L) * kUnitsLayer * kUnit;
  cudaMalloc(&ws, bytes);
  cudaMemset(ws, 1, bytes);
  // flush L2 between modes with a 256 MB write
  uint8_t* junk;
  cudaMalloc(&junk, 256 << 20);
  auto flush = [&] { cudaMemset(junk, 2, 256 << 20); cudaDeviceSynchronize(); };
  flush(); run(ws, L, 4, 32768, 0, 4, "4x32KB");
  flush(); run(ws, L, 4, 32768, 1, 4, "4x32KB + L2 prefetch");
  flush(); run(ws, L, 2, 65536, 0, 4, "2x64KB");
  flush(); run(ws, L, 6, 32768, 0, 4, "6x32KB");
  flush(); run(ws, L, 8, 16384, 0, 4, "8x16KB");
  flush(); run(ws, L, 4, 32768, 0, 1, "4x32KB one cluster");
  run(ws, 1, 4, 32768, 0, 4, "4x32KB layer 0 L2-warm (after a pass)");
  return 0;
}
