// tcgen05.mma kind::tf32 semantics probe (sm_100a): instruction-descriptor format codes and how
// the tensor core reduces an fp32 operand to tf32 (truncation vs round-to-nearest) -- the
// 3xTF32 split used by the fp32-policy GEMMs depends on it.  One CTA, M=128 N=64 K=8.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2603_28708_b200/csrc -o probe_tf32 probe_tf32.cu
#include <cstdio>
#include <cstring>
#include "common.cuh"
using namespace prlab_gpu;

__device__ __forceinline__ void umma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc),
               "r"(acc)
               : "memory");
}

// element (row, k) of a K-major SW128 tile of 4-byte elements (32 per 128-byte row)
__device__ __forceinline__ uint32_t sw_off(int row, int k) {
  const int chunk = (k * 4) >> 4;
  return row * 128 + ((chunk ^ (row & 7)) << 4) + ((k * 4) & 15);
}

__global__ void k(float a0, float b0, uint32_t fmt, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  float* A = reinterpret_cast<float*>(s);            // 128 rows x 32
  float* B = reinterpret_cast<float*>(s + 16384);    // 64 rows x 32
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
    const int r = i / 32, kk = i % 32;
    *reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(A) + sw_off(r, kk)) = kk == 0 ? a0 : (kk == 1 ? 1.0f : 0.0f);
  }
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) {
    const int r = i / 32, kk = i % 32;
    *reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(B) + sw_off(r, kk)) = kk == 0 ? b0 : (kk == 1 ? (float)r : 0.0f);
  }
  const int warp = threadIdx.x / 32;
  if (warp == 0) { tmem_alloc(&slot, 64); tmem_relinquish(); }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    umma_tf32(tmem, sw128_desc(smem_u32(A), 0, 1024), sw128_desc(smem_u32(B), 0, 1024), idesc, 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  if (warp < 4) {
    uint32_t u[32];
    tmem_ld32(tmem + ((warp * 32) << 16), u);
    tmem_wait_ld();
    const int row = warp * 32 + threadIdx.x % 32;
    for (int j = 0; j < 32; ++j) out[row * 64 + j] = __uint_as_float(u[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 64); }
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 64 * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const float a0 = 1.0f + 0.75f / 1024.0f;  // between tf32 neighbours 1 and 1 + 2^-10
  for (uint32_t fmt : {2u, 1u, 0u}) {
    cudaMemset(d, 0, 128 * 64 * 4);
    k<<<1, 128, 64 * 1024>>>(a0, 1.0f, fmt, d);
    cudaError_t e = cudaDeviceSynchronize();
    float h[128 * 64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    // D[r][n] = a0 * 1 + 1 * n (n < 32 here): n = 0 -> a0 as the unit rounded it; n = 5 -> a0 + 5
    printf("{\"probe\": \"tf32\", \"fmt\": %u, \"err\": \"%s\", \"d00\": %.10f, \"d05\": %.10f, \"d_r77_n31\": %.10f, "
           "\"exact\": %.10f, \"trunc\": 1.0, \"rn\": %.10f}\n",
           fmt, cudaGetErrorString(e), h[0], h[5], h[77 * 64 + 31], a0, 1.0 + 1.0 / 1024.0);
  }
  return 0;
}
