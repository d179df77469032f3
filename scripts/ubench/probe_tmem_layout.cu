// TMEM accumulator layouts the round-2 kernels rely on (sm_100a, tcgen05.mma cta_group::1,
// kind::f16, A/B from smem, 128B-swizzled K-major):
//   (a) M = 64 with an fp32 accumulator: which TMEM lanes / columns hold D[m][n]?
//   (b) M = 128 and M = 64 with an FP16 accumulator (idesc c_format = F16): how are the
//       f16 values placed in the 32-bit TMEM cells?
// Probe P sets D[m][n] = m + 1 (A[m][0] = m+1, B[n][0] = 1), probe Q sets D[m][n] = n + 1;
// every lane 0..127 x column 0..63 is dumped raw.  Output: one JSON line per config with
// the decoded (m, n) -> (lane, column, half) map summary.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2603_28708_b200/csrc -o probe_tmem_layout probe_tmem_layout.cu
#include <cstdio>
#include <vector>
#include "common.cuh"
using namespace prlab_gpu;

template <int M, bool F16D, bool PQ>  // PQ false: D = m+1, true: D = n+1
__global__ void __launch_bounds__(128, 1) probe(uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  constexpr int N = 32;
  uint8_t* sA = sm;            // 128 rows x 128 B
  uint8_t* sB = sm + 16384;    // 32 rows x 128 B
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  __syncthreads();
  auto put = [&](uint8_t* base, int r, int k, float v) {
    __half h = __float2half_rn(v);
    const int off = (r / 8) * 1024 + (r % 8) * 128 + (((k / 8) ^ (r % 8)) * 16) + (k % 8) * 2;
    *reinterpret_cast<__half*>(base + off) = h;
  };
  if (threadIdx.x < M) put(sA, threadIdx.x, 0, PQ ? 1.0f : static_cast<float>(threadIdx.x + 1));
  if (threadIdx.x < N) put(sB, threadIdx.x, 0, PQ ? static_cast<float>(threadIdx.x + 1) : 1.0f);
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    tmem_alloc(&slot, 64);
    tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // zero the accumulator region first (all 128 lanes x 64 columns)
  {
    uint32_t z[16] = {};
    for (int c = 0; c < 64; c += 16) tmem_st16(tmem + ((warp * 32) << 16) + c, z);
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    uint32_t idesc = idesc_f16_f32(M, N, 0, 0);
    if (F16D) idesc &= ~(3u << 4);  // c_format = F16
    umma_f16_ss(tmem, sw128_desc(smem_u32(sA), 0, 1024), sw128_desc(smem_u32(sB), 0, 1024), idesc, 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  for (int c = 0; c < 64; c += 32) {
    tmem_ld32(tmem + ((warp * 32) << 16) + c, r);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) out[threadIdx.x * 64 + c + j] = r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

template <int M, bool F16D>
void run(const char* tag) {
  uint32_t* d;
  cudaMalloc(&d, 128 * 64 * 4);
  std::vector<uint32_t> hp(128 * 64), hq(128 * 64);
  cudaFuncSetAttribute(probe<M, F16D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  cudaFuncSetAttribute(probe<M, F16D, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  probe<M, F16D, false><<<1, 128, 40000>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hp.data(), d, hp.size() * 4, cudaMemcpyDeviceToHost);
  probe<M, F16D, true><<<1, 128, 40000>>>(d);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaMemcpy(hq.data(), d, hq.size() * 4, cudaMemcpyDeviceToHost);
  printf("{\"config\": \"%s\", \"M\": %d, \"f16_acc\": %d, \"err\": \"%s\", \"cells\": [", tag, M, (int)F16D,
         cudaGetErrorString(e));
  bool first = true;
  for (int lane = 0; lane < 128; ++lane)
    for (int c = 0; c < 64; ++c) {
      const uint32_t p = hp[lane * 64 + c], q = hq[lane * 64 + c];
      if (p == 0 && q == 0) continue;
      printf("%s[%d,%d,%u,%u]", first ? "" : ",", lane, c, p, q);
      first = false;
    }
  printf("]}\n");
  cudaFree(d);
}

int main() {
  run<128, false>("M128 fp32 acc (reference layout)");
  run<64, false>("M64 fp32 acc");
  run<128, true>("M128 f16 acc");
  run<64, true>("M64 f16 acc");
  return 0;
}
