// tcgen05.mma issue-to-completion cost for the attention P.V shapes (sm_100a):
// M=128, K=16 per instruction, fp16 -> fp32, N in {64, 128}; A from smem (ss) or TMEM (ts);
// B K-major or MN-major (128B swizzle).  One CTA per SM, 256 MMAs back to back, one commit.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2603_28708_b200/csrc -o ubench_mma ubench_mma.cu
#include <cstdio>
#include "common.cuh"
using namespace prlab_gpu;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int N, bool TS, bool BMN, int M = 128>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0x3c003c00u;
  if (warp == 0) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_f16_f32(M, N, 0, BMN ? 1 : 0);
    const uint32_t a0 = smem_u32(s), b0 = smem_u32(s + 32768);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint64_t bdesc = BMN ? sw128_desc(b0 + (it & 7) * 2048, 128 * 128, 1024) : sw128_desc(b0 + (it & 3) * 32, 0, 1024);
      if (TS)
        umma_ts(tmem + 256, tmem + (it & 7) * 8, bdesc, idesc, it != 0);
      else
        umma_f16_ss(tmem + 256, sw128_desc(a0 + (it & 3) * 32, 0, 1024), bdesc, idesc, it != 0);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool TS, bool BMN, int M = 128>
void run(int sms, unsigned long long* d_out, const char* tag) {
  const int iters = 256;
  const size_t smem = 65536 + 1024;
  cudaFuncSetAttribute(k<N, TS, BMN, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) k<N, TS, BMN, M><<<sms, 128, smem>>>(iters, d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("{\"err\": \"%s\"}\n", cudaGetErrorString(e)); return; }
  unsigned long long h[1024];
  cudaMemcpy(h, d_out, sms * 8, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < sms; ++i) cyc += h[i];
  cyc /= sms;
  printf("{\"mma\": \"%s\", \"M\": %d, \"N\": %d, \"cycles_per_mma\": %.1f, \"ideal\": %.1f}\n", tag, M, N, cyc / iters,
         M * N / 256.0);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 1024 * 8);
  run<64, false, false>(sms, d_out, "ss B K-major");
  run<64, false, true>(sms, d_out, "ss B MN-major");
  run<64, true, false>(sms, d_out, "ts B K-major");
  run<64, true, true>(sms, d_out, "ts B MN-major");
  run<128, false, false>(sms, d_out, "ss B K-major");
  run<128, true, true>(sms, d_out, "ts B MN-major");
  run<256, false, false>(sms, d_out, "ss B K-major");
  // narrow tiles (batch-1 forward kernel: 128 token rows x 16/32 weight rows)
  run<16, false, false>(sms, d_out, "ss B K-major");
  run<32, false, false>(sms, d_out, "ss B K-major");
  run<32, false, false>(1, d_out, "ss B K-major, one SM");
  // transposed batch-1 tiles: M = 64/128 weight rows x N = 128 tokens
  run<128, false, false, 64>(sms, d_out, "ss B K-major");
  run<64, false, false, 64>(sms, d_out, "ss B K-major");
  return 0;
}
