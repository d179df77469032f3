// tcgen05.mma cost for the batch-1 trunk's skinny tiles (sm_100a): is the ~47-cycle floor per
// K=16 instruction a dependent-accumulation latency (independent accumulators would overlap) or
// an issue/throughput floor?  One CTA per SM, `iters` MMAs round-robin over C accumulators,
// one commit; A from smem (ss) or TMEM (ts).
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2603_28708_b200/csrc -o ubench_mma2 ubench_mma2.cu
#include <cstdio>
#include "common.cuh"
using namespace prlab_gpu;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int M, int N, int C, bool TS>
__global__ void __launch_bounds__(128, 1) k(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0x3c003c00u;
  if (warp == 0) { tmem_alloc(&slot, 512); tmem_relinquish(); }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_f16_f32(M, N, 0, 0);
    const uint32_t a0 = smem_u32(s), b0 = smem_u32(s + 65536);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const int ch = it % C;
      const uint32_t d = tmem + 256 + ch * 64;
      // walk a 48 KB A region / 24 KB B region like a K = 768 task
      const uint64_t bdesc = sw128_desc(b0 + ((it >> 2) % 12) * (N * 128) + (it & 3) * 32, 0, 1024);
      if (TS)
        umma_ts(d, tmem + (it & 31) * 8, bdesc, idesc, it >= C);
      else
        umma_f16_ss(d, sw128_desc(a0 + ((it >> 2) % 12) * (M * 128 / 2 >= 4096 ? M * 128 : 8192) % 65536 + (it & 3) * 32, 0, 1024),
                    bdesc, idesc, it >= C);
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

template <int M, int N, int C, bool TS>
void run(int sms, unsigned long long* d_out, int iters) {
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k<M, N, C, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) k<M, N, C, TS><<<sms, 128, smem>>>(iters, d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("{\"err\": \"%s\"}\n", cudaGetErrorString(e)); return; }
  unsigned long long h[1024];
  cudaMemcpy(h, d_out, sms * 8, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < sms; ++i) cyc += h[i];
  cyc /= sms;
  printf("{\"probe\": \"mma2\", \"M\": %d, \"N\": %d, \"accumulators\": %d, \"a\": \"%s\", \"iters\": %d, \"cycles_total\": %.0f, \"cycles_per_mma\": %.1f}\n",
         M, N, C, TS ? "tmem" : "smem", iters, cyc, cyc / iters);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 1024 * 8);
  for (int iters : {48, 256}) {
    run<64, 32, 1, false>(sms, d_out, iters);
    run<64, 32, 2, false>(sms, d_out, iters);
    run<64, 32, 4, false>(sms, d_out, iters);
    run<64, 64, 1, false>(sms, d_out, iters);
    run<64, 16, 1, false>(sms, d_out, iters);
    run<128, 16, 1, false>(sms, d_out, iters);
    run<128, 16, 4, false>(sms, d_out, iters);
    run<128, 32, 1, false>(sms, d_out, iters);
    run<128, 32, 2, false>(sms, d_out, iters);
    run<128, 32, 4, false>(sms, d_out, iters);
    run<128, 64, 1, false>(sms, d_out, iters);
    run<128, 64, 4, false>(sms, d_out, iters);
    run<128, 32, 1, true>(sms, d_out, iters);
    run<128, 32, 4, true>(sms, d_out, iters);
    run<64, 32, 1, true>(sms, d_out, iters);
    run<64, 32, 4, true>(sms, d_out, iters);
  }
  return 0;
}
