// MUFU ex2 throughput on one SM (f32 and f16x2), and the FFMA2 rate for reference:
// 1 CTA x W warps, 8 independent chains per thread, clock64 around the loop.
#include <cstdio>
#include <cuda_fp16.h>
__global__ void k_ex2(float* out, long long* cyc, int iters) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_ex2h(float* out, long long* cyc, int iters) {
  unsigned x[8];
  for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(-0.001f * threadIdx.x, -0.002f * i); x[i] = *reinterpret_cast<unsigned*>(&h); }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x[i]));
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += __half2float(__low2half(*reinterpret_cast<__half2*>(&x[i])));
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 4096 * 4); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    for (int v = 0; v < 2; ++v) {
      for (int rep = 0; rep < 2; ++rep) {
        if (v == 0) k_ex2<<<1, 32 * warps>>>(out, cyc, iters); else k_ex2h<<<1, 32 * warps>>>(out, cyc, iters);
      }
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double ops = 8.0 * iters * 32 * warps;  // instructions x threads
      printf("{\"op\": \"%s\", \"warps\": %d, \"cycles\": %lld, \"thread_ops_per_clk_per_sm\": %.2f}\n",
             v == 0 ? "ex2.approx.ftz.f32" : "ex2.approx.f16x2", warps, c, ops / c);
    }
  }
  return 0;
}
