// Per-SM throughput of the softmax/epilogue instruction mix on sm_100a:
// FFMA, FFMA2, HADD2.F32 (cvt.f32.f16), F2FP (cvt.rn.f16x2.f32), MUFU.EX2 and mixes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_pipes ubench_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define N 16
template <int mode>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* out, float* sink) {
  float f[N];
  uint32_t h[N];
  uint64_t d[N];
  for (int i = 0; i < N; ++i) {
    f[i] = 0.001f * (threadIdx.x + i) - 1.0f;
    h[i] = 0x3c003c00u + threadIdx.x + i;
    asm("mov.b64 %0, {%1,%1};" : "=l"(d[i]) : "f"(f[i]));
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if constexpr (mode == 0) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A000000;" : "+f"(f[i]));
      if constexpr (mode == 1) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(d[i]));
      if constexpr (mode == 2) { float x; asm volatile("cvt.f32.f16 %0, %1;" : "=f"(x) : "h"((unsigned short)h[i])); f[i] += 0.0f; asm volatile("mov.b32 %0, %1;" : "=r"(h[i]) : "r"(__float_as_uint(x))); }
      if constexpr (mode == 3) asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h[i]) : "f"(f[i]), "f"(__uint_as_float(h[i])));
      if constexpr (mode == 4) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if constexpr (mode == 5) asm volatile("add.rn.f32x2 %0, %0, %0;" : "+l"(d[i]));
      if constexpr (mode == 6) asm volatile("max.f32 %0, %0, %1, %0;" : "+f"(f[i]) : "f"(f[(i + 1) % N]));
      if constexpr (mode == 7) asm volatile("mad.lo.u32 %0, %0, 8388608, %0;" : "+r"(h[i]));
      // mixes: one op of each kind per i (independent chains)
      if constexpr (mode == 8) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i])); asm volatile("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(h[i]) : "f"(__uint_as_float(h[i]))); }
      if constexpr (mode == 9) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i])); float x; asm volatile("cvt.f32.f16 %0, %1;" : "=f"(x) : "h"((unsigned short)h[i])); h[i] = __float_as_uint(x); }
      if constexpr (mode == 10) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i])); asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(d[i])); }
      if constexpr (mode == 11) { asm volatile("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(h[i]) : "f"(__uint_as_float(h[i]))); asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(d[i])); }
      if constexpr (mode == 12) { float x; asm volatile("cvt.f32.f16 %0, %1;" : "=f"(x) : "h"((unsigned short)h[i])); h[i] = __float_as_uint(x); asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(d[i])); }
      if constexpr (mode == 13) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i])); asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A000000;" : "+f"(f[(i + 8) % N])); }
      if constexpr (mode == 14) { asm volatile("cvt.rn.f16x2.f32 %0, %1, %1;" : "=r"(h[i]) : "f"(__uint_as_float(h[i]))); asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3A000000;" : "+f"(f[i])); }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  float s = 0;
  for (int i = 0; i < N; ++i) {
    float a, b;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(d[i]));
    s += f[i] + a + b + __uint_as_float(h[i]);
  }
  sink[blockIdx.x * 512 + threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d_out;
  float* d_sink;
  cudaMalloc(&d_out, sms * 8);
  cudaMalloc(&d_sink, sms * 512 * 4);
  const char* names[] = {"FFMA", "FFMA2 (pair)", "cvt.f32.f16 (HADD2.F32)", "cvt.rn.f16x2.f32 (F2FP)", "MUFU.EX2",
                         "FADD2 (pair)", "FMNMX3", "IMAD", "mix MUFU+F2FP", "mix MUFU+HADD2.F32", "mix MUFU+FFMA2",
                         "mix F2FP+FFMA2", "mix HADD2.F32+FFMA2", "mix MUFU+FFMA", "mix F2FP+FFMA"};
  unsigned long long hb[1024];
  for (int mode = 0; mode < 15; ++mode) {
    const int iters = 2048;
    for (int rep = 0; rep < 2; ++rep) {
      switch (mode) {
        case 0: k<0><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 1: k<1><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 2: k<2><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 3: k<3><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 4: k<4><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 5: k<5><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 6: k<6><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 7: k<7><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 8: k<8><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 9: k<9><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 10: k<10><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 11: k<11><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 12: k<12><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 13: k<13><<<sms, 512>>>(iters, d_out, d_sink); break;
        case 14: k<14><<<sms, 512>>>(iters, d_out, d_sink); break;
      }
    }
    cudaDeviceSynchronize();
    cudaMemcpy(hb, d_out, sms * 8, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < sms; ++i) cyc += hb[i];
    cyc /= sms;
    printf("{\"op\": \"%s\", \"warp_instr_per_clk_per_sm\": %.3f}\n", names[mode], (mode >= 8 ? 2.0 : 1.0) * 16.0 * iters * N / cyc);
  }
  return 0;
}
