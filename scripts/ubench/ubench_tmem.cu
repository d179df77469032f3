// Microbenchmarks for the attention softmax design (sm_100a): TMEM load/store
// throughput per SM with 16 warps, MUFU.EX2 throughput, 3-input fmax.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_tmem ubench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld<32>(uint32_t a, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),
                 "=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31])
               : "r"(a));
}
__device__ __forceinline__ void st32(uint32_t a, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               :: "r"(a), "r"(r[0]),"r"(r[1]),"r"(r[2]),"r"(r[3]),"r"(r[4]),"r"(r[5]),"r"(r[6]),"r"(r[7]),"r"(r[8]),"r"(r[9]),"r"(r[10]),"r"(r[11]),"r"(r[12]),"r"(r[13]),"r"(r[14]),"r"(r[15]),
                 "r"(r[16]),"r"(r[17]),"r"(r[18]),"r"(r[19]),"r"(r[20]),"r"(r[21]),"r"(r[22]),"r"(r[23]),"r"(r[24]),"r"(r[25]),"r"(r[26]),"r"(r[27]),"r"(r[28]),"r"(r[29]),"r"(r[30]),"r"(r[31]) : "memory");
}

__global__ void __launch_bounds__(512, 1) k_tmem(int iters, int mode, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t quad = warp & 3, grp = warp >> 2;
  const uint32_t base = tmem + ((quad * 32) << 16) + grp * 128;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = threadIdx.x * 32 + i;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {  // loads, wait after each
    for (int it = 0; it < iters; ++it) {
      ld<32>(base + (it & 3) * 32, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc ^= r[it & 31];
    }
  } else if (mode == 1) {  // 4 loads in flight then wait (needs 128 regs)
    uint32_t q[4][32];
    for (int it = 0; it < iters; it += 4) {
      ld<32>(base + 0, q[0]);
      ld<32>(base + 32, q[1]);
      ld<32>(base + 64, q[2]);
      ld<32>(base + 96, q[3]);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc ^= q[0][it & 31] ^ q[1][3] ^ q[2][5] ^ q[3][7];
    }
  } else if (mode == 2) {  // stores
    for (int it = 0; it < iters; ++it) {
      r[it & 31] += 1;
      st32(base + (it & 3) * 32, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  } else if (mode == 3) {  // ld + st alternating (read-modify-write of the row)
    for (int it = 0; it < iters; ++it) {
      ld<32>(base + (it & 3) * 32, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      r[0] += 1;
      st32(base + (it & 3) * 32, r);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  sink[blockIdx.x * 512 + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

__global__ void __launch_bounds__(512, 1) k_mufu(int iters, int mode, unsigned long long* out, float* sink) {
  float v[8];
  for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  if (mode == 0) {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
  } else {
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(v[i]) : "f"(v[(i + 1) & 7]), "f"(v[(i + 2) & 7]));
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  sink[blockIdx.x * 512 + threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned long long* d_out;
  uint32_t* d_sink;
  cudaMalloc(&d_out, sms * 8);
  cudaMalloc(&d_sink, sms * 512 * 4);
  unsigned long long h[256];
  const int iters = 4096;
  const char* names[] = {"ld32x32b.x32 (wait each)", "ld x32 x4 in flight", "st32x32b.x32", "ld+st rmw"};
  for (int mode = 0; mode < 4; ++mode) {
    k_tmem<<<sms, 512>>>(iters, mode, d_out, d_sink);
    k_tmem<<<sms, 512>>>(iters, mode, d_out, d_sink);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d_out, sms * 8, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < sms; ++i) cyc += h[i];
    cyc /= sms;
    double bytes = 16.0 * 32 * 32 * 4 * iters * (mode == 3 ? 2 : 1);  // per SM
    printf("{\"bench\": \"tmem %s\", \"cycles\": %.0f, \"bytes_per_clk_per_sm\": %.1f}\n", names[mode], cyc, bytes / cyc);
  }
  for (int mode = 0; mode < 2; ++mode) {
    k_mufu<<<sms, 512>>>(iters, mode, d_out, (float*)d_sink);
    k_mufu<<<sms, 512>>>(iters, mode, d_out, (float*)d_sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d_out, sms * 8, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < sms; ++i) cyc += h[i];
    cyc /= sms;
    double ops = 512.0 * 8 * iters;
    printf("{\"bench\": \"%s\", \"cycles\": %.0f, \"lanes_per_clk_per_sm\": %.2f}\n", mode == 0 ? "mufu ex2" : "max3.f32", cyc, ops / cyc);
  }
  return 0;
}
