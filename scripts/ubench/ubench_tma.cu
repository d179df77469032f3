// TMA (cp.async.bulk) ingest microbenchmark: per-SM and chip-wide global->shared
// throughput from L2-resident data, 1 CTA per SM, STAGES x CHUNK bytes in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_tma ubench_tma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(n), "r"(smem_u32(b)) : "memory");
}

template <int STAGES, int CHUNK>
__global__ void k(const uint8_t* src, size_t span, int iters, unsigned long long* out, int order) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + STAGES * CHUNK);
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = span / CHUNK;
  // order 0: CTAs start at scattered chunks; 1: all CTAs read the same chunks in the same
  // order (every SM streams one small activation matrix); 2: same chunks, rotated start
  size_t c = order == 0 ? (size_t)blockIdx.x * 97 : order == 1 ? 0 : (size_t)blockIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < STAGES; ++i) {
    expect_tx(&bars[i], CHUNK);
    bulk(sm + i * CHUNK, src + (c++ % nchunks) * CHUNK, CHUNK, &bars[i]);
  }
  for (int it = 0; it < iters; ++it) {
    const int s = it % STAGES;
    wait(&bars[s], (it / STAGES) & 1);
    expect_tx(&bars[s], CHUNK);
    bulk(sm + s * CHUNK, src + (c++ % nchunks) * CHUNK, CHUNK, &bars[s]);
  }
  for (int i = 0; i < STAGES; ++i) {
    const int it = iters + i;
    wait(&bars[it % STAGES], (it / STAGES) & 1);
  }
  long long t1 = clock64();
  out[blockIdx.x] = (unsigned long long)(t1 - t0);
}

template <int STAGES, int CHUNK>
void run(const uint8_t* d, size_t span, int grid, unsigned long long* d_out, const char* tag, int order = 0) {
  const int iters = 2000;
  size_t smem = STAGES * CHUNK + 1024;
  cudaFuncSetAttribute(k<STAGES, CHUNK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 2; ++rep) k<STAGES, CHUNK><<<grid, 32, smem>>>(d, span, iters, d_out, order);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  unsigned long long h[1024];
  cudaMemcpy(h, d_out, grid * 8, cudaMemcpyDeviceToHost);
  double cyc = 0, mx = 0;
  for (int i = 0; i < grid; ++i) { cyc += h[i]; mx = h[i] > mx ? h[i] : mx; }
  cyc /= grid;
  double bytes = (double)(iters + STAGES) * CHUNK;
  printf("{\"bench\": \"%s\", \"grid\": %d, \"stages\": %d, \"chunk\": %d, \"span_mb\": %.1f, \"B_per_clk_per_sm\": %.1f, \"chip_B_per_clk\": %.0f}\n",
         tag, grid, STAGES, CHUNK, span / 1e6, bytes / cyc, bytes / mx * grid);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* d;
  size_t big = 1ull << 30;
  cudaMalloc(&d, big);
  cudaMemset(d, 1, big);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 1024 * 8);
  run<6, 32768>(d, 32u << 20, sms, d_out, "L2 32MB");
  run<6, 32768>(d, 32u << 20, 1, d_out, "L2 32MB one SM");
  run<6, 32768>(d, 32u << 20, 16, d_out, "L2 32MB 16 SMs");
  run<6, 32768>(d, 32u << 20, 74, d_out, "L2 32MB 74 SMs");
  run<12, 16384>(d, 32u << 20, sms, d_out, "L2 32MB");
  run<3, 65536>(d, 32u << 20, sms, d_out, "L2 32MB");
  run<6, 32768>(d, 1ull << 30, sms, d_out, "DRAM 1GB");
  run<6, 32768>(d, 4u << 20, sms, d_out, "L2 4MB");
  run<8, 16384>(d, 196608, sms, d_out, "hot 196KB same order", 1);
  run<8, 16384>(d, 196608, sms, d_out, "hot 196KB rotated", 2);
  run<8, 16384>(d, 196608, 1, d_out, "hot 196KB one SM", 1);
  run<8, 16384>(d, 32u << 20, sms, d_out, "L2 32MB 8x16KB");
  return 0;
}
