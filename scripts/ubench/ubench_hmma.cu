// Warp-level tensor-core throughput on B200 (mma.sync m16n8k16 fp16 -> fp32): the
// instruction a 16-row-per-cluster batch-1 trunk would use.
// Each warp runs ITERS rounds of INDEP independent MMAs (no dependency between them);
// FLOP/clk/SM = warps_per_sm * ITERS * INDEP * 4096 / cycles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_hmma ubench_hmma.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int INDEP>
__global__ void hmma_kernel(int iters, long long* out, float* sink) {
  float d[INDEP][4];
#pragma unroll
  for (int j = 0; j < INDEP; ++j) d[j][0] = d[j][1] = d[j][2] = d[j][3] = 0.0f;
  const unsigned a0 = 0x3c003c00u ^ threadIdx.x, a1 = 0x3c003c00u, a2 = 0x3c003c00u, a3 = 0x3c003c00u;
  const unsigned b0 = 0x3c003c00u, b1 = 0x3c003c00u ^ (threadIdx.x << 3);
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < INDEP; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
          "{%0, %1, %2, %3};"
          : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  float s = 0.0f;
#pragma unroll
  for (int j = 0; j < INDEP; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
  if (s == 12345.0f) sink[threadIdx.x] = s;
}

template <int INDEP>
void run(int warps, long long* d_out, float* sink) {
  const int iters = 4096;
  hmma_kernel<INDEP><<<1, 32 * warps>>>(iters, d_out, sink);
  cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(&cyc, d_out, sizeof(cyc), cudaMemcpyDeviceToHost);
  const double flop = 2.0 * 16 * 8 * 16 * static_cast<double>(iters) * INDEP * warps;
  printf("{\"probe\": \"mma.sync.m16n8k16.f16.f32\", \"warps_per_sm\": %d, \"independent\": %d, "
         "\"flop_per_clk_per_sm\": %.0f, \"cycles_per_mma_per_warp\": %.2f}\n",
         warps, INDEP, flop / cyc, static_cast<double>(cyc) / (static_cast<double>(iters) * INDEP));
}

int main() {
  long long* d_out;
  float* sink;
  cudaMalloc(&d_out, 1024 * sizeof(long long));
  cudaMalloc(&sink, 1024 * sizeof(float));
  for (int w : {1, 4, 8, 16}) {
    run<1>(w, d_out, sink);
    run<4>(w, d_out, sink);
    run<8>(w, d_out, sink);
  }
  return 0;
}
