// Tensor-map TMA ingest of ONE small activation matrix (A = [128 rows x K] fp16, SW128)
// streamed by every SM at once -- the A-operand pattern of the batch-1 forward kernel.
// Compares request sizes: 2D boxes of 64 or 128 rows (8 / 16 KB per request) against a
// 3D view (k-block index as the outer dimension) whose boxes cover 2 or 4 k-blocks
// (32 / 64 KB per request) with the same bytes in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_tma2d ubench_tma2d.cu -lcuda
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
                   smem_u32(b)), "r"(ph)
               : "memory");
}
__device__ __forceinline__ void load2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)), "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void load3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)), "l"(m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// mode 0: 2D, `sub` requests of (64 cols x 128/sub rows) per k-block; mode 1: 3D, one
// request of `kpr` k-blocks.  Stage = kpr k-blocks (kpr * 16 KB).
__global__ void k(const __grid_constant__ CUtensorMap m, int mode, int sub, int kpr, int stages, int nkb, int iters,
                  unsigned long long* out, int br, int nrb) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t kb_bytes = br * 128, stage_bytes = kpr * kb_bytes;
  const int row0 = (blockIdx.x % nrb) * br;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + stages * stage_bytes);
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int nunits = nkb / kpr;
  auto issue = [&](int u, int s) {
    const int kb0 = (u % nunits) * kpr;
    expect_tx(&bars[s], stage_bytes);
    uint8_t* dst = sm + s * stage_bytes;
    if (mode == 0) {
      for (int j = 0; j < kpr; ++j)
        for (int r = 0; r < sub; ++r)
          load2d(dst + j * kb_bytes + r * (kb_bytes / sub), &m, &bars[s], (kb0 + j) * 64, row0 + r * (br / sub));
    } else {
      load3d(dst, &m, &bars[s], 0, row0, kb0);
    }
  };
  long long t0 = clock64();
  for (int i = 0; i < stages; ++i) issue(i, i);
  for (int it = 0; it < iters; ++it) {
    const int s = it % stages;
    wait(&bars[s], (it / stages) & 1);
    issue(it + stages, s);
  }
  for (int i = 0; i < stages; ++i) {
    const int it = iters + i;
    wait(&bars[it % stages], (it / stages) & 1);
  }
  long long t1 = clock64();
  out[blockIdx.x] = (unsigned long long)(t1 - t0);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fnp;
  unsigned long long* d_out;
  cudaMalloc(&d_out, 1024 * 8);
  struct Shape { int R, K, br; const char* what; };
  Shape shapes[] = {{128, 768, 128, "hot A 128x768 (batch-1)"}, {4096, 768, 128, "A 4096x768, 128-row boxes"},
                    {2304, 768, 256, "W 2304x768, 256-row boxes"}, {4096, 768, 64, "A 4096x768, 64-row boxes"}};
  for (auto& sh : shapes) {
    const int K = sh.K, br = sh.br, nrb = sh.R / br;
    void* a;
    cudaMalloc(&a, (size_t)sh.R * K * 2);
    cudaMemset(a, 0, (size_t)sh.R * K * 2);
    const int nkb = K / 64;
    struct Cfg { int mode, kpr, stages; const char* tag; };
    const int kbk = br * 128 / 1024;  // KB per k-block
    Cfg cfgs[] = {{0, 1, 128 / kbk, "2d, 1 k-block per request"}, {0, 2, 64 / kbk, "2d x2 requests per stage"},
                  {1, 1, 128 / kbk, "3d, 1 k-block per request"}, {1, 2, 64 / kbk, "3d, 2 k-blocks per request"},
                  {1, 4, 32 / kbk > 0 ? 32 / kbk : 1, "3d, 4 k-blocks per request"}};
    for (auto& c : cfgs) {
      CUtensorMap m;
      CUresult r;
      if (c.mode == 0) {
        cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)sh.R};
        cuuint64_t strides[1] = {(cuuint64_t)K * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)br};
        cuuint32_t es[2] = {1, 1};
        r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      } else {
        cuuint64_t dims[3] = {64, (cuuint64_t)sh.R, (cuuint64_t)nkb};
        cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
        cuuint32_t box[3] = {64, (cuuint32_t)br, (cuuint32_t)c.kpr};
        cuuint32_t es[3] = {1, 1, 1};
        r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
      if (r != CUDA_SUCCESS) {
        printf("{\"shape\": \"%s\", \"tag\": \"%s\", \"encode_error\": %d}\n", sh.what, c.tag, (int)r);
        continue;
      }
      const size_t smem = (size_t)c.stages * c.kpr * br * 128 + 1024;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int iters = 3000 / c.kpr;
      for (int grid : {1, sms}) {
        for (int rep = 0; rep < 2; ++rep)
          k<<<grid, 32, smem>>>(m, c.mode, 1, c.kpr, c.stages, nkb, iters, d_out, br, nrb);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("{\"tag\": \"%s\", \"err\": \"%s\"}\n", c.tag, cudaGetErrorString(e));
          return 1;
        }
        unsigned long long h[1024];
        cudaMemcpy(h, d_out, grid * 8, cudaMemcpyDeviceToHost);
        double cyc = 0, mx = 0;
        for (int i = 0; i < grid; ++i) {
          cyc += h[i];
          mx = h[i] > mx ? h[i] : mx;
        }
        cyc /= grid;
        const double bytes = (double)(iters + c.stages) * c.kpr * br * 128;
        printf("{\"shape\": \"%s\", \"tag\": \"%s\", \"in_flight_kb\": %d, \"grid\": %d, \"B_per_clk_per_sm\": %.1f, \"chip_B_per_clk\": %.0f}\n",
               sh.what, c.tag, (int)(c.stages * c.kpr * kbk), grid, bytes / cyc, bytes / mx * grid);
      }
    }
    cudaFree(a);
  }
  return 0;
}
