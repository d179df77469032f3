// Grid-barrier protocols, round 2 part 2 (cooperative grid, one CTA per SM, 256 threads).
// ubench_gridbar2 found: counter barrier ~2 400 cycles, a release/acquire flag hop ~1 200,
// a relaxed hop ~500.  Here: barriers built from PER-CTA FLAGS instead of one atomic counter.
//   0 counter   : baseline (red.release.gpu on one counter, ld.acquire spin)
//   1 flags-acq : t0 st.release.gpu my flag := it; warp 0 polls all flags, each lane owning
//                 ceil(n/32) flags, every load ld.acquire, all of a lane's loads issued before
//                 the vote
//   2 flags-rlx : as 1 with ld.relaxed polls and ONE fence.acq_rel.gpu after the vote
//   3 flags-rlx + 64 B stores per thread before the barrier
//   4 counter + 64 B stores per thread (baseline with stores)
//   5 flags-rlx, release by fence.acq_rel + st.relaxed (same semantics as st.release)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_gridbar3 ubench_gridbar3.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(unsigned* ctr, unsigned* flags, float* sink, int iters, long long* out) {
  const unsigned n = gridDim.x;
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    if (MODE == 3 || MODE == 4) {
      float4* p = reinterpret_cast<float4*>(sink) + (static_cast<size_t>(blockIdx.x) * 256 + threadIdx.x) * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) p[j] = make_float4(it, it, it, it);
    }
    __syncthreads();
    if (MODE == 0 || MODE == 4) {
      if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_acq(ctr) < it * n) {
        }
      }
    } else if (threadIdx.x < 32) {
      if (lane == 0) {
        if (MODE == 5) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 32), "r"(it) : "memory");
        } else {
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x * 32), "r"(it) : "memory");
        }
      }
      __syncwarp();
      bool done = false;
      while (!done) {
        unsigned v[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          const unsigned i = lane + 32 * j;
          v[j] = i < n ? (MODE == 1 ? ld_acq(flags + i * 32) : ld_rlx(flags + i * 32)) : 0xffffffffu;
        }
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 5; ++j) ok &= v[j] >= static_cast<unsigned>(it);
        done = __all_sync(0xffffffffu, ok);
      }
      if (MODE != 1 && lane == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(int sms, const char* tag, float* sink) {
  unsigned *ctr, *flags;
  long long* out;
  cudaMalloc(&ctr, 4096);
  cudaMalloc(&flags, 160 * 128);
  cudaMalloc(&out, 8 * 1024);
  int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(ctr, 0, 4096);
    cudaMemset(flags, 0, 160 * 128);
    void* args[] = {&ctr, &flags, &sink, &iters, &out};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k<MODE>, dim3(sms), dim3(256), args, 0, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("{\"mode\": \"%s\", \"err\": \"%s\"}\n", tag, cudaGetErrorString(e));
      return;
    }
  }
  long long h[1024];
  cudaMemcpy(h, out, sms * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("{\"probe\": \"gridbar3\", \"mode\": \"%s\", \"grid\": %d, \"cycles\": %.0f}\n", tag, sms, mx / iters);
  cudaFree(ctr);
  cudaFree(flags);
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, static_cast<size_t>(sms) * 256 * 64 + 4096);
  run<0>(sms, "counter (baseline)", sink);
  run<1>(sms, "flags, ld.acquire polls", sink);
  run<2>(sms, "flags, ld.relaxed polls + fence", sink);
  run<3>(sms, "flags relaxed + 64 B stores/thread", sink);
  run<4>(sms, "counter + 64 B stores/thread", sink);
  run<5>(sms, "flags relaxed, fence + st.relaxed release", sink);
  return 0;
}
