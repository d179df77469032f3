// Grid-barrier latency on a cooperative grid (one CTA per SM, 256 threads): cost per
// barrier of the protocols the batch-1 forward kernel could use.
//   counter: bar.sync; thread 0 red.release.gpu.add on ONE counter, spins ld.acquire; bar.sync
//   flags:   bar.sync; thread 0 st.release.gpu of the stage number into ITS flag word; warp 0
//            polls all flags (ld.acquire, lanes stride the array) until every flag >= stage
//   flags_relaxed: as flags, polled with ld.relaxed + one fence.acq_rel.gpu after
//   counter_relaxed: red.relaxed (no release) -- NOT a valid barrier, a floor for the atomic path
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_gridbar ubench_gridbar.cu
#include <cooperative_groups.h>
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
__global__ void __launch_bounds__(256, 1) k(unsigned* ctr, unsigned* flags, int iters, long long* out) {
  const int n = gridDim.x;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    __syncthreads();
    if (MODE == 0 || MODE == 3) {
      if (threadIdx.x == 0) {
        if (MODE == 0)
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        else
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        const unsigned target = static_cast<unsigned>(it) * n;
        while (ld_acq(ctr) < target) {
        }
      }
    } else {
      if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(it) : "memory");
      if (threadIdx.x < 32) {
        bool done = false;
        while (!done) {
          bool ok = true;
          for (int i = threadIdx.x; i < n; i += 32) ok &= (MODE == 1 ? ld_acq(flags + i) : ld_rlx(flags + i)) >= static_cast<unsigned>(it);
          done = __all_sync(0xffffffffu, ok);
        }
        if (MODE == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(int sms, const char* tag) {
  unsigned *ctr, *flags;
  long long* out;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&flags, 4096);
  cudaMalloc(&out, 8 * 1024);
  int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(ctr, 0, 4);
    cudaMemset(flags, 0, 4096);
    void* args[] = {&ctr, &flags, &iters, &out};
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
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"mode\": \"%s\", \"grid\": %d, \"cycles_per_barrier\": %.0f, \"us_per_barrier_at_max_clock\": %.3f}\n", tag, sms,
         mx / iters, mx / iters / (clk / 1e3));
  cudaFree(ctr);
  cudaFree(flags);
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>(sms, "counter (red.release + ld.acquire spin)");
  run<1>(sms, "flags (st.release + ld.acquire poll of all flags)");
  run<2>(sms, "flags (st.release + ld.relaxed poll + fence)");
  run<3>(sms, "counter_relaxed (invalid floor)");
  run<0>(74, "counter, 74 CTAs");
  run<1>(74, "flags, 74 CTAs");
  return 0;
}
