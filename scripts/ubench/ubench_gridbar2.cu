// Grid-barrier protocol costs on a cooperative grid (one CTA per SM, 256 threads), round 2:
// where do the ~2 400 cycles of the round-1 counter barrier go, and which protocol is cheapest?
//   0 base      : bar.sync; t0: red.release.gpu.add ONE counter, spin ld.acquire.gpu; bar.sync
//   1 rlx-spin  : bar.sync; t0: red.release.gpu.add, spin ld.relaxed.gpu, fence.acq_rel.gpu once; bar.sync
//   2 split8    : as 1, CTA i adds into counter[i % 8] (separate 128 B lines); lanes 0..7 poll one each
//   3 fence+rlx : bar.sync; t0: fence.acq_rel.gpu; red.relaxed.gpu.add; spin ld.relaxed; fence; bar.sync
//   4 base+st   : as 1 with every thread storing 64 B to global just before the barrier (release cost
//                 with outstanding stores, like a GEMM epilogue)
//   5 atom-ret  : t0: atom.add.release.gpu (returns the old value); the LAST arriver flips a flag word;
//                 everyone spins ld.relaxed on the flag (one writer, 147 readers)
//   6 pingpong  : CTA 0 and CTA 1 only: alternate st.release / ld.acquire on two flags
//                 -> one-way signal latency (cycles per hop)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_gridbar2 ubench_gridbar2.cu
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
__device__ __forceinline__ void red_rel(unsigned* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(unsigned* ctr, float* sink, int iters, long long* out) {
  const unsigned n = gridDim.x;
  long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    if (MODE == 4) {
      float4* p = reinterpret_cast<float4*>(sink) + (static_cast<size_t>(blockIdx.x) * 256 + threadIdx.x) * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) p[j] = make_float4(it, it, it, it);
    }
    __syncthreads();
    if (MODE == 0) {
      if (threadIdx.x == 0) {
        red_rel(ctr);
        while (ld_acq(ctr) < it * n) {
        }
      }
    } else if (MODE == 1 || MODE == 4) {
      if (threadIdx.x == 0) {
        red_rel(ctr);
        while (ld_rlx(ctr) < it * n) {
        }
        fence_acqrel();
      }
    } else if (MODE == 2) {
      if (threadIdx.x < 32) {
        const unsigned lane = threadIdx.x;
        if (lane == 0) red_rel(ctr + 32 * (blockIdx.x & 7));
        __syncwarp();
        // counter c receives the CTAs i with i % 8 == c
        const unsigned mine = lane < 8 ? (n / 8 + (lane < n % 8 ? 1u : 0u)) * it : 0u;
        bool done = false;
        while (!done) {
          const bool ok = lane >= 8 || ld_rlx(ctr + 32 * lane) >= mine;
          done = __all_sync(0xffffffffu, ok);
        }
        if (lane == 0) fence_acqrel();
      }
    } else if (MODE == 3) {
      if (threadIdx.x == 0) {
        fence_acqrel();
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_rlx(ctr) < it * n) {
        }
        fence_acqrel();
      }
    } else if (MODE == 5) {
      if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
        if (old == it * n - 1) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ctr + 32), "r"(it) : "memory");
        while (ld_rlx(ctr + 32) < static_cast<unsigned>(it)) {
        }
        fence_acqrel();
      }
    } else if (MODE == 6) {
      if (threadIdx.x == 0 && blockIdx.x < 2) {
        unsigned* mine = ctr + 32 * blockIdx.x;
        unsigned* other = ctr + 32 * (1 - blockIdx.x);
        if (blockIdx.x == 0) {
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(it) : "memory");
          while (ld_acq(other) < static_cast<unsigned>(it)) {
          }
        } else {
          while (ld_acq(other) < static_cast<unsigned>(it)) {
          }
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(it) : "memory");
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(int sms, const char* tag, float* sink) {
  unsigned* ctr;
  long long* out;
  cudaMalloc(&ctr, 4096);
  cudaMalloc(&out, 8 * 1024);
  int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(ctr, 0, 4096);
    void* args[] = {&ctr, &sink, &iters, &out};
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
  const double per = mx / iters / (MODE == 6 ? 2.0 : 1.0);
  printf("{\"probe\": \"gridbar2\", \"mode\": \"%s\", \"grid\": %d, \"cycles\": %.0f}\n", tag, sms, per);
  cudaFree(ctr);
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, static_cast<size_t>(sms) * 256 * 64 + 4096);
  run<0>(sms, "base: red.release + ld.acquire spin", sink);
  run<1>(sms, "red.release + ld.relaxed spin + fence", sink);
  run<2>(sms, "split over 8 counters, relaxed poll", sink);
  run<3>(sms, "fence + red.relaxed + relaxed spin + fence", sink);
  run<4>(sms, "as rlx-spin with 64 B stores per thread before", sink);
  run<5>(sms, "atom.add.release, last arriver flips a flag", sink);
  run<6>(sms, "pingpong one-way hop (CTA 0 <-> 1)", sink);
  run<0>(64, "base, 64 CTAs", sink);
  run<1>(64, "rlx-spin, 64 CTAs", sink);
  run<1>(16, "rlx-spin, 16 CTAs", sink);
  return 0;
}
