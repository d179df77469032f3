// Primitive costs that decide the round-2 batch-1 trunk design:
//  (P1) bulk DSMEM copies: cp.async.bulk.shared::cluster.shared::cta with complete_tx on the
//       receiver's mbarrier -- every CTA of a cluster sends `bytes` to its neighbour in
//       `chunk`-sized requests; bytes/clock per receiving SM and first-chunk latency.
//  (P2) shared-memory port sharing: one CTA per SM; warp 0 streams an L2-resident buffer
//       into a smem ring with 32 KB cp.async.bulk requests (4 in flight), warp 1 issues
//       back-to-back SS tcgen05 MMAs (M=128, N=32, K=16) on a fixed tile.  Each alone,
//       then both at once: does the MMA rate drop while TMA writes smem?
//  (P3) signal hop with pipelined polling: as ubench_gridbar2's ping-pong, but the waiter
//       keeps 8 loads in flight (lanes 0..7 re-issue staggered) instead of one.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2603_28708_b200/csrc -o ubench_prims ubench_prims.cu
#include <cstdio>
#include "common.cuh"
using namespace prlab_gpu;

// ---------------- P1 ----------------
__global__ void dsmem_kernel(int bytes, int chunk, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t rank = cluster_ctarank();
  uint32_t csize;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  uint8_t* src = sm;
  uint8_t* dst = sm + 96 * 1024;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) mbar_expect_tx(&bar, bytes);
  cluster_sync_all();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t peer = (rank + 1) % csize;
    const uint32_t rdst = mapa_shared(smem_u32(dst), peer), rbar = mapa_shared(smem_u32(&bar), peer);
    for (int off = 0; off < bytes; off += chunk)
      asm volatile(
          "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(rdst + off),
          "r"(smem_u32(src + off)), "r"(chunk), "r"(rbar)
          : "memory");
  }
  if (threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  cluster_sync_all();
}

void run_dsmem(int csize, int bytes, int chunk) {
  long long* d;
  cudaMalloc(&d, 4096 * 8);
  cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (csize > 8) cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  const int grid = csize * (csize > 8 ? 7 : 148 / csize / 2 * 2 / 2);
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 200 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < 3 && e == cudaSuccess; ++r) e = cudaLaunchKernelEx(&cfg, dsmem_kernel, bytes, chunk, d);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"probe\": \"dsmem_bulk\", \"cluster\": %d, \"err\": \"%s\"}\n", csize, cudaGetErrorString(e));
    cudaGetLastError();
    return;
  }
  long long h[4096];
  cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  double mx = 0, sum = 0;
  for (int i = 0; i < grid; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    sum += h[i];
  }
  printf("{\"probe\": \"dsmem_bulk\", \"cluster\": %d, \"ctas\": %d, \"bytes\": %d, \"chunk\": %d, \"cycles_max\": %.0f, "
         "\"cycles_avg\": %.0f, \"B_per_clk_per_sm\": %.1f}\n",
         csize, grid, bytes, chunk, mx, sum / grid, bytes / (sum / grid));
  cudaFree(d);
}

// ---------------- P2 ----------------
constexpr int kRing = 4, kChunk = 32 * 1024;
template <int MODE>  // 1 = ingest only, 2 = mma only, 3 = both
__global__ void __launch_bounds__(128, 1) port_kernel(const uint8_t* buf, long long per_cta, int mma_iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bars[kRing + 1];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint8_t* ring = sm + 32768;  // first 32 KB: the MMA operand tile (A 4 KB + B)
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (warp == 1) {
    tmem_alloc(&slot, 64);
    tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i <= kRing; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t_ing = 0, t_mma = 0;
  const uint8_t* base = buf + (blockIdx.x % 16) * per_cta;  // 16 distinct slices, L2 resident
  if (warp == 0 && lane == 0 && (MODE & 1)) {
    const long long t0 = clock64();
    const int n = static_cast<int>(per_cta / kChunk);
    uint32_t ph[kRing] = {0, 0, 0, 0};
    for (int c = 0; c < n; ++c) {
      const int s = c % kRing;
      if (c >= kRing) {
        mbar_wait(&bars[s], ph[s]);
        ph[s] ^= 1;
      }
      mbar_expect_tx(&bars[s], kChunk);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(ring + s * kChunk)),
                   "l"(base + static_cast<long long>(c) * kChunk), "r"(kChunk), "r"(smem_u32(&bars[s]))
                   : "memory");
    }
    for (int s = 0; s < kRing; ++s) mbar_wait(&bars[s], ph[s]);
    t_ing = clock64() - t0;
  }
  if (warp == 1 && lane == 0 && (MODE & 2)) {
    const long long t0 = clock64();
    constexpr uint32_t idesc = idesc_f16_f32(128, 32, 0, 0);
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 16384);
    for (int it = 0; it < mma_iters; ++it)
      umma_f16_ss(tmem, sw128_desc(a0 + (it & 3) * 32, 0, 1024), sw128_desc(b0 + (it & 3) * 32, 0, 1024), idesc, it != 0);
    umma_commit(&bars[kRing]);
    mbar_wait(&bars[kRing], 0);
    t_mma = clock64() - t0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = t_ing;
  }
  if (threadIdx.x == 32) out[2 * blockIdx.x + 1] = t_mma;
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

template <int MODE>
void run_port(int sms, const uint8_t* buf, long long per_cta, int mma_iters, const char* tag) {
  long long* d;
  cudaMalloc(&d, 4096 * 8);
  const int smem = 32768 + kRing * kChunk + 1024;
  cudaFuncSetAttribute(port_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int r = 0; r < 3; ++r) port_kernel<MODE><<<sms, 128, smem>>>(buf, per_cta, mma_iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"probe\": \"port\", \"err\": \"%s\"}\n", cudaGetErrorString(e));
    return;
  }
  long long h[4096];
  cudaMemcpy(h, d, sms * 16, cudaMemcpyDeviceToHost);
  double ing = 0, mma = 0;
  for (int i = 0; i < sms; ++i) {
    ing += h[2 * i];
    mma += h[2 * i + 1];
  }
  ing /= sms;
  mma /= sms;
  printf("{\"probe\": \"smem_port\", \"mode\": \"%s\", \"ingest_B_per_clk\": %.1f, \"mma_cycles_each\": %.1f, "
         "\"mma_smem_B_per_clk\": %.1f}\n",
         tag, ing > 0 ? per_cta / ing : 0.0, mma > 0 ? mma / mma_iters : 0.0,
         mma > 0 ? mma_iters * 5120.0 / mma : 0.0);
  cudaFree(d);
}

// ---------------- P3 ----------------
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
template <int MODE>  // 0: single ld.acquire poll; 1: 8 lanes ld.relaxed staggered + fence; 2: st.relaxed + relaxed polls (floor)
__global__ void pingpong(unsigned* flags, int iters, long long* out) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  unsigned* mine = flags + 32 * blockIdx.x;
  unsigned* other = flags + 32 * (1 - blockIdx.x);
  auto wait = [&](unsigned v) {
    if (MODE == 0) {
      if (lane == 0)
        while (ld_acq(other) < v) {
        }
    } else {
      bool done = false;
      if (lane < 8) {
        // stagger the lanes so that one load is always in flight
        const long long t = clock64();
        while (clock64() - t < lane * 64) {
        }
      }
      while (!done) {
        const bool ok = lane < 8 && ld_rlx(other) >= v;
        done = __any_sync(0xffffffffu, ok);
      }
      if (MODE == 1 && lane == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncwarp();
  };
  auto signal = [&](unsigned v) {
    if (lane == 0) {
      if (MODE == 2)
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(v) : "memory");
      else
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(v) : "memory");
    }
    __syncwarp();
  };
  const long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    if (blockIdx.x == 0) {
      signal(it);
      wait(it);
    } else {
      wait(it);
      signal(it);
    }
  }
  if (lane == 0) out[blockIdx.x] = clock64() - t0;
}

template <int MODE>
void run_pp(const char* tag) {
  unsigned* f;
  long long* d;
  cudaMalloc(&f, 4096);
  cudaMalloc(&d, 64);
  cudaMemset(f, 0, 4096);
  const int iters = 2000;
  pingpong<MODE><<<2, 32>>>(f, iters, d);
  cudaMemset(f, 0, 4096);
  pingpong<MODE><<<2, 32>>>(f, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2] = {0, 0};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("{\"probe\": \"hop\", \"mode\": \"%s\", \"cycles_per_hop\": %.0f, \"err\": \"%s\"}\n", tag, h[0] / (2.0 * iters),
         cudaGetErrorString(e));
  cudaFree(f);
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_pp<0>("st.release / one ld.acquire poll");
  run_pp<1>("st.release / 8 staggered ld.relaxed polls + fence");
  run_pp<2>("st.relaxed / 8 staggered ld.relaxed polls (floor)");
  for (int cs : {2, 8, 16})
    for (int chunk : {4096, 16384})
      run_dsmem(cs, 64 * 1024, chunk);
  run_dsmem(8, 8192, 8192);
  uint8_t* buf;
  const long long per = 2ll << 20;  // 2 MB per CTA slice, 16 slices = 32 MB (L2 resident)
  cudaMalloc(&buf, 16 * per);
  cudaMemset(buf, 0, 16 * per);
  run_port<1>(sms, buf, per, 4096, "ingest only");
  run_port<2>(sms, buf, per, 4096, "mma only (M128 N32 SS)");
  run_port<3>(sms, buf, per, 4096, "ingest + mma concurrently");
  return 0;
}
