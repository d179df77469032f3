// fp32-policy linears on the tensor cores: 3xTF32 tcgen05 GEMM.
//
// out[m, n] = epi( sum_k A[m, k] * W[n, k] ), A and W fp32, K-major (the generic path's
// activations and the fp32 arena's W^T), with the reference linear_bias epilogue under the
// fp32 policy (src/kernels.cpp:40-83, model.cpp:64-82): v = acc (+ bias), then GELU (exact erf,
// kernels.cpp:221-235) or the residual add (kernels.cpp:237-254), all in fp32.
//
// kind::tf32 reads the top 19 bits of each fp32 operand: the tensor core TRUNCATES the low 13
// mantissa bits (measured, scripts/ubench/probe_tf32.cu).  With x_lo = x - trunc(x) (exact in
// fp32, then rounded to nearest tf32) the product is recovered to ~2^-20 relative from three MMAs,
//   x . w  ~=  trunc(x) trunc(w) + x_lo trunc(w) + trunc(x) w_lo,
// fp32-accumulated in TMEM: every product is fp32-accurate to ~1e-6 and only the summation
// order differs from the reference's sequential fp32 sum (the fp32 parity contract is 1e-3
// relative).  w_lo is precomputed once per weight (split_lo); the A tile's x_lo is formed in
// shared memory by the converter warps as each k-block lands.
//
// Tile 128 x BN x 32 (one 128-byte SW128 row = 32 fp32); one output tile per CTA, K optionally
// split over gridDim.z with fp32 partials reduced in fixed order by gemm_tf32_reduce_kernel
// (deterministic).  Warps: 0 TMA, 1 MMA issuer (+ TMEM), 2..5 converter then epilogue.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

constexpr int kBM = 128, kBK = 32;
constexpr uint32_t kMask = 0xFFFFE000u;  // the bits kind::tf32 keeps

// x - trunc19(x), rounded to nearest tf32 (the MMA would truncate it: a biased error)
__device__ __forceinline__ float lo_part(float x) {
  const float lo = __fsub_rn(x, __uint_as_float(__float_as_uint(x) & kMask));
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(lo));
  return __uint_as_float(r);
}

__device__ __forceinline__ void umma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// instruction descriptor, kind::tf32: fp32 D, tf32 A/B (format code 2), K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int BN>
struct TfCfg {
  static constexpr uint32_t A_BYTES = kBM * kBK * 4;  // 16 KB
  static constexpr uint32_t W_BYTES = BN * kBK * 4;
  static constexpr uint32_t STAGE = 2 * A_BYTES + 2 * W_BYTES;  // A, A_lo, W, W_lo
  static constexpr int STAGES = BN >= 128 ? 3 : 4;
  static constexpr uint32_t BAR = STAGES * STAGE;
  static constexpr size_t SMEM = 1024 + BAR + 256;
};

struct TfArgs {
  int M, N, K, kb_per_split;
  const float* bias;   // may be null
  int op;              // 0 none, 1 GELU, 2 residual add of resid
  const float* resid;  // op 2 (may alias out)
  float* out;          // final output, or the split's partial slab (split > 1)
  int64_t ldo;
  int split;           // K splits (gridDim.z)
};

__device__ __forceinline__ float epi_value(const TfArgs& a, float acc, int m, int n) {
  float v = acc;
  if (a.bias) v = __fadd_rn(v, a.bias[n]);
  if (a.op == 1) v = gelu_erf(v);
  if (a.op == 2) v = __fadd_rn(a.resid[static_cast<int64_t>(m) * a.ldo + n], v);
  return v;
}

template <int BN>
__global__ void __launch_bounds__(192, 1) gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap tmA,
                                                             const __grid_constant__ CUtensorMap tmW,
                                                             const __grid_constant__ CUtensorMap tmWlo,
                                                             const TfArgs a) {
  using C = TfCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR);  // TMA landed A, W, W_lo
  uint64_t* conv = full + C::STAGES;                            // converters wrote A_lo
  uint64_t* empty = conv + C::STAGES;                           // MMAs done with the stage
  uint64_t* accf = empty + C::STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accf + 1);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * BN;
  const int kb0 = blockIdx.z * a.kb_per_split;
  const int nkb = min(a.kb_per_split, (a.K + kBK - 1) / kBK - kb0);
  auto sA = [&](int s) { return smem + s * C::STAGE; };
  auto sAlo = [&](int s) { return smem + s * C::STAGE + C::A_BYTES; };
  auto sW = [&](int s) { return smem + s * C::STAGE + 2 * C::A_BYTES; };
  auto sWlo = [&](int s) { return smem + s * C::STAGE + 2 * C::A_BYTES + C::W_BYTES; };

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmWlo);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tslot, BN < 32 ? 32 : BN);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      pdl_wait();
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        mbar_wait(&empty[s], ((i / C::STAGES) & 1) ^ 1);
        mbar_expect_tx(&full[s], C::A_BYTES + 2 * C::W_BYTES);
        const int kc = (kb0 + i) * kBK;
        tma_load_2d(sA(s), &tmA, &full[s], kc, m0);
        tma_load_2d(sW(s), &tmW, &full[s], kc, n0);
        tma_load_2d(sWlo(s), &tmWlo, &full[s], kc, n0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(kBM, BN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        mbar_wait(&conv[s], (i / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA(s)), al = smem_u32(sAlo(s)), w0 = smem_u32(sW(s)), wl = smem_u32(sWlo(s));
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {  // K = 8 per kind::tf32 instruction (32 bytes)
          const uint32_t o = kk * 32;
          // the small terms first, then the main product
          umma_tf32(tmem, sw128_desc(al + o, 0, 1024), sw128_desc(w0 + o, 0, 1024), idesc, (i | kk) != 0);
          umma_tf32(tmem, sw128_desc(a0 + o, 0, 1024), sw128_desc(wl + o, 0, 1024), idesc, 1);
          umma_tf32(tmem, sw128_desc(a0 + o, 0, 1024), sw128_desc(w0 + o, 0, 1024), idesc, 1);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(accf);
    }
    __syncwarp();
  } else {
    // ---------------- converters: A_lo = A - trunc(A) for every landed stage
    const int t = static_cast<int>(threadIdx.x) - 64;  // 0..127
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::STAGES;
      const uint32_t ph = (i / C::STAGES) & 1;
      mbar_wait(&full[s], ph);
      // the previous use of this A_lo slot was read by MMAs that completed (empty) before the
      // TMA refilled the stage, which happened before full[s] fired
      const float4* src = reinterpret_cast<const float4*>(sA(s)) + t * 8;
      float4* dst = reinterpret_cast<float4*>(sAlo(s)) + t * 8;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 x = src[q];
        dst[q] = make_float4(lo_part(x.x), lo_part(x.y), lo_part(x.z), lo_part(x.w));
      }
      fence_proxy_async_smem();  // generic writes -> tensor-core (async proxy) reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
    }
    // ---------------- epilogue: warp w reads TMEM lane quadrant w % 4
    const uint32_t quad = warp & 3;
    const int m = m0 + static_cast<int>(quad * 32 + lane);
    mbar_wait(accf, 0);
    tc_fence_after();
    for (int c = 0; c < BN; c += 32) {
      uint32_t u[32];
      tmem_ld32(tmem + ((quad * 32) << 16) + c, u);
      tmem_wait_ld();
      if (m >= a.M) continue;
      float* orow = a.out + static_cast<int64_t>(m) * a.ldo + n0 + c;
      if (a.split > 1) {  // partial slab [split][M][ldo]: the reduce kernel applies the epilogue
        orow += static_cast<int64_t>(blockIdx.z) * a.M * a.ldo;
        if (n0 + c + 32 <= a.N && (a.ldo % 4) == 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(orow + j) = make_float4(__uint_as_float(u[j]), __uint_as_float(u[j + 1]),
                                                               __uint_as_float(u[j + 2]), __uint_as_float(u[j + 3]));
        } else {
          for (int j = 0; j < 32; ++j)
            if (n0 + c + j < a.N) orow[j] = __uint_as_float(u[j]);
        }
      } else {
        for (int j = 0; j < 32; ++j) {
          const int n = n0 + c + j;
          if (n < a.N) orow[j] = epi_value(a, __uint_as_float(u[j]), m, n);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, BN < 32 ? 32 : BN);
  }
}

// out[m, n] = epi( sum over splits in order of part[s][m][n] )
__global__ void gemm_tf32_reduce_kernel(const float* __restrict__ part, int split, int64_t slab, TfArgs a) {
  const int64_t total = static_cast<int64_t>(a.M) * a.N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int m = static_cast<int>(e / a.N), n = static_cast<int>(e % a.N);
    const int64_t off = static_cast<int64_t>(m) * a.ldo + n;
    float acc = part[off];
    for (int s = 1; s < split; ++s) acc = __fadd_rn(acc, part[s * slab + off]);
    a.out[off] = epi_value(a, acc, m, n);
  }
}

__global__ void split_lo_kernel(const float* __restrict__ w, float* __restrict__ lo, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    lo[i] = lo_part(w[i]);
  }
}

template <int BN>
void configure_tf32() {
  static std::mutex mu;
  static uint64_t done = 0;
  once_per_device(mu, done, [] {
    PRLAB_CUDA(cudaFuncSetAttribute(gemm_tf32x3_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(TfCfg<BN>::SMEM)));
  });
}

}  // namespace

void split_lo(const float* w, float* lo, int64_t n, cudaStream_t st) {
  split_lo_kernel<<<std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4 * num_sms())), 256, 0, st>>>(w, lo, n);
  PRLAB_CUDA(cudaGetLastError());
}

bool gemm_tf32_ok(const float* A, int64_t lda, const float* W, int64_t ldw, int64_t K) {
  if (std::getenv("PRLAB_NO_TF32X3")) return false;
  return K % kBK == 0 && lda % 4 == 0 && ldw % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(W) & 15) == 0;
}

// ws: at least split x M x ldo floats when the GEMM is split (chosen here from the tile count)
void gemm_tf32(const float* A, int64_t lda, const float* W, const float* Wlo, int64_t ldw, float* out, int64_t ldo,
               int M, int N, int K, const float* bias, int op, const float* resid, float* ws, size_t ws_floats,
               cudaStream_t st) {
  const int BN = N >= 128 * 148 / 2 || N % 128 == 0 ? 128 : 64;
  const int tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN);
  const int nkb = K / kBK;
  int split = 1;
  if (tiles < num_sms() && ws != nullptr) {
    split = std::max(1, std::min(num_sms() / tiles, nkb / 4));  // >= 4 k-blocks per split
    while (split > 1 && static_cast<size_t>(split) * M * ldo > ws_floats) --split;
  }
  const int kbs = (nkb + split - 1) / split;
  split = (nkb + kbs - 1) / kbs;
  TfArgs a{M, N, K, kbs, bias, op, resid, split > 1 ? ws : out, ldo, split};
  const CUtensorMap tmA = make_tmap_f32_2d(A, M, K, lda, kBM, kBK);
  const CUtensorMap tmW = make_tmap_f32_2d(W, N, K, ldw, BN, kBK);
  const CUtensorMap tmWlo = make_tmap_f32_2d(Wlo, N, K, ldw, BN, kBK);
  const dim3 grid((M + kBM - 1) / kBM, (N + BN - 1) / BN, split);
  if (BN == 128) {
    configure_tf32<128>();
    launch_pdl(gemm_tf32x3_kernel<128>, grid, dim3(192), TfCfg<128>::SMEM, st, tmA, tmW, tmWlo, a);
  } else {
    configure_tf32<64>();
    launch_pdl(gemm_tf32x3_kernel<64>, grid, dim3(192), TfCfg<64>::SMEM, st, tmA, tmW, tmWlo, a);
  }
  if (split > 1) {
    TfArgs r = a;
    r.out = out;
    const int64_t total = static_cast<int64_t>(M) * N;
    gemm_tf32_reduce_kernel<<<static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * num_sms())), 256, 0, st>>>(
        ws, split, static_cast<int64_t>(M) * ldo, r);
    PRLAB_CUDA(cudaGetLastError());
  }
}

}  // namespace prlab_gpu
