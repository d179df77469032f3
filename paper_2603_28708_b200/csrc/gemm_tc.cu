// tcgen05 GEMM for the hybrid Linear class (reference matmul + linear_bias,
// src/kernels.cpp:40-83 and src/model.cpp:66-78, under the hybrid config
// {F16E compute, F32 accum}: fp16 operands, fp32 accumulation, one final
// round16, then the bias add on the fp16 lattice).
//
//   out[m, n] = epi( sum_k A[m, k] * Wt[n, k] )      A: [M, K] fp16, Wt: [N, K] fp16
//
// Persistent, warp-specialised kernel, one CTA per SM:
//   warp 0      TMA producer: 128x64 A tile + BNx64 W tile per stage (128B swizzle)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..5  epilogue: tcgen05.ld (thread = output row), fused bias / GELU /
//               residual, fp16 or fp32 stores
// Two TMEM accumulator stages (2*BN columns) let the epilogue of tile i overlap
// the main loop of tile i+1.
#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

constexpr int BM = 128, BK = 64;
constexpr int kThreads = 192;

struct GemmArgs {
  int M, N, K;
  int num_m_blocks, num_n_blocks, num_tiles, num_k_blocks;
  const float* bias;
  void* out;
  int64_t ldo;
};

template <int BN>
struct Cfg {
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr size_t SMEM = 1024 + STAGES * STAGE_BYTES + 256;
};

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const uint32_t (&r)[32], const GemmArgs& g, int row,
                                               int col0) {
  if (row >= g.M) return;
  const bool full = col0 + 32 <= g.N;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    float a = r16(__uint_as_float(r[i]));  // round16(fp32 acc): matmul output lattice
    if (EPI != EPI_F16) {
      const int c = col0 + i;
      const float b = (g.bias != nullptr && c < g.N) ? __ldg(g.bias + c) : 0.0f;
      a = r16(__fadd_rn(a, b));  // conform(row + conform(b)), bias stored pre-rounded
      if (EPI == EPI_BIAS_GELU_F16) a = r16(gelu_erf(a));
    }
    v[i] = a;
  }
  if (EPI == EPI_BIAS_RESID_F32) {
    float* o = reinterpret_cast<float*>(g.out) + static_cast<int64_t>(row) * g.ldo + col0;
    if (full && (g.ldo % 4) == 0) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 x = *reinterpret_cast<float4*>(o + i);
        x.x = __fadd_rn(x.x, v[i + 0]);
        x.y = __fadd_rn(x.y, v[i + 1]);
        x.z = __fadd_rn(x.z, v[i + 2]);
        x.w = __fadd_rn(x.w, v[i + 3]);
        *reinterpret_cast<float4*>(o + i) = x;
      }
    } else {
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) o[i] = __fadd_rn(o[i], v[i]);
    }
  } else {
    __half* o = reinterpret_cast<__half*>(g.out) + static_cast<int64_t>(row) * g.ldo + col0;
    if (full && (g.ldo % 8) == 0) {
      uint32_t p[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        __half2 h2 = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        p[i] = *reinterpret_cast<uint32_t*>(&h2);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        reinterpret_cast<uint4*>(o)[i] = make_uint4(p[4 * i], p[4 * i + 1], p[4 * i + 2], p[4 * i + 3]);
    } else {
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) o[i] = __float2half_rn(v[i]);
    }
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmArgs g) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    uint32_t stage = 0, phase = 0;
    for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x) {
      const int m_blk = tile % g.num_m_blocks, n_blk = tile / g.num_m_blocks;
      for (int kb = 0; kb < g.num_k_blocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
          tma_load_2d(sB + stage * C::B_BYTES, &tmB, &full[stage], kb * BK, n_blk * BN);
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = idesc_f16_f32(BM, BN, 0, 0);
    uint32_t stage = 0, phase = 0, t = 0;
    for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x, ++t) {
      const uint32_t acc = t & 1, acc_phase = (t >> 1) & 1;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < g.num_k_blocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_f16_ss(d_tmem, sw128_desc(a0 + k * 32, 0, 1024), sw128_desc(b0 + k * 32, 0, 1024),
                        idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue ----------------
    const uint32_t quad = warp & 3;  // TMEM lane quadrant this warp may access
    uint32_t t = 0;
    for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x, ++t) {
      const int m_blk = tile % g.num_m_blocks, n_blk = tile / g.num_m_blocks;
      const uint32_t acc = t & 1, acc_phase = (t >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m_blk * BM + quad * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((quad * 32) << 16) + acc * BN + c * 32, r);
        tmem_wait_ld();
        epilogue_chunk<EPI>(r, g, row, n_blk * BN + c * 32);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int BN, int EPI>
void configure_one() {
  PRLAB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Cfg<BN>::SMEM)));
}

template <int BN, int EPI>
void launch_one(const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
  gemm_tc_kernel<BN, EPI><<<p.grid, kThreads, Cfg<BN>::SMEM, st>>>(p.tmA, p.tmB, g);
  PRLAB_CUDA(cudaGetLastError());
}

template <int BN>
void configure_bn() {
  configure_one<BN, EPI_BIAS_F16>();
  configure_one<BN, EPI_BIAS_GELU_F16>();
  configure_one<BN, EPI_BIAS_RESID_F32>();
  configure_one<BN, EPI_F16>();
}

template <int BN>
void launch_bn(const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
  switch (p.epi) {
    case EPI_BIAS_F16: launch_one<BN, EPI_BIAS_F16>(p, g, st); break;
    case EPI_BIAS_GELU_F16: launch_one<BN, EPI_BIAS_GELU_F16>(p, g, st); break;
    case EPI_BIAS_RESID_F32: launch_one<BN, EPI_BIAS_RESID_F32>(p, g, st); break;
    case EPI_F16: launch_one<BN, EPI_F16>(p, g, st); break;
    default: throw std::invalid_argument("unknown gemm epilogue");
  }
}

}  // namespace

GemmPlan plan_gemm_tc(const void* A, int64_t lda, const void* Wt, int64_t ldw, const float* bias,
                      void* out, int64_t ldo, int M, int N, int K, int epi) {
  if (M < 1 || N < 1 || K < 1) throw std::invalid_argument("tc gemm: empty extent");
  if (K % 8 != 0 || lda % 8 != 0 || ldw % 8 != 0)
    throw std::invalid_argument("tc gemm: K and row pitches must be multiples of 8");
  GemmPlan p{};
  const int sms = num_sms();
  const int mb = (M + BM - 1) / BM;
  // Pick the widest N tile that still gives every SM work; narrow tiles stream
  // the weights through more SMs when M is small (weight-bandwidth bound).
  int bn = 256;
  while (bn > 64 && static_cast<int64_t>(mb) * ((N + bn - 1) / bn) < sms) bn /= 2;
  p.M = M;
  p.N = N;
  p.K = K;
  p.bn = bn;
  p.epi = epi;
  p.bias = bias;
  p.out = out;
  p.ldo = ldo;
  p.tmA = make_tmap_f16_2d(A, M, K, lda, BM, BK);
  p.tmB = make_tmap_f16_2d(Wt, N, K, ldw, bn, BK);
  const int tiles = mb * ((N + bn - 1) / bn);
  p.grid = tiles < sms ? tiles : sms;
  return p;
}

void configure_gemm_tc() {
  static bool done = false;  // per process; the library drives one device per process
  if (done) return;
  configure_bn<256>();
  configure_bn<128>();
  configure_bn<64>();
  done = true;
}

void launch_gemm_tc(const GemmPlan& p, cudaStream_t st) {
  configure_gemm_tc();
  GemmArgs g;
  g.M = p.M;
  g.N = p.N;
  g.K = p.K;
  g.num_m_blocks = (p.M + BM - 1) / BM;
  g.num_n_blocks = (p.N + p.bn - 1) / p.bn;
  g.num_tiles = g.num_m_blocks * g.num_n_blocks;
  g.num_k_blocks = (p.K + BK - 1) / BK;
  g.bias = p.bias;
  g.out = p.out;
  g.ldo = p.ldo;
  switch (p.bn) {
    case 256: launch_bn<256>(p, g, st); break;
    case 128: launch_bn<128>(p, g, st); break;
    case 64: launch_bn<64>(p, g, st); break;
    default: throw std::invalid_argument("bad tile width");
  }
}

}  // namespace prlab_gpu
