// Fused hybrid attention on tcgen05 tensor cores.
//
// Reference semantics (hybrid policy; src/model.cpp:393-427, kernels.cpp:85-168):
//   s_ij = round16( fp32dot(q_i, k_j) * 0.125 )          AttentionScoreMatmul {F16E, F32}
//   s_ij = -inf for j > i                                 decoder causal mask (after scaling)
//   p_ij = e_ij / sum_j e_ij,  e_ij = exp(s_ij - max_j)   Softmax {F32, F32, stabilized}
//   o_i  = round16( fp32dot(round16(p_i), v) )            AttentionScoreMatmul {F16E, F32}
// The whole score row is resident (S <= 512 -> 128 x 512 fp32 = all of TMEM), so
// the softmax is the reference's exact two-pass form (max, then exp/sum, then
// normalise-then-round), not an online rescaling.
//
// One CTA per (batch, head, 128-query tile).  Warp roles:
//   warp 0       TMA: Q tile, all K blocks and all V blocks (separate buffers, issued
//                back to back so V streams in under Q.K^T and the softmax)
//   warp 1       TMEM owner + tcgen05.mma issuer: S = Q.K^T (A, B from smem), then
//                O = P.V with P read straight from TMEM (the "A in TMEM" form)
//   warps 2..17  softmax: 4 warps per TMEM lane quadrant.
//     pass 1  row max of the raw accumulators (round16(x*0.125) is monotone, so the
//             max is rounded once at the end)
//     pass 2  e = 2^(s*log2e - max*log2e) on the SFU, stored back over S (fp32)
//     pass 3  p = round16(e * (1/sum)) packed 2 x fp16 per TMEM column over the
//             already-consumed part of S -> the A operand of the P.V MMA
//
// TMEM columns: S block kb at [128kb, 128kb+128).  "wide" mode (>= 3 key blocks):
// column group g owns key block g and writes P_g into [128g, 128g+64); O lives in
// [64, 128).  "narrow" mode (<= 2 key blocks): group g owns 32*nkb contiguous keys,
// P goes to [256, 256 + 64*nkb), O to [384, 448).
#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

constexpr int kSoftmaxWarps = 16;
constexpr int kThreads = 64 + kSoftmaxWarps * 32;  // 576
constexpr int kMaxKB = 4;                          // S <= 512
constexpr uint32_t kTile = 128 * 64 * 2;           // one 128 x 64 fp16 tile, 16 KB

struct AttnArgs {
  int B, S, H, hd, causal, nqt;
  int h;  // hidden = H * hd (column offset of K; V at 2h)
  __half* ctx;
  int64_t ld_ctx;
  long long* dbg;  // optional per-CTA phase timestamps [grid][8] (clock64), null = off
};

struct Smem {
  static constexpr uint32_t Q = 0;
  static constexpr uint32_t K = Q + kTile;             // 4 tiles
  static constexpr uint32_t V = K + kMaxKB * kTile;    // 4 tiles
  static constexpr uint32_t RED = V + kMaxKB * kTile;  // float [2][4][128]
  static constexpr uint32_t BAR = RED + 2 * 4 * 128 * 4;
  static constexpr uint32_t TOTAL = BAR + 256;
};
constexpr size_t kSmemBytes = 1024 + Smem::TOTAL;

// D[tmem] (+)= A[tmem] * B[smem], kind::f16
__device__ __forceinline__ void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  float* red_max = reinterpret_cast<float*>(smem + Smem::RED);  // [4][128]
  float* red_sum = red_max + 4 * 128;                            // [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;        // [4]
  uint64_t* v_full = bars + 5;        // [4]
  uint64_t* s_full = bars + 9;        // S in TMEM
  uint64_t* p_ready = bars + 10;      // P in TMEM, S consumed
  uint64_t* o_full = bars + 11;       // O in TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int qt = blockIdx.x % a.nqt;
  const int bh = blockIdx.x / a.nqt;
  const int head = bh % a.H, b = bh / a.H;
  const int nkb_all = (a.S + 127) / 128;
  const int nkb = a.causal ? min(qt + 1, nkb_all) : nkb_all;  // key blocks that matter
  const bool wide = nkb > 2;
  const uint32_t o_col = wide ? 64u : 384u;
  const uint32_t warp = warp_id(), lane = lane_id();
  long long* dbg = a.dbg ? a.dbg + static_cast<int64_t>(blockIdx.x) * 8 : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = clock64();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < 12; ++i) mbar_init(&bars[i], i == 10 ? kSoftmaxWarps : 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem = *tmem_slot;
  if (dbg && threadIdx.x == 0) dbg[1] = clock64();

  if (warp == 0) {
    if (lane == 0) {
      pdl_wait();  // q/k/v are written by the upstream QKV GEMM
      mbar_expect_tx(q_full, kTile);
      tma_load_3d(smem + Smem::Q, &tm, q_full, head * 64, qt * 128, b);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_expect_tx(&k_full[kb], kTile);
        tma_load_3d(smem + Smem::K + kb * kTile, &tm, &k_full[kb], a.h + head * 64, kb * 128, b);
      }
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_expect_tx(&v_full[kb], kTile);
        tma_load_3d(smem + Smem::V + kb * kTile, &tm, &v_full[kb], 2 * a.h + head * 64, kb * 128, b);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- S = Q . K^T : M=128 queries, N=128 keys per block, K = 64 (4 x 16)
      constexpr uint32_t idesc_s = idesc_f16_f32(128, 128, 0, 0);
      mbar_wait(q_full, 0);
      if (dbg) dbg[2] = clock64();
      const uint32_t q0 = smem_u32(smem + Smem::Q);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&k_full[kb], 0);
        tc_fence_after();
        const uint32_t k0 = smem_u32(smem + Smem::K + kb * kTile);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_f16_ss(tmem + kb * 128, sw128_desc(q0 + k * 32, 0, 1024),
                      sw128_desc(k0 + k * 32, 0, 1024), idesc_s, k != 0);
      }
      umma_commit(s_full);
      // ---- O = P . V : M=128, N=64 (head dim, V MN-major in smem), K = keys, P in TMEM
      constexpr uint32_t idesc_o = idesc_f16_f32(128, 64, 0, 1);
      mbar_wait(p_ready, 0);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&v_full[kb], 0);
        tc_fence_after();
        const uint32_t v0 = smem_u32(smem + Smem::V + kb * kTile);
        const uint32_t pcol = wide ? 128u * kb : 256u + 64u * kb;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // 16 keys per MMA = 8 packed TMEM columns of P
          umma_f16_ts(tmem + o_col, tmem + pcol + 8 * kk, sw128_desc(v0 + kk * 2048, 128 * 128, 1024),
                      idesc_o, (kb | kk) != 0);
      }
      umma_commit(o_full);
    }
    __syncwarp();
  } else {
    // ---------------- softmax warps ----------------
    const uint32_t sw = warp - 2;
    const uint32_t quad = warp & 3;  // TMEM lane quadrant accessible to this warp
    const uint32_t grp = sw >> 2;    // column group 0..3
    const int r = quad * 32 + lane;  // row within the tile (TMEM lane)
    const int qrow = qt * 128 + r;
    int c_begin, c_end;
    if (wide) {  // group g owns key block g (idle when g >= nkb)
      const bool own = grp < static_cast<uint32_t>(nkb);
      c_begin = own ? static_cast<int>(grp) * 128 : 0;
      c_end = own ? c_begin + 128 : 0;
    } else {
      const int cpg = nkb * 32;
      c_begin = static_cast<int>(grp) * cpg;
      c_end = c_begin + cpg;
    }
    const uint32_t lane_addr = tmem + ((quad * 32) << 16);
    const float NEG_INF = __int_as_float(0xff800000);

    mbar_wait(s_full, 0);
    tc_fence_after();
    const bool stamp = dbg && sw == 0 && lane == 0;
    if (stamp) dbg[3] = clock64();
    // the mask only matters on chunks that cross the sequence end or the diagonal
    // (warp-uniform test: rows of this warp are qt*128 + quad*32 + [0, 32))
    const int row_lo = qt * 128 + quad * 32;
    auto chunk_unmasked = [&](int c) { return c + 32 <= a.S && (!a.causal || c + 31 <= row_lo); };
    // pass 1: max of the raw accumulators over the unmasked keys
    float mraw = NEG_INF;
    for (int c = c_begin; c < c_end; c += 32) {
      uint32_t v[32];
      tmem_ld32(lane_addr + c, v);
      tmem_wait_ld();
      if (chunk_unmasked(c)) {
#pragma unroll
        for (int i = 0; i < 32; ++i) mraw = fmaxf(mraw, __uint_as_float(v[i]));
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int j = c + i;
          const bool valid = j < a.S && (!a.causal || j <= qrow);
          mraw = fmaxf(mraw, valid ? __uint_as_float(v[i]) : NEG_INF);
        }
      }
    }
    red_max[grp * 128 + r] = mraw;
    named_bar_sync(1, kSoftmaxWarps * 32);
    mraw = fmaxf(fmaxf(red_max[r], red_max[128 + r]), fmaxf(red_max[256 + r], red_max[384 + r]));
    const float mx = r16(__fmul_rn(mraw, 0.125f));  // == max_j round16(acc_j * 0.125)
    if (stamp) dbg[4] = clock64();
    // pass 2: e = exp(s - max) kept in TMEM (fp32), partial sums in key order.
    // exp(s - mx) = 2^(s*log2e - mx*log2e): one FFMA + one SFU op per element.
    constexpr float LOG2E = 1.4426950408889634f;
    const float mxl = __fmul_rn(mx, LOG2E);
    float sum = 0.0f;
    for (int c = c_begin; c < c_end; c += 32) {
      uint32_t v[32];
      tmem_ld32(lane_addr + c, v);
      tmem_wait_ld();
      if (chunk_unmasked(c)) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float s = r16(__fmul_rn(__uint_as_float(v[i]), 0.125f));
          const float e = ex2_approx(fmaf(s, LOG2E, -mxl));
          sum = __fadd_rn(sum, e);
          v[i] = __float_as_uint(e);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int j = c + i;
          const float s = r16(__fmul_rn(__uint_as_float(v[i]), 0.125f));
          const bool valid = j < a.S && (!a.causal || j <= qrow);
          const float e = valid ? ex2_approx(fmaf(s, LOG2E, -mxl)) : 0.0f;
          sum = __fadd_rn(sum, e);
          v[i] = __float_as_uint(e);
        }
      }
      tmem_st32(lane_addr + c, v);
    }
    tmem_wait_st();
    if (stamp) dbg[5] = clock64();
    red_sum[grp * 128 + r] = sum;
    named_bar_sync(1, kSoftmaxWarps * 32);
    sum = __fadd_rn(__fadd_rn(__fadd_rn(red_sum[r], red_sum[128 + r]), red_sum[256 + r]),
                    red_sum[384 + r]);
    // pass 3: p = round16(e * (1/sum)), packed fp16 pairs into TMEM (the P.V A operand)
    const float inv = __frcp_rn(sum);
    for (int c = c_begin; c < c_end; c += 32) {
      uint32_t v[32];
      tmem_ld32(lane_addr + c, v);
      tmem_wait_ld();  // the whole chunk is in registers before P overwrites S columns
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        __half2 h2 = __floats2half2_rn(__fmul_rn(__uint_as_float(v[2 * i]), inv),
                                       __fmul_rn(__uint_as_float(v[2 * i + 1]), inv));
        pk[i] = *reinterpret_cast<uint32_t*>(&h2);
      }
      const uint32_t pcol = wide ? static_cast<uint32_t>((c / 128) * 128 + (c % 128) / 2)
                                 : 256u + static_cast<uint32_t>(c / 2);
      tmem_st16(lane_addr + pcol, pk);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(p_ready);
    if (stamp) dbg[6] = clock64();

    // epilogue: O (128 x 64 fp32 in TMEM) -> round16 -> ctx
    mbar_wait(o_full, 0);
    tc_fence_after();
    if (stamp) dbg[7] = clock64();
    if (grp < 2) {
      uint32_t v[32];
      tmem_ld32(lane_addr + o_col + grp * 32, v);
      tmem_wait_ld();
      if (qrow < a.S) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          __half2 h2 = __floats2half2_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
          pk[i] = *reinterpret_cast<uint32_t*>(&h2);
        }
        uint4* dst = reinterpret_cast<uint4*>(a.ctx + (static_cast<int64_t>(b) * a.S + qrow) * a.ld_ctx +
                                              head * 64 + grp * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool attn_tc_supported(int S, int hd) { return hd == 64 && S >= 1 && S <= 512; }

AttnPlan plan_attn_tc(const void* qkv, int64_t ld_qkv, void* ctx, int64_t ld_ctx, int B, int S,
                      int H, int hd, int causal) {
  if (!attn_tc_supported(S, hd)) throw std::invalid_argument("tc attention: needs hd 64, S <= 512");
  if (ld_qkv % 8 != 0 || ld_ctx % 8 != 0) throw std::invalid_argument("tc attention: pitch % 8");
  AttnPlan p{};
  p.tmQKV = make_tmap_f16_3d(qkv, static_cast<uint64_t>(3 * H * hd), S, B, ld_qkv,
                             static_cast<uint64_t>(S) * ld_qkv, 64, 128, 1);
  p.ctx = ctx;
  p.B = B;
  p.S = S;
  p.H = H;
  p.hd = hd;
  p.causal = causal;
  p.ld_qkv = ld_qkv;
  p.ld_ctx = ld_ctx;
  return p;
}

void configure_attn_tc() {
  static bool done = false;
  if (done) return;
  PRLAB_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kSmemBytes)));
  done = true;
}

void launch_attn_tc(const AttnPlan& p, cudaStream_t st) {
  configure_attn_tc();
  AttnArgs a;
  a.B = p.B;
  a.S = p.S;
  a.H = p.H;
  a.hd = p.hd;
  a.causal = p.causal;
  a.nqt = (p.S + 127) / 128;
  a.h = p.H * p.hd;
  a.ctx = reinterpret_cast<__half*>(p.ctx);
  a.ld_ctx = p.ld_ctx;
  a.dbg = p.dbg;
  const int grid = p.B * p.H * a.nqt;
  launch_pdl(attn_tc_kernel, dim3(grid), dim3(kThreads), kSmemBytes, st, p.tmQKV, a);
}

}  // namespace prlab_gpu
