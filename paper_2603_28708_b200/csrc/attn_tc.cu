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
//   warp 0       TMA: Q tile, K blocks (128 keys each), then V blocks into the K buffers
//   warp 1       TMEM owner + tcgen05.mma issuer (S = Q.K^T, then O = P.V)
//   warps 2..17  softmax: 4 warps per TMEM lane quadrant, each owning a quarter of
//                the key columns; P is written as fp16 into a 128B-swizzled K-major
//                smem operand that the P.V MMA reads directly.
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
  static constexpr uint32_t KV = Q + kTile;                 // 4 tiles
  static constexpr uint32_t P = KV + kMaxKB * kTile;        // 8 tiles (128 x 512 fp16)
  static constexpr uint32_t RED = P + 2 * kMaxKB * kTile;   // float [2][4][128]
  static constexpr uint32_t BAR = RED + 2 * 4 * 128 * 4;
  static constexpr uint32_t TOTAL = BAR + 256;
};
constexpr size_t kSmemBytes = 1024 + Smem::TOTAL;

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
  uint64_t* s_full = bars + 9;        // S in TMEM (and K buffers free)
  uint64_t* p_ready = bars + 10;      // P in smem, S consumed
  uint64_t* o_full = bars + 11;       // O in TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int qt = blockIdx.x % a.nqt;
  const int bh = blockIdx.x / a.nqt;
  const int head = bh % a.H, b = bh / a.H;
  const int nkb_all = (a.S + 127) / 128;
  const int nkb = a.causal ? min(qt + 1, nkb_all) : nkb_all;  // key blocks that matter
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
  // V tiles get their own buffers when K uses at most half of the KV region
  // (S <= 256): then V streams in concurrently with Q.K^T instead of after it.
  const int v_slot0 = nkb <= kMaxKB / 2 ? kMaxKB / 2 : 0;

  if (warp == 0) {
    if (lane == 0) {
      pdl_wait();  // q/k/v are written by the upstream QKV GEMM
      mbar_expect_tx(q_full, kTile);
      tma_load_3d(smem + Smem::Q, &tm, q_full, head * 64, qt * 128, b);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_expect_tx(&k_full[kb], kTile);
        tma_load_3d(smem + Smem::KV + kb * kTile, &tm, &k_full[kb], a.h + head * 64, kb * 128, b);
      }
      if (v_slot0 == 0) mbar_wait(s_full, 0);  // QK^T done reading K: reuse the buffers for V
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_expect_tx(&v_full[kb], kTile);
        tma_load_3d(smem + Smem::KV + (v_slot0 + kb) * kTile, &tm, &v_full[kb], 2 * a.h + head * 64,
                    kb * 128, b);
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
        const uint32_t k0 = smem_u32(smem + Smem::KV + kb * kTile);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_f16_ss(tmem + kb * 128, sw128_desc(q0 + k * 32, 0, 1024),
                      sw128_desc(k0 + k * 32, 0, 1024), idesc_s, k != 0);
      }
      umma_commit(s_full);
      // ---- O = P . V : M=128, N=64 (head dim, V is MN-major), K = keys
      constexpr uint32_t idesc_o = idesc_f16_f32(128, 64, 0, 1);
      mbar_wait(p_ready, 0);
      tc_fence_after();
      const uint32_t p0 = smem_u32(smem + Smem::P);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&v_full[kb], 0);
        tc_fence_after();
        const uint32_t v0 = smem_u32(smem + Smem::KV + (v_slot0 + kb) * kTile);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 16 keys per MMA
          const uint32_t pa = p0 + (kb * 2 + kk / 4) * kTile + (kk % 4) * 32;
          const uint32_t vb = v0 + kk * 2048;
          umma_f16_ss(tmem, sw128_desc(pa, 0, 1024), sw128_desc(vb, 128 * 128, 1024), idesc_o,
                      (kb | kk) != 0);
        }
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
    const int ncols = nkb * 128;
    const int cpg = ncols / 4;  // columns per group (multiple of 32)
    const int c_begin = grp * cpg, c_end = c_begin + cpg;
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
    // pass 1: row max of round16(acc * 0.125) with the mask applied
    float mx = NEG_INF;
    for (int c = c_begin; c < c_end; c += 32) {
      uint32_t v[32];
      tmem_ld32(lane_addr + c, v);
      tmem_wait_ld();
      if (chunk_unmasked(c)) {
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, r16(__fmul_rn(__uint_as_float(v[i]), 0.125f)));
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int j = c + i;
          float s = r16(__fmul_rn(__uint_as_float(v[i]), 0.125f));
          const bool valid = j < a.S && (!a.causal || j <= qrow);
          mx = fmaxf(mx, valid ? s : NEG_INF);
        }
      }
    }
    red_max[grp * 128 + r] = mx;
    named_bar_sync(1, kSoftmaxWarps * 32);
    mx = fmaxf(fmaxf(red_max[r], red_max[128 + r]), fmaxf(red_max[256 + r], red_max[384 + r]));
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
    // pass 3: p = round16(e / sum) -> fp16 into the swizzled P operand
    // (e * (1/sum): one correctly rounded reciprocal per row instead of a divide per element)
    const float inv = __frcp_rn(sum);
    uint8_t* prow = smem + Smem::P;
    for (int c = c_begin; c < c_end; c += 32) {
      uint32_t v[32];
      tmem_ld32(lane_addr + c, v);
      tmem_wait_ld();
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float p0 = __fmul_rn(__uint_as_float(v[2 * i]), inv);
        const float p1 = __fmul_rn(__uint_as_float(v[2 * i + 1]), inv);
        __half2 h2 = __floats2half2_rn(p0, p1);
        pk[i] = *reinterpret_cast<uint32_t*>(&h2);
      }
      // columns c..c+31 live in atom c/64, 16-byte chunks (c%64)/8 .. +3
      uint8_t* atom = prow + (c / 64) * kTile + r * 128;
      const int ch0 = (c % 64) / 8;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int ch = (ch0 + q) ^ (r & 7);
        *reinterpret_cast<uint4*>(atom + ch * 16) =
            make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    }
    fence_proxy_async_smem();  // generic-proxy P writes -> visible to the tensor core
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(p_ready);
    if (stamp) dbg[6] = clock64();

    // epilogue: O (128 x 64 fp32 in TMEM cols 0..63) -> round16 -> ctx
    mbar_wait(o_full, 0);
    tc_fence_after();
    if (stamp) dbg[7] = clock64();
    if (grp < 2) {
      uint32_t v[32];
      tmem_ld32(lane_addr + grp * 32, v);
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
