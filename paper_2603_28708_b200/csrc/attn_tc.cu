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
// Persistent CTAs (one per SM) over work units (unit_at below): a (batch, head) item
// with every 128-query tile back to back (last tile first; non-causal), or one causal
// tile.  K and V of a unit are loaded into shared memory once and Q is double-buffered: the
// next tile's Q -- and, across items, the next item's K (after the last Q.K^T) and V
// (after the last P.V) -- stream in under the current tile's softmax.
// Warp roles:
//   warp 0       TMA producer (Q ring of 2, K[4], V[4])
//   warp 1       TMEM owner + tcgen05.mma issuer: S = Q.K^T one 128-key block at a
//                time (s_full[kb] per block, so the softmax starts on block 0 while
//                later blocks multiply), then O = P.V with P read from TMEM
//   warps 2..17  softmax + epilogue: 4 warps per TMEM lane quadrant.
//     pass 1  row max of the raw accumulators (3-input FMNMX; round16(x*0.125) is
//             monotone, so the max is rounded once at the end)
//     pass 2  s = round16(acc*0.125) (FMUL2 + cvt.f16x2), e = 2^(s*log2e - max*log2e)
//             (FFMA2 + SFU), stored back over S (fp32), partial sums (FADD2)
//     pass 3  p = round16(e * (1/sum)) packed 2 x fp16 per TMEM column over the
//             already-consumed part of S -> the A operand of the P.V MMA
//   Chunks of 32 keys wholly above the causal diagonal or past the sequence end skip
//   passes 1-2 and store P = 0; only chunks crossing the diagonal test per element.
//
// TMEM columns: S block kb at [128kb, 128kb+128).  "wide" mode (>= 3 key blocks):
// column group g owns key block g and writes P_g into [128g, 128g+64); O lives in
// [64, 128).  "narrow" mode (<= 2 key blocks): group g owns 32*nkb contiguous keys,
// P goes to [256, 256 + 64*nkb), O to [384, 448).
#include <cstdlib>

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
  float* tap;  // optional [B][H][S][S] fp32 pre-mask scores acc * 0.125 (retain_scores), null = off
  int h;  // hidden = H * hd (column offset of K; V at 2h)
  __half* ctx;
  int64_t ld_ctx;
  long long* dbg;  // optional per-CTA stamps [grid][128] (clock64), null = off
  int split_tiles;  // causal: one work unit per (batch, head, query tile) instead of per (batch, head)
};

struct Smem {
  static constexpr uint32_t Q = 0;                     // 2 tiles (ring)
  static constexpr uint32_t K = Q + 2 * kTile;         // 4 tiles
  static constexpr uint32_t V = K + kMaxKB * kTile;    // 4 tiles
  static constexpr uint32_t RED = V + kMaxKB * kTile;  // float [2][4][128]
  static constexpr uint32_t BAR = RED + 2 * 4 * 128 * 4;
  static constexpr uint32_t TOTAL = BAR + 256;
};
constexpr size_t kSmemBytes = 1024 + Smem::TOTAL;

// barrier slots
enum : int {
  B_QFULL = 0,    // [2]
  B_QEMPTY = 2,   // [2]
  B_KFULL = 4,    // [4]
  B_VFULL = 8,    // [4]
  B_SFULL = 12,   // [4]
  B_KEMPTY = 16,
  B_VEMPTY = 17,
  B_PREADY = 18,  // 16 softmax warps
  B_OFULL = 19,
  B_TFREE = 20,   // 16 softmax warps: TMEM of the tile consumed
  B_COUNT = 21
};

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


__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// tile order inside an item: the causal diagonal tiles with the most key blocks first
__device__ __forceinline__ int tile_of(const AttnArgs& a, int j) { return a.nqt - 1 - j; }
__device__ __forceinline__ int nkb_of(const AttnArgs& a, int qt) {
  const int nkb_all = (a.S + 127) / 128;
  // the retain_scores tap needs every key block (the mask is applied after the tap)
  return (a.causal && a.tap == nullptr) ? min(qt + 1, nkb_all) : nkb_all;
}

// Work units.  Non-causal (every tile costs the same): a unit is a whole (batch, head)
// item, its tiles back to back so K/V are loaded once.  Causal: tile qt costs qt + 1 key
// blocks, and whole items (1 + 2 + 3 + 4 = 10 blocks at S = 512) deal unevenly onto the
// SMs (384 items on 148 SMs: 3 items = 30 blocks on the busiest SM for an average of 26),
// so a unit is one tile, units ordered by cost (all last tiles first) and dealt in a
// snake over the CTAs (max 27 blocks per SM); K/V of a unit are its key blocks only.
struct Unit {
  int b, head, qt0, ntile, kbn;  // tiles qt0, qt0 - 1, ... (ntile of them); K/V blocks [0, kbn)
};
__device__ __forceinline__ int unit_at(const AttnArgs& a, int k) {
  const int n = a.B * a.H * (a.split_tiles ? a.nqt : 1);
  const int g = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  const int u = k * g + ((k & 1) ? g - 1 - c : c);
  return u < n ? u : -1;
}
__device__ __forceinline__ Unit unit_decode(const AttnArgs& a, int u) {
  Unit x;
  int bh;
  if (a.split_tiles) {
    const int items = a.B * a.H;
    bh = u % items;
    x.qt0 = a.nqt - 1 - u / items;
    x.ntile = 1;
  } else {
    bh = u;
    x.qt0 = tile_of(a, 0);
    x.ntile = a.nqt;
  }
  x.head = bh % a.H;
  x.b = bh / a.H;
  x.kbn = nkb_of(a, x.qt0);  // the unit's first tile needs the most key blocks
  return x;
}

__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  float* red_max = reinterpret_cast<float*>(smem + Smem::RED);  // [4][128]
  float* red_sum = red_max + 4 * 128;                            // [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + B_COUNT);

  const uint32_t warp = warp_id(), lane = lane_id();
  long long* dbg = a.dbg ? a.dbg + static_cast<int64_t>(blockIdx.x) * 128 : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = clock64();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < B_COUNT; ++i)
      mbar_init(&bars[i], (i == B_PREADY || i == B_TFREE) ? kSoftmaxWarps : 1);
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

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      pdl_wait();  // q/k/v are written by the upstream QKV GEMM
      uint32_t t = 0;
      for (int it = 0, u; (u = unit_at(a, it)) >= 0; ++it) {
        const Unit x = unit_decode(a, u);
        const int head = x.head, b = x.b;
        if (it > 0) mbar_wait(&bars[B_KEMPTY], (it - 1) & 1);
        for (int kb = 0; kb < x.kbn; ++kb) {
          mbar_expect_tx(&bars[B_KFULL + kb], kTile);
          tma_load_3d(smem + Smem::K + kb * kTile, &tm, &bars[B_KFULL + kb], a.h + head * 64, kb * 128, b);
        }
        for (int j = 0; j < x.ntile; ++j, ++t) {
          const int qt = x.qt0 - j;
          const uint32_t qb = t & 1;
          mbar_wait(&bars[B_QEMPTY + qb], ((t >> 1) & 1) ^ 1);
          mbar_expect_tx(&bars[B_QFULL + qb], kTile);
          tma_load_3d(smem + Smem::Q + qb * kTile, &tm, &bars[B_QFULL + qb], head * 64, qt * 128, b);
          if (j == 0) {  // V after the first Q: it is needed only once the first P exists
            if (it > 0) mbar_wait(&bars[B_VEMPTY], (it - 1) & 1);
            for (int kb = 0; kb < x.kbn; ++kb) {
              mbar_expect_tx(&bars[B_VFULL + kb], kTile);
              tma_load_3d(smem + Smem::V + kb * kTile, &tm, &bars[B_VFULL + kb], 2 * a.h + head * 64, kb * 128, b);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_f16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc_o = idesc_f16_f32(128, 64, 0, 1);
      uint32_t t = 0, kvph = 0;  // kvph: parity bit per K/V block barrier
      for (int it = 0, u; (u = unit_at(a, it)) >= 0; ++it) {
        const Unit x = unit_decode(a, u);
        for (int j = 0; j < x.ntile; ++j, ++t) {
          const int qt = x.qt0 - j;
          const int nkb = nkb_of(a, qt);
          const bool wide = nkb > 2;
          const uint32_t o_col = wide ? 64u : 384u;
          const uint32_t qb = t & 1;
          if (t > 0) mbar_wait(&bars[B_TFREE], (t - 1) & 1);  // previous tile's TMEM consumed
          mbar_wait(&bars[B_QFULL + qb], (t >> 1) & 1);
          tc_fence_after();
          if (dbg && t < 14) dbg[8 + t * 8 + 7] = clock64();
          const uint32_t q0 = smem_u32(smem + Smem::Q + qb * kTile);
          // ---- S = Q . K^T : M=128 queries, N=128 keys per block, K = 64 (4 x 16)
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&bars[B_KFULL + kb], (kvph >> kb) & 1);
            tc_fence_after();
            const uint32_t k0 = smem_u32(smem + Smem::K + kb * kTile);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_f16_ss(tmem + kb * 128, sw128_desc(q0 + k * 32, 0, 1024),
                          sw128_desc(k0 + k * 32, 0, 1024), idesc_s, k != 0);
            umma_commit(&bars[B_SFULL + kb]);
          }
          umma_commit(&bars[B_QEMPTY + qb]);
          if (j == x.ntile - 1) umma_commit(&bars[B_KEMPTY]);
          // ---- O = P . V : M=128, N=64 (head dim, V MN-major in smem), K = keys, P in TMEM
          mbar_wait(&bars[B_PREADY], t & 1);
          tc_fence_after();
          for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&bars[B_VFULL + kb], (kvph >> kb) & 1);
            tc_fence_after();
            const uint32_t v0 = smem_u32(smem + Smem::V + kb * kTile);
            const uint32_t pcol = wide ? 128u * kb : 256u + 64u * kb;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // 16 keys per MMA = 8 packed TMEM columns of P
              umma_f16_ts(tmem + o_col, tmem + pcol + 8 * kk, sw128_desc(v0 + kk * 2048, 128 * 128, 1024),
                          idesc_o, (kb | kk) != 0);
          }
          umma_commit(&bars[B_OFULL]);
          if (j == x.ntile - 1) umma_commit(&bars[B_VEMPTY]);
        }
        kvph ^= (1u << x.kbn) - 1;  // blocks [0, kbn) completed one phase in this unit
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax + epilogue warps ----------------
    const uint32_t sw = warp - 2;
    const uint32_t quad = warp & 3;  // TMEM lane quadrant accessible to this warp
    const uint32_t grp = sw >> 2;    // column group 0..3
    const int r = quad * 32 + lane;  // row within the tile (TMEM lane)
    const uint32_t lane_addr = tmem + ((quad * 32) << 16);
    const float NEG_INF = __int_as_float(0xff800000);
    constexpr float LOG2E = 1.4426950408889634f;
    uint32_t t = 0, sph = 0;  // sph: parity bit per s_full barrier
    for (int it = 0, u; (u = unit_at(a, it)) >= 0; ++it) {
      const Unit x = unit_decode(a, u);
      const int head = x.head, b = x.b;
      for (int j = 0; j < x.ntile; ++j, ++t) {
        const int qt = x.qt0 - j;
        const int nkb = nkb_of(a, qt);
        const bool wide = nkb > 2;
        const uint32_t o_col = wide ? 64u : 384u;
        const int qrow = qt * 128 + r;
        long long* ts = (dbg && sw == 0 && lane == 0 && t < 14) ? dbg + 8 + t * 8 : nullptr;
        if (ts) ts[0] = clock64();
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
        // wait for the S blocks this group reads (every block in narrow mode: cheap)
        if (wide) {
          if (grp < static_cast<uint32_t>(nkb)) mbar_wait(&bars[B_SFULL + grp], (sph >> grp) & 1);
        } else {
          for (int kb = 0; kb < nkb; ++kb) mbar_wait(&bars[B_SFULL + kb], (sph >> kb) & 1);
        }
        sph ^= (1u << nkb) - 1;  // every block of this tile completed one phase
        tc_fence_after();
        if (ts) ts[1] = clock64();
        // chunk classes (warp-uniform: rows of this warp are qt*128 + quad*32 + [0, 32))
        const int row_lo = qt * 128 + quad * 32, row_hi = row_lo + 31;
        auto chunk_full = [&](int c) { return c + 32 <= a.S && (!a.causal || c + 31 <= row_lo); };
        auto chunk_dead = [&](int c) { return c >= a.S || (a.causal && c > row_hi); };
        // pass 1: max of the raw accumulators over the unmasked keys
        float m0 = NEG_INF, m1 = NEG_INF;
        for (int c = c_begin; c < c_end; c += 32) {
          if (chunk_dead(c) && a.tap == nullptr) continue;
          uint32_t v[32];
          tmem_ld32(lane_addr + c, v);
          tmem_wait_ld();
          if (a.tap != nullptr && qrow < a.S) {  // retain_scores: fp32 acc * scale, pre-mask
            float* trow = a.tap + ((static_cast<int64_t>(b) * a.H + head) * a.S + qrow) * a.S;
            for (int i = 0; i < 32; ++i)
              if (c + i < a.S) trow[c + i] = __fmul_rn(__uint_as_float(v[i]), 0.125f);
          }
          if (chunk_dead(c)) continue;
          if (chunk_full(c)) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              m0 = fmax3(m0, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
              m1 = fmax3(m1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int jj = c + i;
              const bool valid = jj < a.S && (!a.causal || jj <= qrow);
              m0 = fmaxf(m0, valid ? __uint_as_float(v[i]) : NEG_INF);
            }
          }
        }
        red_max[grp * 128 + r] = fmaxf(m0, m1);
        named_bar_sync(1, kSoftmaxWarps * 32);
        const float mraw = fmaxf(fmaxf(red_max[r], red_max[128 + r]), fmaxf(red_max[256 + r], red_max[384 + r]));
        const float mx = r16(__fmul_rn(mraw, 0.125f));  // == max_j round16(acc_j * 0.125)
        if (ts) ts[2] = clock64();
        // pass 2: e = exp(s - max) kept in TMEM (fp32), partial sums in key order.
        // exp(s - mx) = 2^(s*log2e - mx*log2e): one FFMA + one SFU op per element.
        const float mxl = __fmul_rn(mx, LOG2E);
        const uint64_t k8 = f2_pack(0.125f, 0.125f), kl = f2_pack(LOG2E, LOG2E), nm = f2_pack(-mxl, -mxl);
        uint64_t sum2 = f2_pack(0.0f, 0.0f);
        for (int c = c_begin; c < c_end; c += 32) {
          if (chunk_dead(c)) continue;
          uint32_t v[32];
          tmem_ld32(lane_addr + c, v);
          tmem_wait_ld();
          const bool full = chunk_full(c);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float s0, s1;
            const uint64_t sc = f2_mul(f2_pack(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), k8);
            f2_unpack(sc, s0, s1);
            h2_unpack(h2_pack_rn(s0, s1), s0, s1);  // s = round16(acc * 0.125)
            const uint64_t x = f2_fma(f2_pack(s0, s1), kl, nm);
            float x0, x1;
            f2_unpack(x, x0, x1);
            float e0 = ex2_approx(x0), e1 = ex2_approx(x1);
            if (!full) {
              const int jj = c + i;
              e0 = (jj < a.S && (!a.causal || jj <= qrow)) ? e0 : 0.0f;
              e1 = (jj + 1 < a.S && (!a.causal || jj + 1 <= qrow)) ? e1 : 0.0f;
            }
            const uint64_t e2 = f2_pack(e0, e1);
            sum2 = f2_add(sum2, e2);
            v[i] = __float_as_uint(e0);
            v[i + 1] = __float_as_uint(e1);
          }
          tmem_st32(lane_addr + c, v);
        }
        tmem_wait_st();
        float sa, sb;
        f2_unpack(sum2, sa, sb);
        red_sum[grp * 128 + r] = __fadd_rn(sa, sb);
        named_bar_sync(1, kSoftmaxWarps * 32);
        const float sum = __fadd_rn(__fadd_rn(__fadd_rn(red_sum[r], red_sum[128 + r]), red_sum[256 + r]),
                                    red_sum[384 + r]);
        // pass 3: p = round16(e * (1/sum)), packed fp16 pairs into TMEM (the P.V A operand)
        if (ts) ts[3] = clock64();
        const float inv = __frcp_rn(sum);
        const uint64_t inv2 = f2_pack(inv, inv);
        for (int c = c_begin; c < c_end; c += 32) {
          const uint32_t pcol = wide ? static_cast<uint32_t>((c / 128) * 128 + (c % 128) / 2)
                                     : 256u + static_cast<uint32_t>(c / 2);
          uint32_t pk[16];
          if (chunk_dead(c)) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          } else {
            uint32_t v[32];
            tmem_ld32(lane_addr + c, v);
            tmem_wait_ld();  // the whole chunk is in registers before P overwrites S columns
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float p0, p1;
              f2_unpack(f2_mul(f2_pack(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), inv2), p0, p1);
              pk[i] = h2_pack_rn(p0, p1);
            }
          }
          tmem_st16(lane_addr + pcol, pk);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_PREADY]);
        if (ts) ts[4] = clock64();

        // epilogue: O (128 x 64 fp32 in TMEM) -> round16 -> ctx
        mbar_wait(&bars[B_OFULL], t & 1);
        tc_fence_after();
        if (ts) ts[5] = clock64();
        if (grp < 2) {
          uint32_t v[32];
          tmem_ld32(lane_addr + o_col + grp * 32, v);
          tmem_wait_ld();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[B_TFREE]);  // O is in registers: TMEM free
          if (ts) ts[6] = clock64();
          if (qrow < a.S) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = h2_pack_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
            uint4* dst = reinterpret_cast<uint4*>(a.ctx + (static_cast<int64_t>(b) * a.S + qrow) * a.ld_ctx +
                                                  head * 64 + grp * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[B_TFREE]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (dbg && threadIdx.x == 0) dbg[1] = clock64();
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
  if (attn_fa_enabled()) p.fa_sched = attn_fa_schedule(B, S, H, causal);
  return p;
}

void configure_attn_tc() {
  static std::mutex mu;
  static uint64_t done = 0;
  once_per_device(mu, done, [] {
    PRLAB_CUDA(cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemBytes)));
  });
}

void launch_attn_tc(const AttnPlan& p, cudaStream_t st, float* tap) {
  // The streaming kernel wins once a sequence spans several key blocks or the (b, h)
  // items fill the SMs; with S <= 128 and fewer items than SMs (one 128-key tile each) the
  // resident-row kernel's 16 softmax warps per tile finish first (C3 sweep A/B,
  // profiles/r01/ab_attn_c3_sweep.txt: B=8 S=32 0.557 vs 0.590 ms, B=16 S=32 0.698 vs 0.653).
  const int nqt = (p.S + 127) / 128;
  if (p.unstab && tap != nullptr) throw std::invalid_argument("unstabilised softmax has no score tap");
  if (p.unstab || (tap == nullptr && attn_fa_enabled() && (nqt > 1 || p.B * p.H > num_sms()))) {
    launch_attn_fa(p, st);
    return;
  }
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
  a.tap = tap;
  static const bool split_env = [] {  // PRLAB_ATTN_SPLIT=0: whole (batch, head) units (A/B)
    const char* e = std::getenv("PRLAB_ATTN_SPLIT");
    return e == nullptr || std::atoi(e) != 0;
  }();
  a.split_tiles = (split_env && p.causal && tap == nullptr && a.nqt > 1) ? 1 : 0;
  const int grid = std::min(p.B * p.H * (a.split_tiles ? a.nqt : 1), num_sms());
  launch_pdl(attn_tc_kernel, dim3(grid), dim3(kThreads), kSmemBytes, st, p.tmQKV, a);
}

}  // namespace prlab_gpu
