// Fused hybrid attention on tcgen05 tensor cores.
//
// Reference semantics (hybrid policy; src/model.cpp:393-427, kernels.cpp:85-168):
//   s_ij = round16( fp32dot(q_i, k_j) * 0.125 )          AttentionScoreMatmul {F16E, F32}
//   s_ij = -inf for j > i                                 decoder causal mask (after scaling)
//   p_ij = e_ij / sum_j e_ij,  e_ij = exp(s_ij - max_j)   Softmax {F32, F32, stabilized}
//   o_i  = round16( fp32dot(round16(p_i), v) )            AttentionScoreMatmul {F16E, F32}
// The whole score row is resident (S <= 512 -> 128 x 512 fp32 = all of TMEM), so
// the softmax is the reference's exact two-pass form (max, then exp/sum, then
// normalise-then-round), not an online rescaling; e is computed once and kept.
//
// Persistent CTAs (one per SM): CTA c owns the (batch, head) items c, c + grid, ...
// and runs every 128-query tile of an item back to back (last tile first), so K and
// V of the item are loaded into shared memory once; Q is double-buffered so the next
// tile's Q (and the next item's K / V) stream in under the current softmax.
// Warp roles (576 threads):
//   warp 0       TMA producer (Q ring of 2, K[4], V[4])
//   warp 1       TMEM owner + tcgen05.mma issuer: S = Q.K^T one 128-key block at a
//                time (s_full[kb]), then O = P.V one block at a time as soon as that
//                block's P exists (p_full[kb]), P read straight from TMEM
//   warps 2..17  softmax + epilogue.  Warp (quad q = warp & 3, group g) owns rows
//                32q..32q+31 (its TMEM lane quadrant) and keys 32g..32g+31 of every
//                128-key block, so all 16 warps work on every block in block order
//                for any causal block count:
//     pass 1  per block as its S lands: row max of the raw accumulators (FMNMX3;
//             round16(x*0.125) is monotone, so the max is rounded once at the end)
//     pass 2  e = 2^(s*log2e - max*log2e), s = round16(acc*0.125) (FMUL2, cvt.f16x2,
//             FFMA2, SFU), stored back over S (fp32), row sums (FADD2); the next
//             block's TMEM load is in flight while a block computes
//     pass 3  per block: p = round16(e * (1/sum)) packed 2 x fp16 per column into the
//             first half of the block's columns (after the 4 warps of the quadrant
//             have read the block), then p_full[kb]: the block's P.V MMAs overlap
//             the next block's pass 3
//   Key chunks wholly above the causal diagonal or past the sequence end skip the
//   arithmetic (P = 0); only chunks crossing them mask per element.
// TMEM columns: S / e block kb at [128kb, 128kb+128); P_kb packed in [128kb, 128kb+64);
// O (128 x 64 fp32) in [64, 128) once P_0 is written.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

constexpr int kSoftmaxWarps = 16;
constexpr int kThreads = 64 + kSoftmaxWarps * 32;  // 576
constexpr int kMaxKB = 4;                          // S <= 512
constexpr uint32_t kTile = 128 * 64 * 2;           // one 128 x 64 fp16 tile, 16 KB
// kPolyPairs (template): pairs (of the 8 per 16-key unit) whose exponentials run on
// the FMA pipe instead of the SFU -- balances the 16/clk/SM SFU against issue slots.
constexpr uint32_t kPolyDefault = 0x22;

struct AttnArgs {
  int B, S, H, hd, causal, nqt;
  int h;  // hidden = H * hd (column offset of K; V at 2h)
  __half* ctx;
  int64_t ld_ctx;
  long long* dbg;  // optional per-CTA stamps [grid][256] (clock64), null = off
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
  B_SFULL = 12,   // [4] S block kb in TMEM
  B_PFULL = 16,   // [4] P block kb in TMEM (16 softmax warps)
  B_PVDONE = 20,  // [4] the P.V MMAs of block kb completed (TMEM block reusable)
  B_KEMPTY = 24,
  B_VEMPTY = 25,
  B_OFULL = 26,
  B_OFREE = 27,   // 16 softmax warps: O of the tile read into registers
  B_COUNT = 28
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

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
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
  return a.causal ? min(qt + 1, nkb_all) : nkb_all;
}

template <uint32_t kPolyPairs>
__global__ void __launch_bounds__(kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  float* red_max = reinterpret_cast<float*>(smem + Smem::RED);  // [4][128]
  float* red_sum = red_max + 4 * 128;                            // [4][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + B_COUNT);

  const int items = a.B * a.H;
  const int nkb_all = (a.S + 127) / 128;
  const uint32_t warp = warp_id(), lane = lane_id();
  long long* dbg = a.dbg ? a.dbg + static_cast<int64_t>(blockIdx.x) * 256 : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = clock64();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < B_COUNT; ++i)
      mbar_init(&bars[i], ((i >= B_PFULL && i < B_PFULL + 4) || i == B_OFREE) ? kSoftmaxWarps : 1);
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
      uint32_t t = 0, it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int head = item % a.H, b = item / a.H;
        if (it > 0) mbar_wait(&bars[B_KEMPTY], (it - 1) & 1);
        for (int kb = 0; kb < nkb_all; ++kb) {
          mbar_expect_tx(&bars[B_KFULL + kb], kTile);
          tma_load_3d(smem + Smem::K + kb * kTile, &tm, &bars[B_KFULL + kb], a.h + head * 64, kb * 128, b);
        }
        for (int j = 0; j < a.nqt; ++j, ++t) {
          const int qt = tile_of(a, j);
          const uint32_t qb = t & 1;
          mbar_wait(&bars[B_QEMPTY + qb], ((t >> 1) & 1) ^ 1);
          mbar_expect_tx(&bars[B_QFULL + qb], kTile);
          tma_load_3d(smem + Smem::Q + qb * kTile, &tm, &bars[B_QFULL + qb], head * 64, qt * 128, b);
          if (j == 0) {  // V after the first Q: it is needed only once the first P exists
            if (it > 0) mbar_wait(&bars[B_VEMPTY], (it - 1) & 1);
            for (int kb = 0; kb < nkb_all; ++kb) {
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
      // parity bits per barrier of a block ring: p_full[kb] and pv_done[kb]
      uint32_t pph = 0, dph = 0, t = 0, it = 0;
      int nkb_prev = 0;  // previous tile: its P blocks and (in its last block) its O
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        for (int j = 0; j < a.nqt; ++j, ++t) {
          const int nkb = nkb_of(a, tile_of(a, j));
          const int L = nkb - 1;  // O of this tile lives in the upper half of block L
          const uint32_t qb = t & 1;
          mbar_wait(&bars[B_QFULL + qb], (t >> 1) & 1);
          tc_fence_after();
          const uint32_t q0 = smem_u32(smem + Smem::Q + qb * kTile);
          // ---- S = Q . K^T : M=128 queries, N=128 keys per block, K = 64 (4 x 16).
          // Block kb's columns are reusable once the previous tile's P.V of that block
          // finished and, for the block that held its O, once O was read.
          long long* ms = (dbg && t < 14) ? dbg + 8 + 14 * 8 + t * 4 : nullptr;  // MMA-thread stamps
          if (ms) ms[0] = clock64();
          for (int kb = 0; kb < nkb; ++kb) {
            if (kb < nkb_prev) {
              mbar_wait(&bars[B_PVDONE + kb], (dph >> kb) & 1);
              dph ^= 1u << kb;
              if (kb == nkb_prev - 1) mbar_wait(&bars[B_OFREE], (t - 1) & 1);
            }
            mbar_wait(&bars[B_KFULL + kb], it & 1);
            tc_fence_after();
            const uint32_t k0 = smem_u32(smem + Smem::K + kb * kTile);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_f16_ss(tmem + kb * 128, sw128_desc(q0 + k * 32, 0, 1024),
                          sw128_desc(k0 + k * 32, 0, 1024), idesc_s, k != 0);
            umma_commit(&bars[B_SFULL + kb]);
          }
          // blocks the previous tile used but this one does not: retire their pv_done phase
          for (int kb = nkb; kb < nkb_prev; ++kb) {
            mbar_wait(&bars[B_PVDONE + kb], (dph >> kb) & 1);
            dph ^= 1u << kb;
          }
          if (ms) ms[1] = clock64();
          umma_commit(&bars[B_QEMPTY + qb]);
          if (j == a.nqt - 1) umma_commit(&bars[B_KEMPTY]);
          // ---- O = P . V block by block (last block first: its upper half then holds O),
          // M=128, N=64 (V MN-major in smem), P in TMEM
          const uint32_t o_col = 128u * L + 64u;
          for (int q = 0; q < nkb; ++q) {
            const int kb = q == 0 ? L : q - 1;
            mbar_wait(&bars[B_PFULL + kb], (pph >> kb) & 1);
            mbar_wait(&bars[B_VFULL + kb], it & 1);
            tc_fence_after();
            const uint32_t v0 = smem_u32(smem + Smem::V + kb * kTile);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)  // 16 keys per MMA = 8 packed TMEM columns of P
              umma_f16_ts(tmem + o_col, tmem + kb * 128 + 8 * kk, sw128_desc(v0 + kk * 2048, 128 * 128, 1024),
                          idesc_o, (q | kk) != 0);
            umma_commit(&bars[B_PVDONE + kb]);
            if (ms && q == 0) ms[2] = clock64();
            if (dbg && t == 1) dbg[224 + q] = clock64();
          }
          if (ms) ms[3] = clock64();
          pph ^= (1u << nkb) - 1;
          umma_commit(&bars[B_OFULL]);
          if (j == a.nqt - 1) umma_commit(&bars[B_VEMPTY]);
          nkb_prev = nkb;
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax + epilogue warps ----------------
    const uint32_t quad = warp & 3;        // TMEM lane quadrant accessible to this warp
    const uint32_t grp = (warp - 2) >> 2;  // 32-key chunk of every block
    const int r = quad * 32 + lane;        // row within the tile (TMEM lane)
    const uint32_t lane_addr = tmem + ((quad * 32) << 16);
    const float NEG_INF = __int_as_float(0xff800000);
    constexpr float LOG2E = 1.4426950408889634f;
    const uint64_t k8 = f2_pack(0.125f, 0.125f), kl = f2_pack(LOG2E, LOG2E);
    uint32_t t = 0, sph = 0;  // sph: parity bit per s_full barrier
    // the previous tile's epilogue runs inside this tile's pass 1 (its O sits in the
    // upper half of its last block; the next tile overwrites that block only if it
    // has more blocks, and then the epilogue goes right before that block's wait)
    int pv_b = -1, pv_head = 0, pv_qt = 0, pv_L = 0;
    auto epilogue = [&](uint32_t tt) {
      mbar_wait(&bars[B_OFULL], tt & 1);
      tc_fence_after();
      if (grp < 2) {
        uint32_t v[32];
        tmem_ld32(lane_addr + 128u * pv_L + 64u + grp * 32, v);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_OFREE]);  // O is in registers
        const int erow = pv_qt * 128 + r;
        if (erow < a.S) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = h2_pack_rn(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
          uint4* dst = reinterpret_cast<uint4*>(a.ctx + (static_cast<int64_t>(pv_b) * a.S + erow) * a.ld_ctx +
                                                pv_head * 64 + grp * 32);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[B_OFREE]);
      }
      pv_b = -1;
    };
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int head = item % a.H, b = item / a.H;
      for (int j = 0; j < a.nqt; ++j, ++t) {
        const int qt = tile_of(a, j);
        const int nkb = nkb_of(a, qt);
        const int qrow = qt * 128 + r;
        const int row_lo = qt * 128 + quad * 32, row_hi = row_lo + 31;  // this warp's rows
        long long* ts = (dbg && warp == 2 && lane == 0 && t < 14) ? dbg + 8 + t * 8 : nullptr;
        if (ts) ts[0] = clock64();
        auto cbase = [&](int kb) { return kb * 128 + static_cast<int>(grp) * 32; };  // first key of chunk
        auto dead = [&](int kb) { const int c0 = cbase(kb); return c0 >= a.S || (a.causal && c0 > row_hi); };
        auto full = [&](int kb) { const int c0 = cbase(kb); return c0 + 32 <= a.S && (!a.causal || c0 + 31 <= row_lo); };
        auto valid = [&](int jj) { return jj < a.S && (!a.causal || jj <= qrow); };
        const uint32_t col = grp * 32;  // this warp's columns inside a block
        // ---- pass 1: max of the raw accumulators, block by block as S lands
        float m0 = NEG_INF, m1 = NEG_INF;
        for (int kb = 0; kb < nkb; ++kb) {
          if (pv_b >= 0 && kb == pv_L) epilogue(t - 1);  // this block still holds the previous O
          mbar_wait(&bars[B_SFULL + kb], (sph >> kb) & 1);
          tc_fence_after();
          if (dead(kb)) continue;
          uint32_t v[32];
          tmem_ld32(lane_addr + kb * 128 + col, v);
          tmem_wait_ld();
          if (full(kb)) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              m0 = fmax3(m0, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
              m1 = fmax3(m1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            }
          } else {
            const int c0 = cbase(kb);
#pragma unroll
            for (int i = 0; i < 32; ++i) m0 = fmaxf(m0, valid(c0 + i) ? __uint_as_float(v[i]) : NEG_INF);
          }
        }
        sph ^= (1u << nkb) - 1;
        red_max[grp * 128 + r] = fmaxf(m0, m1);
        if (pv_b >= 0) epilogue(t - 1);
        if (ts) ts[1] = clock64();
        named_bar_sync(1, kSoftmaxWarps * 32);
        const float mraw = fmaxf(fmaxf(red_max[r], red_max[128 + r]), fmaxf(red_max[256 + r], red_max[384 + r]));
        const float mx = r16(__fmul_rn(mraw, 0.125f));  // == max_j round16(acc_j * 0.125)
        const uint64_t nm = f2_pack(-__fmul_rn(mx, LOG2E), -__fmul_rn(mx, LOG2E));
        // ---- pass 2: e = exp(s - max) kept in TMEM (fp32), row sums; next block's load in flight
        uint64_t sum2 = f2_pack(0.0f, 0.0f);
        {
          // units u = 2*kb + half (16 columns each); ping-pong buffers, the load of
          // unit u+1 is in flight while unit u computes
          uint32_t va[16], vb[16];
          auto live = [&](int u) { return (u >> 1) < nkb && !dead(u >> 1); };
          auto ld_unit = [&](int u, uint32_t (&buf)[16]) {
            tmem_ld16(lane_addr + (u >> 1) * 128 + col + (u & 1) * 16, buf);
          };
          auto compute = [&](int u, uint32_t (&v)[16]) {
            const int kb = u >> 1;
            const int c0 = cbase(kb) + (u & 1) * 16;
            float e[16];
            if (full(kb)) {  // hot path: no masks
#pragma unroll
              for (int i = 0; i < 16; i += 2) {
                float s0, s1;
                f2_unpack(f2_mul(f2_pack(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), k8), s0, s1);
                h2_unpack(h2_pack_rn(s0, s1), s0, s1);  // s = round16(acc * 0.125)
                float x0, x1;
                f2_unpack(f2_fma(f2_pack(s0, s1), kl, nm), x0, x1);
                if ((kPolyPairs >> (i / 2)) & 1) {  // this pair's exponentials on the FMA pipe
                  f2_unpack(exp2_pair_poly(x0, x1), e[i], e[i + 1]);
                } else {
                  e[i] = ex2_approx(x0);
                  e[i + 1] = ex2_approx(x1);
                }
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; i += 2) {
                float s0, s1;
                f2_unpack(f2_mul(f2_pack(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), k8), s0, s1);
                h2_unpack(h2_pack_rn(s0, s1), s0, s1);
                float x0, x1;
                f2_unpack(f2_fma(f2_pack(s0, s1), kl, nm), x0, x1);
                e[i] = valid(c0 + i) ? ex2_approx(x0) : 0.0f;
                e[i + 1] = valid(c0 + i + 1) ? ex2_approx(x1) : 0.0f;
              }
            }
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              sum2 = f2_add(sum2, f2_pack(e[i], e[i + 1]));
              v[i] = __float_as_uint(e[i]);
              v[i + 1] = __float_as_uint(e[i + 1]);
            }
            tmem_st16(lane_addr + kb * 128 + col + (u & 1) * 16, v);
          };
          if (live(0)) {
            ld_unit(0, va);
            tmem_wait_ld();
          }
#pragma unroll
          for (int u = 0; u < 2 * kMaxKB; ++u) {
            uint32_t(&cur)[16] = (u & 1) ? vb : va;
            uint32_t(&nxt)[16] = (u & 1) ? va : vb;
            const bool ln = u + 1 < 2 * kMaxKB && live(u + 1);
            if (ln) ld_unit(u + 1, nxt);
            if (live(u)) compute(u, cur);
            if (ln) tmem_wait_ld();
          }
        }
        tmem_wait_st();
        float sa, sb;
        f2_unpack(sum2, sa, sb);
        red_sum[grp * 128 + r] = __fadd_rn(sa, sb);
        if (ts) ts[2] = clock64();
        named_bar_sync(1, kSoftmaxWarps * 32);
        const float sum = __fadd_rn(__fadd_rn(__fadd_rn(red_sum[r], red_sum[128 + r]), red_sum[256 + r]),
                                    red_sum[384 + r]);
        if (ts) ts[3] = clock64();
        // ---- pass 3: p = round16(e * (1/sum)) -> first half of the block's columns
        const float inv = __frcp_rn(sum);
        const uint64_t inv2 = f2_pack(inv, inv);
        for (int q = 0; q < nkb; ++q) {
          const int kb = q == 0 ? nkb - 1 : q - 1;  // last block first: it will hold O
          uint32_t pk[16];
          if (dead(kb)) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          } else {
            uint32_t v[32];
            tmem_ld32(lane_addr + kb * 128 + col, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float p0, p1;
              f2_unpack(f2_mul(f2_pack(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])), inv2), p0, p1);
              pk[i] = h2_pack_rn(p0, p1);
            }
          }
          // the quadrant's 4 warps have read block kb before its P overwrites e columns
          named_bar_sync(2 + quad, 128);
          tmem_st16(lane_addr + kb * 128 + grp * 16, pk);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars[B_PFULL + kb]);
        }
        if (ts) ts[4] = clock64();
        if (dbg && t == 1 && lane == 0) dbg[200 + (warp - 2)] = clock64();  // pass-3 end per warp
        pv_b = b;
        pv_head = head;
        pv_qt = qt;
        pv_L = nkb - 1;
        if (ts) ts[5] = ts[6] = clock64();
      }
    }
    if (pv_b >= 0) epilogue(t - 1);
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
  return p;
}

void configure_attn_tc() {
  static bool done = false;
  if (done) return;
  for (auto k : {attn_tc_kernel<kPolyDefault>, attn_tc_kernel<0u>, attn_tc_kernel<0x55u>})
    PRLAB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes)));
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
  const int grid = std::min(p.B * p.H, num_sms());
  // tuning knob: PRLAB_ATTN_POLY=0 (all exponentials on the SFU) / 0x55 (half on the FMA pipe)
  static const int poly = std::getenv("PRLAB_ATTN_POLY") ? std::atoi(std::getenv("PRLAB_ATTN_POLY")) : -1;
  if (poly == 0)
    launch_pdl(attn_tc_kernel<0u>, dim3(grid), dim3(kThreads), kSmemBytes, st, p.tmQKV, a);
  else if (poly == 0x55)
    launch_pdl(attn_tc_kernel<0x55u>, dim3(grid), dim3(kThreads), kSmemBytes, st, p.tmQKV, a);
  else
    launch_pdl(attn_tc_kernel<kPolyDefault>, dim3(grid), dim3(kThreads), kSmemBytes, st, p.tmQKV, a);
}

}  // namespace prlab_gpu
