// Hybrid attention, key-block streaming form (two CTAs per SM).
//
// Same scores and masking as attn_tc.cu (src/model.cpp:393-427, kernels.cpp:85-168):
//   s_ij = round16(fp32dot(q_i, k_j) * 0.125), -inf above the causal diagonal,
// but the softmax is computed online over 128-key blocks instead of over the resident
// row: per row a running max m and sum l,
//   e_ij = exp(s_ij - m),  P~_ij = round16(e_ij)  (fp16 A operand of P.V),
//   O = O * exp(m_old - m) + P~ . V,   o_i = round16(O_i / l_i),
// where m follows the running max lazily (moved only when it grew by > 5).
// The reference normalises before rounding p (round16(e / sum), kernels.cpp:154-165);
// here the fp16 rounding falls on e and the division on O -- the same number of
// roundings of the same relative size (2^-11), in a different place.  Hybrid parity is
// a cosine budget; tests/test_gpu_kernels.py holds both kernels to the
// same bound against the fp32 restatement, and attn_tc.cu (exact two-pass form) remains
// the kernel for the retain_scores tap and for PRLAB_ATTN_FA=0.
//
// Why: attn_tc.cu keeps a whole 128 x S score tile in TMEM (all 512 columns at S = 512),
// so one CTA per SM alternates strictly between tensor-core and softmax phases.  Here a
// CTA needs 192 TMEM columns (S block 128 fp32, O 64 fp32; P packed over consumed S
// columns) and ~97 KB of shared memory, so two CTAs share an SM and one's softmax runs
// under the other's MMAs.
//
// Per CTA: warp 0 TMA (Q ring 2, K ring 2, V ring 2), warp 1 tcgen05 issuer, warps 2..5
// one query row per thread (TMEM lane = row).  Work units are (batch, head, 128-query
// tile); causal units are ordered by key-block count and dealt in a snake over the CTAs.
#include <cstdlib>

#include <algorithm>
#include <map>
#include <queue>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

constexpr int kSoftmaxWarps = 8;  // 2 per TMEM lane quadrant, each half of the 128 key columns
constexpr int kThreads = 64 + 32 * kSoftmaxWarps;
constexpr uint32_t kTile = 128 * 64 * 2;  // Q tile / one K or V block of 128 keys, 16 KB
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kColS = 0;    // S block [0, 128)
constexpr uint32_t kColO = 128;  // O [128, 192)
constexpr uint32_t kColP = 192;  // P~ packed fp16 [192, 256): S of the next block can land while P.V reads P

struct FaSmem {
  static constexpr uint32_t Q = 0;               // 2 tiles
  static constexpr uint32_t K = Q + 2 * kTile;   // 2 blocks
  static constexpr uint32_t V = K + 2 * kTile;   // 2 blocks
  // float [3][2][128]: partial row max per half (double-buffered by block parity: a fast
  // warp may write the next block's before a slow one read this one's), partial row sums
  static constexpr uint32_t RED = V + 2 * kTile;
  static constexpr uint32_t BAR = RED + 6 * 256 * 4;  // row kernel TPR 4: rmax 2 x 4 x 128, rsum 4 x 128
  static constexpr uint32_t TOTAL = BAR + 512;
};
constexpr size_t kFaSmemBytes = 1024 + FaSmem::TOTAL;

enum : int {
  F_QFULL = 0,   // [2]
  F_QEMPTY = 2,  // [2]
  F_KFULL = 4,   // [2]
  F_KEMPTY = 6,  // [2]
  F_VFULL = 8,   // [2]
  F_VEMPTY = 10, // [2]
  F_SFULL = 12,  // S block in TMEM
  F_PREADY = 13, // softmax warps: S read, P in TMEM, O rescaled
  F_OFULL = 14,  // last P.V of the unit done
  F_TFREE = 15,  // softmax warps: O read by the epilogue
  F_PVDONE = 16, // P.V of a block done: P columns and O free for the next block's softmax
  F_COUNT = 17
};

struct FaArgs {
  int* work;         // dynamic unit counter [2] (next unit, CTAs done; zero between launches) or null
  const int* sched;  // balanced static schedule ([grid + 1] offsets, then unit ids; attn_fa_schedule) or null
  int B, S, H, causal, nqt, h;
  int unstab;  // full_fp16 fast path: unstabilised softmax (no max shift, kernels.cpp:155)
  __half* ctx;
  int64_t ld_ctx;
  long long* dbg;  // optional clock64 stamps of CTA 0, [block][8] (scripts/fa_phases.py), null = off
};

__device__ __forceinline__ void umma_f16_ts_fa(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// MMA-thread wait without the try_wait suspend: the issuer wakes as soon as the softmax
// arrives (it is one thread; its polling costs one issue slot per iteration)
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
  const long long t0 = clock64();
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (!ok && clock64() - t0 > (1ll << 31)) {
      printf("prlab_gpu watchdog: mbarrier spin timeout block %d thread %d\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}

__device__ __forceinline__ float fmax3_fa(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// unit u -> (b, head, qt); causal: all last tiles first (most key blocks), snake over CTAs
__device__ __forceinline__ int fa_unit_at(const FaArgs& a, int k) {
  if (a.sched != nullptr) {
    const int o0 = __ldg(a.sched + blockIdx.x), o1 = __ldg(a.sched + blockIdx.x + 1);
    return o0 + k < o1 ? __ldg(a.sched + gridDim.x + 1 + o0 + k) : -1;
  }
  const int n = a.B * a.H * a.nqt;
  const int g = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  const int u = k * g + ((k & 1) ? g - 1 - c : c);
  return u < n ? u : -1;
}
__device__ __forceinline__ void fa_decode(const FaArgs& a, int u, int& b, int& head, int& qt, int& nkb) {
  const int items = a.B * a.H;
  const int bh = u % items;
  qt = a.nqt - 1 - u / items;
  head = bh % a.H;
  b = bh / a.H;
  const int nkb_all = (a.S + 127) / 128;
  nkb = a.causal ? min(qt + 1, nkb_all) : nkb_all;
}

__global__ void __launch_bounds__(kThreads, 2) attn_fa_kernel(const __grid_constant__ CUtensorMap tm, const FaArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FaSmem::BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + F_COUNT);
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < F_COUNT; ++i) mbar_init(&bars[i], (i == F_PREADY || i == F_TFREE) ? kSoftmaxWarps : 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer: per unit Q, then K/V blocks in consumption order
    if (lane == 0) {
      pdl_wait();  // q/k/v are written by the upstream QKV GEMM
      uint32_t qc = 0, kc = 0;
      for (int it = 0, u; (u = fa_unit_at(a, it)) >= 0; ++it, ++qc) {
        int b, head, qt, nkb;
        fa_decode(a, u, b, head, qt, nkb);
        const uint32_t qs = qc & 1;
        mbar_wait(&bars[F_QEMPTY + qs], ((qc >> 1) & 1) ^ 1);
        mbar_expect_tx(&bars[F_QFULL + qs], kTile);
        tma_load_3d(smem + FaSmem::Q + qs * kTile, &tm, &bars[F_QFULL + qs], head * 64, qt * 128, b);
        for (int kb = 0; kb < nkb; ++kb, ++kc) {
          const uint32_t s = kc & 1, ph = ((kc >> 1) & 1) ^ 1;
          mbar_wait(&bars[F_KEMPTY + s], ph);
          mbar_expect_tx(&bars[F_KFULL + s], kTile);
          tma_load_3d(smem + FaSmem::K + s * kTile, &tm, &bars[F_KFULL + s], a.h + head * 64, kb * 128, b);
          mbar_wait(&bars[F_VEMPTY + s], ph);
          mbar_expect_tx(&bars[F_VFULL + s], kTile);
          tma_load_3d(smem + FaSmem::V + s * kTile, &tm, &bars[F_VFULL + s], 2 * a.h + head * 64, kb * 128, b);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer.  Per block, once the softmax released S_kb (PREADY):
    // S_kb+1 first, then P.V_kb -- the next block's pass 1 (block max) runs while P.V_kb
    // executes; the softmax waits PVDONE before it rewrites P or rescales O.
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_f16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc_o = idesc_f16_f32(128, 64, 0, 1);
      uint32_t qc = 0, kc = 0, bc = 0;  // units, K/V blocks, blocks (single-slot barriers)
      auto issue_s = [&](uint32_t q0, uint32_t kcount, bool last_of_unit, uint32_t qs) {
        const uint32_t s = kcount & 1;
        mbar_wait(&bars[F_KFULL + s], (kcount >> 1) & 1);
        tc_fence_after();
        const uint32_t k0 = smem_u32(smem + FaSmem::K + s * kTile);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_f16_ss(tmem + kColS, sw128_desc(q0 + k * 32, 0, 1024), sw128_desc(k0 + k * 32, 0, 1024), idesc_s,
                      k != 0);
        umma_commit(&bars[F_SFULL]);
        umma_commit(&bars[F_KEMPTY + s]);
        if (last_of_unit) umma_commit(&bars[F_QEMPTY + qs]);
      };
      for (int it = 0, u; (u = fa_unit_at(a, it)) >= 0; ++it, ++qc) {
        int b, head, qt, nkb;
        fa_decode(a, u, b, head, qt, nkb);
        const uint32_t qs = qc & 1;
        mbar_wait(&bars[F_QFULL + qs], (qc >> 1) & 1);
        const uint32_t q0 = smem_u32(smem + FaSmem::Q + qs * kTile);
        // S of the unit's first block: the S columns are free once the softmax of the
        // previous block (previous unit) signalled PREADY
        if (bc > 0) mbar_wait(&bars[F_PREADY], (bc - 1) & 1);
        issue_s(q0, kc, nkb == 1, qs);
        for (int kb = 0; kb < nkb; ++kb, ++kc, ++bc) {
          const uint32_t s = kc & 1, ph = (kc >> 1) & 1;
          // O (+)= P~ . V once the softmax packed P and rescaled O; the unit's first P.V
          // overwrites O, so the previous unit's epilogue must have read it
          mbar_wait_spin(&bars[F_PREADY], bc & 1);
          long long* ms = (a.dbg && blockIdx.x == 0 && bc < 32) ? a.dbg + bc * 8 : nullptr;
          if (ms) ms[4] = clock64();
          if (kb + 1 < nkb) issue_s(q0, kc + 1, kb + 2 == nkb, qs);
          if (kb == 0 && qc > 0) mbar_wait(&bars[F_TFREE], (qc - 1) & 1);
          mbar_wait(&bars[F_VFULL + s], ph);
          tc_fence_after();
          const uint32_t v0 = smem_u32(smem + FaSmem::V + s * kTile);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // 16 keys per MMA = 8 packed TMEM columns of P
            umma_f16_ts_fa(tmem + kColO, tmem + kColP + 8 * kk, sw128_desc(v0 + kk * 2048, 128 * 128, 1024), idesc_o,
                           (kb | kk) != 0);
          umma_commit(&bars[F_PVDONE]);
          umma_commit(&bars[F_VEMPTY + s]);
          if (kb == nkb - 1) umma_commit(&bars[F_OFULL]);
          if (ms) ms[5] = clock64();
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax + epilogue: thread = query row (TMEM lane) x half of the
    // key columns (warps 2..5 the first 64, warps 6..9 the second 64)
    const uint32_t quad = warp & 3, half = (warp - 2) >> 2;
    const int r = static_cast<int>(quad * 32 + lane);
    const uint32_t lane_addr = tmem + ((quad * 32) << 16);
    float* red = reinterpret_cast<float*>(smem + FaSmem::RED);
    const float NEG_INF = __int_as_float(0xff800000);
    constexpr float LOG2E = 1.4426950408889634f;
    const int cb = static_cast<int>(half) * 64;  // this thread's first key column of a block
    uint32_t qc = 0, bc = 0;
    for (int it = 0, u; (u = fa_unit_at(a, it)) >= 0; ++it, ++qc) {
      int b, head, qt, nkb;
      fa_decode(a, u, b, head, qt, nkb);
      const int qrow = qt * 128 + r;
      const int row_lo = qt * 128 + static_cast<int>(quad) * 32, row_hi = row_lo + 31;  // this warp's rows
      float m = NEG_INF, l = 0.0f;  // l: this half's share of the row sum
      for (int kb = 0; kb < nkb; ++kb, ++bc) {
        mbar_wait(&bars[F_SFULL], bc & 1);
        long long* ts = (a.dbg && blockIdx.x == 0 && warp == 2 && lane == 0 && bc < 32) ? a.dbg + bc * 8 : nullptr;
        if (ts) ts[0] = clock64();
        tc_fence_after();
        const int key0 = kb * 128 + cb;
        auto chunk_full = [&](int c) { return key0 + c + 32 <= a.S && (!a.causal || key0 + c + 31 <= row_lo); };
        auto chunk_dead = [&](int c) { return key0 + c >= a.S || (a.causal && key0 + c > row_hi); };
        const bool dead0 = chunk_dead(0), dead1 = chunk_dead(32);
        // block max over both halves of the raw accumulators (round16(x * 0.125) is monotone)
        float m0 = NEG_INF, m1 = NEG_INF;
#pragma unroll
        for (int h = 0; h < 2 && !a.unstab; ++h) {
          const int c = 32 * h;
          if (h == 0 ? dead0 : dead1) continue;
          uint32_t v[32];
          tmem_ld32(lane_addr + kColS + cb + c, v);
          tmem_wait_ld();
          if (chunk_full(c)) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              m0 = fmax3_fa(m0, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
              m1 = fmax3_fa(m1, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int j = key0 + c + i;
              const bool valid = j < a.S && (!a.causal || j <= qrow);
              m0 = fmaxf(m0, valid ? __uint_as_float(v[i]) : NEG_INF);
            }
          }
        }
        float mnew = 0.0f;  // unstabilised: e = exp(s) (the reference's full_fp16 softmax)
        if (!a.unstab) {
          float* rmax = red + (bc & 1) * 256;
          rmax[half * 128 + r] = fmaxf(m0, m1);
          if (ts) ts[1] = clock64();
          named_bar_sync(1, 32 * kSoftmaxWarps);
          if (ts) ts[2] = clock64();
          const float mraw = fmaxf(rmax[r], rmax[128 + r]);
          const float mblk = mraw == NEG_INF ? NEG_INF : __fmul_rn(r16(mraw), 0.125f);
          mnew = fmaxf(m, mblk);
        }
        // Lazy rescaling: O and l are rescaled (and m moved) only when some row of the
        // warp saw its max grow by more than kLazy; otherwise this block's exponentials use
        // the stale max, e <= e^kLazy, well inside fp16 -- and fp16 rounding is relative, so
        // P~ keeps its precision.  Saves the O round trip through TMEM on most blocks.
        constexpr float kLazy = 5.0f;
        const bool rescale = !a.unstab && kb > 0 && __any_sync(0xffffffffu, mnew > m + kLazy);
        const float mold = m;
        if (kb == 0 || rescale) m = mnew;
        // e = exp(s - m), P~ = round16(e) -> TMEM
        // P and O are free once the previous block's P.V completed (it was issued after
        // this block's Q.K^T)
        if (bc > 0) mbar_wait(&bars[F_PVDONE], (bc - 1) & 1);
        tc_fence_after();
        const float ml = __fmul_rn(m, LOG2E);
        const uint64_t nm = f2_pack(-ml, -ml);
        const uint64_t kl8 = f2_pack(0.125f * LOG2E, 0.125f * LOG2E);  // exact: 2^-3 scaling
        uint64_t sum2 = f2_pack(0.0f, 0.0f);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = 32 * h;
          uint32_t pk[16];
          if (h == 0 ? dead0 : dead1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          } else {
            uint32_t w[32];  // reloaded: keeping both chunks live across the barrier spills
            tmem_ld32(lane_addr + kColS + cb + c, w);
            tmem_wait_ld();
            const bool full = chunk_full(c);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              // s = round16(acc) * 0.125 (= round16(acc * 0.125) outside the binary16
              // subnormal range); the 2^-3 rides in the exponent FMA
              float s0, s1;
              h2_unpack(h2_pack_rn(__uint_as_float(w[i]), __uint_as_float(w[i + 1])), s0, s1);
              float x0, x1;
              f2_unpack(f2_fma(f2_pack(s0, s1), kl8, nm), x0, x1);
              float e0 = ex2_approx(x0), e1 = ex2_approx(x1);
              if (!full) {
                const int j = key0 + c + i;
                e0 = (j < a.S && (!a.causal || j <= qrow)) ? e0 : 0.0f;
                e1 = (j + 1 < a.S && (!a.causal || j + 1 <= qrow)) ? e1 : 0.0f;
              }
              sum2 = f2_add(sum2, f2_pack(e0, e1));
              pk[i / 2] = h2_pack_rn(e0, e1);
            }
          }
          tmem_st16(lane_addr + kColP + (cb + c) / 2, pk);
        }
        float sa, sb;
        f2_unpack(sum2, sa, sb);
        // rescale this half's 32 columns of O and the partial sum to the new max (the
        // decision is warp-uniform: TMEM access is warp-collective; both halves of a row
        // see the same maxima, so they decide alike)
        if (rescale) {
          const float sc = ex2_approx(__fmul_rn(__fsub_rn(mold, m), LOG2E));
          l = __fmul_rn(l, sc);
          const uint64_t sc2 = f2_pack(sc, sc);
          uint32_t o[32];
          tmem_ld32(lane_addr + kColO + half * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float x0, x1;
            f2_unpack(f2_mul(f2_pack(__uint_as_float(o[i]), __uint_as_float(o[i + 1])), sc2), x0, x1);
            o[i] = __float_as_uint(x0);
            o[i + 1] = __float_as_uint(x1);
          }
          tmem_st32(lane_addr + kColO + half * 32, o);
        }
        l = __fadd_rn(l, __fadd_rn(sa, sb));
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[F_PREADY]);
        if (ts) ts[3] = clock64();
      }
      // epilogue: o = round16(O / l) -> ctx, this half's 32 columns; l = both halves' sums
      float* rsum = red + 512;
      rsum[half * 128 + r] = l;
      mbar_wait(&bars[F_OFULL], qc & 1);
      tc_fence_after();
      uint32_t o[32];
      tmem_ld32(lane_addr + kColO + half * 32, o);
      tmem_wait_ld();
      tc_fence_before();
      // both partial sums visible (the next write of rsum is a unit later, behind at least
      // one block barrier that this warp reaches only after its read)
      named_bar_sync(1, 32 * kSoftmaxWarps);
      // full_fp16: the reference sums e on the binary16 lattice -- a sum past 65504 is inf
      // (p -> 0), an overflowed e is inf (p -> inf / inf = NaN, kernels.cpp:154-165)
      const float lt = a.unstab ? r16(__fadd_rn(rsum[r], rsum[128 + r])) : __fadd_rn(rsum[r], rsum[128 + r]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[F_TFREE]);
      if (qrow < a.S) {
        const float inv = __frcp_rn(lt);
        const uint64_t inv2 = f2_pack(inv, inv);
        uint4* dst = reinterpret_cast<uint4*>(a.ctx + (static_cast<int64_t>(b) * a.S + qrow) * a.ld_ctx + head * 64 +
                                              half * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t pk[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float x0, x1;
            f2_unpack(f2_mul(f2_pack(__uint_as_float(o[8 * q + 2 * i]), __uint_as_float(o[8 * q + 2 * i + 1])), inv2),
                      x0, x1);
            pk[i] = h2_pack_rn(x0, x1);
          }
          dst[q] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// ---------------------------------------------------------------------------------------
// Row-owner variant (default): one softmax thread per query row (warps 0..3 = TMEM lane
// quadrants), the whole 128-key S block loaded from TMEM as packed round16 scores (masked keys
// become -inf halves, so the exponent pass needs no masking) and S released (SFREE) right after
// the load -- the next block's Q.K^T then runs under this block's exponentials.  The block max
// is taken from registers (no second TMEM read, no cross-warp barrier); the lazy running-max /
// O-rescale logic and every rounding point are those of attn_fa_kernel above.
// Measured per-block chain of attn_fa_kernel (scripts/fa_phases.py, C4): max pass 512 cycles,
// exp pass 2 966, wake-up 360, next-S wait ~1 340 = 4.8 K cycles against a MUFU floor of ~1 K.
// ---------------------------------------------------------------------------------------
// TPR threads per query row: 1 (4 softmax warps, 162 registers) or 2 (8 softmax warps, each half
// of the row's keys; the halves' block maxima meet in shared memory behind a 64-thread pairwise
// named barrier -- more warps to hide the TMEM / MUFU latencies at 2 CTAs per SM).  The code is
// written for TPR = 4 too; measured slower (59 vs 48 us at C4: 56 registers, a 4-warp barrier).
template <int TPR>
constexpr int row_threads() { return 128 * TPR + 64; }  // + TMA warp + MMA warp
enum : int {
  R_QFULL = 0, R_QEMPTY = 2, R_KFULL = 4, R_KEMPTY = 6, R_VFULL = 8, R_VEMPTY = 10,
  R_SFULL = 12,   // S block in TMEM
  R_SFREE = 13,   // softmax warps: S read (into registers)
  R_PREADY = 14,  // softmax warps: P in TMEM, O rescaled
  R_OFULL = 15,   // last P.V of the unit done
  R_TFREE = 16,   // softmax warps: O read by the epilogue
  R_PVDONE = 17,  // P.V of a block done: P columns and O free
  R_UFULL = 18,   // [4] unit ring (dynamic schedule): id published by the TMA warp
  R_UEMPTY = 22,  // [4] unit ring: read by the MMA thread and every softmax warp
  R_COUNT = 26
};

__device__ __forceinline__ uint32_t h2_max(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

template <int TPR>
__global__ void __launch_bounds__(row_threads<TPR>(), 2) attn_fa_row_kernel(const __grid_constant__ CUtensorMap tm, const FaArgs a) {
  constexpr int kRowWarps = 4 * TPR, NC = 4 / TPR;  // softmax warps, 32-key chunks per thread
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FaSmem::BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + R_COUNT);
  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t kTmaWarp = kRowWarps, kMmaWarp = kRowWarps + 1;

  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch_desc(&tm);
    for (int i = 0; i < R_COUNT; ++i)
      mbar_init(&bars[i], (i == R_SFREE || i == R_PREADY || i == R_TFREE) ? kRowWarps
                          : (i >= R_UEMPTY && i < R_UEMPTY + 4)      ? 1 + kRowWarps
                                                                      : 1);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem = *tmem_slot;
  if (a.dbg && threadIdx.x == 0) a.dbg[256 + 2 * blockIdx.x] = globaltimer();  // per-CTA span (debug)
  // Dynamic schedule (a.work): the TMA warp claims units (heavy first: unit ids are ordered by
  // key-block count) from a global counter and publishes them through a 4-entry ring, so the two
  // CTAs of an SM -- which the warp scheduler does not serve equally -- and every SM finish
  // together.  Consumers read each entry once and release it at once.
  volatile int* uring = reinterpret_cast<volatile int*>(tmem_slot + 1);
  const int n_units = a.B * a.H * a.nqt;
  auto unit_claim = [&](int k) -> int {  // TMA warp, lane 0
    if (a.work == nullptr) return fa_unit_at(a, k);
    const int slot = k & 3;
    mbar_wait(&bars[R_UEMPTY + slot], ((k >> 2) & 1) ^ 1);
    int u = atomicAdd(a.work, 1);
    if (u >= n_units) u = -1;
    uring[slot] = u;
    mbar_arrive(&bars[R_UFULL + slot]);
    return u;
  };
  auto unit_read = [&](int k, bool warp_wide) -> int {  // MMA thread (warp_wide false) / softmax warps
    if (a.work == nullptr) return fa_unit_at(a, k);
    const int slot = k & 3;
    mbar_wait(&bars[R_UFULL + slot], (k >> 2) & 1);
    const int u = uring[slot];
    if (warp_wide) __syncwarp();
    if (!warp_wide || lane == 0) mbar_arrive(&bars[R_UEMPTY + slot]);
    return u;
  };

  if (warp == kTmaWarp) {
    // ---------------- TMA producer: per unit Q, then K/V blocks in consumption order
    if (lane == 0) {
      pdl_wait();  // q/k/v are written by the upstream QKV GEMM
      uint32_t qc = 0, kc = 0;
      for (int it = 0, u; (u = unit_claim(it)) >= 0; ++it, ++qc) {
        int b, head, qt, nkb;
        fa_decode(a, u, b, head, qt, nkb);
        const uint32_t qs = qc & 1;
        mbar_wait(&bars[R_QEMPTY + qs], ((qc >> 1) & 1) ^ 1);
        mbar_expect_tx(&bars[R_QFULL + qs], kTile);
        tma_load_3d(smem + FaSmem::Q + qs * kTile, &tm, &bars[R_QFULL + qs], head * 64, qt * 128, b);
        for (int kb = 0; kb < nkb; ++kb, ++kc) {
          const uint32_t s = kc & 1, ph = ((kc >> 1) & 1) ^ 1;
          mbar_wait(&bars[R_KEMPTY + s], ph);
          mbar_expect_tx(&bars[R_KFULL + s], kTile);
          tma_load_3d(smem + FaSmem::K + s * kTile, &tm, &bars[R_KFULL + s], a.h + head * 64, kb * 128, b);
          mbar_wait(&bars[R_VEMPTY + s], ph);
          mbar_expect_tx(&bars[R_VFULL + s], kTile);
          tma_load_3d(smem + FaSmem::V + s * kTile, &tm, &bars[R_VFULL + s], 2 * a.h + head * 64, kb * 128, b);
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer: S_kb+1 as soon as the softmax has S_kb in registers (SFREE),
    // P.V_kb once it wrote P (PREADY)
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_f16_f32(128, 128, 0, 0);
      constexpr uint32_t idesc_o = idesc_f16_f32(128, 64, 0, 1);
      uint32_t qc = 0, kc = 0, bc = 0;
      auto issue_s = [&](uint32_t q0, uint32_t kcount, bool last_of_unit, uint32_t qs) {
        const uint32_t s = kcount & 1;
        mbar_wait(&bars[R_KFULL + s], (kcount >> 1) & 1);
        tc_fence_after();
        const uint32_t k0 = smem_u32(smem + FaSmem::K + s * kTile);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_f16_ss(tmem + kColS, sw128_desc(q0 + k * 32, 0, 1024), sw128_desc(k0 + k * 32, 0, 1024), idesc_s,
                      k != 0);
        umma_commit(&bars[R_SFULL]);
        umma_commit(&bars[R_KEMPTY + s]);
        if (last_of_unit) umma_commit(&bars[R_QEMPTY + qs]);
      };
      // The next block's Q.K^T is issued as soon as the softmax has read S -- across unit
      // boundaries too (the next unit's Q is double-buffered), so a unit's first S is ready
      // when the softmax warps come back from the previous unit's epilogue.
      auto q_addr = [&](uint32_t qcount) { return smem_u32(smem + FaSmem::Q + (qcount & 1) * kTile); };
      int u = unit_read(0, false);
      int nkb = 0;
      if (u >= 0) {
        int b_, h_, qt_;
        fa_decode(a, u, b_, h_, qt_, nkb);
        mbar_wait(&bars[R_QFULL], 0);
        issue_s(q_addr(0), 0, nkb == 1, 0);
      }
      for (int it = 0; u >= 0; ++it, ++qc) {
        const uint32_t qs = qc & 1;
        const uint32_t q0 = q_addr(qc);
        int un = -1, nkb_next = 0;  // the next unit: read at this unit's last block (the TMA warp
                                    // publishes it only after issuing this unit's last loads)
        for (int kb = 0; kb < nkb; ++kb, ++kc, ++bc) {
          const uint32_t s = kc & 1, ph = (kc >> 1) & 1;
          if (kb + 1 == nkb) {
            un = unit_read(it + 1, false);
            if (un >= 0) {
              int b_, h_, qt_;
              fa_decode(a, un, b_, h_, qt_, nkb_next);
            }
          }
          if (kb + 1 < nkb) {
            mbar_wait_spin(&bars[R_SFREE], bc & 1);
            issue_s(q0, kc + 1, kb + 2 == nkb, qs);
          } else if (un >= 0) {
            mbar_wait_spin(&bars[R_SFREE], bc & 1);
            mbar_wait(&bars[R_QFULL + (qs ^ 1)], ((qc + 1) >> 1) & 1);
            issue_s(q_addr(qc + 1), kc + 1, nkb_next == 1, qs ^ 1);
          }
          mbar_wait_spin(&bars[R_PREADY], bc & 1);
          long long* ms = (a.dbg && blockIdx.x == 0 && bc < 32) ? a.dbg + bc * 8 : nullptr;
          if (ms) ms[4] = clock64();
          if (kb == 0 && qc > 0) mbar_wait(&bars[R_TFREE], (qc - 1) & 1);
          mbar_wait(&bars[R_VFULL + s], ph);
          tc_fence_after();
          const uint32_t v0 = smem_u32(smem + FaSmem::V + s * kTile);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)  // 16 keys per MMA = 8 packed TMEM columns of P
            umma_f16_ts_fa(tmem + kColO, tmem + kColP + 8 * kk, sw128_desc(v0 + kk * 2048, 128 * 128, 1024), idesc_o,
                           (kb | kk) != 0);
          umma_commit(&bars[R_PVDONE]);
          umma_commit(&bars[R_VEMPTY + s]);
          if (kb == nkb - 1) umma_commit(&bars[R_OFULL]);
          if (ms) ms[5] = clock64();
        }
        u = un;
        nkb = nkb_next;
      }
    }
    __syncwarp();
  } else {
    // ---------------- softmax + epilogue: thread = query row (TMEM lane)
    const uint32_t quad = warp & 3, half = warp >> 2;  // half: which NC chunks of a block (TPR > 1)
    constexpr int OC = 64 / TPR;  // this thread's O columns
    const int r = static_cast<int>(quad * 32 + lane);
    float* red = reinterpret_cast<float*>(smem + FaSmem::RED);
    const uint32_t lane_addr = tmem + ((quad * 32) << 16);
    const float NEG_INF = __int_as_float(0xff800000);
    constexpr uint32_t NEG_INF2 = 0xFC00FC00u;  // (-inf, -inf) as f16x2
    constexpr float LOG2E = 1.4426950408889634f;
    uint32_t qc = 0, bc = 0;
    // A unit's epilogue (o = round16(O / l) -> ctx) runs after the NEXT unit's first block has
    // its exponentials in registers: the wait for the unit's last P.V (OFULL) then hides behind
    // that block's S load and exponent pass instead of stalling the row between units.
    struct Pending { float l; int64_t dst; bool live; } pe{0.0f, 0, false};
    // the row's partial sums meet in shared memory, double-buffered by unit parity: a CTA's last
    // unit may be a single block, and then no block-max barrier separates one epilogue's reads
    // from the next epilogue's writes (compute-sanitizer racecheck)
    static_assert(TPR == 1 || 1024 + 2 * TPR * 128 <= 6 * 256, "rsum double buffer fits the RED region");
    auto epilogue = [&](uint32_t qcount) {
      float* rsum = red + 1024 + (qcount & 1) * (TPR * 128);
      if constexpr (TPR > 1) rsum[half * 128 + r] = pe.l;
      mbar_wait(&bars[R_OFULL], qcount & 1);
      tc_fence_after();
      uint32_t o[OC];
#pragma unroll
      for (int hh = 0; hh < OC / 16; ++hh)
        tmem_ld16(lane_addr + kColO + OC * static_cast<uint32_t>(half) + 16 * hh, *reinterpret_cast<uint32_t(*)[16]>(o + 16 * hh));
      tmem_wait_ld();
      tc_fence_before();
      float l = pe.l;
      if constexpr (TPR > 1) {  // every part's sum visible; the next rsum write is a unit (and a row barrier) later
        named_bar_sync(1 + quad, 32 * TPR);
        float lt2 = rsum[r];
#pragma unroll
        for (int q = 1; q < TPR; ++q) lt2 = __fadd_rn(lt2, rsum[q * 128 + r]);
        l = lt2;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[R_TFREE]);
      // full_fp16: the reference sums e on the binary16 lattice (kernels.cpp:154-165)
      const float lt = a.unstab ? r16(l) : l;
      if (pe.dst >= 0) {
        const float inv = __frcp_rn(lt);
        const uint64_t inv2 = f2_pack(inv, inv);
        uint4* dst = reinterpret_cast<uint4*>(a.ctx + pe.dst);
#pragma unroll
        for (int q = 0; q < OC / 8; ++q) {
          uint32_t pk[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float x0, x1;
            f2_unpack(f2_mul(f2_pack(__uint_as_float(o[8 * q + 2 * i]), __uint_as_float(o[8 * q + 2 * i + 1])), inv2),
                      x0, x1);
            pk[i] = h2_pack_rn(x0, x1);
          }
          dst[q] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
      pe.live = false;
    };
    for (int it = 0, u; (u = unit_read(it, true)) >= 0; ++it, ++qc) {
      int b, head, qt, nkb;
      fa_decode(a, u, b, head, qt, nkb);
      const int qrow = qt * 128 + r;
      const int row_lo = qt * 128 + static_cast<int>(quad) * 32, row_hi = row_lo + 31;  // this warp's rows
      const int key_lim = a.causal ? min(a.S - 1, qrow) : a.S - 1;  // last key this row sees
      float m = NEG_INF, l = 0.0f;
      for (int kb = 0; kb < nkb; ++kb, ++bc) {
        mbar_wait(&bars[R_SFULL], bc & 1);
        long long* ts = (a.dbg && blockIdx.x == 0 && warp == 0 && lane == 0 && bc < 32) ? a.dbg + bc * 8 : nullptr;
        if (ts) ts[0] = clock64();
        tc_fence_after();
        const int key0 = kb * 128;
        // per 32-key chunk (warp-uniform): dead = no key of the chunk is visible to any row of
        // the warp; full = every key visible to every row of the warp
        uint32_t sp[16 * NC];  // round16 scores, packed pairs; masked keys -inf
        uint32_t hm[4] = {NEG_INF2, NEG_INF2, NEG_INF2, NEG_INF2};  // independent max chains
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          const int c = static_cast<int>(half) * NC + cc;
          const int k0c = key0 + 32 * c;
          const bool dead = k0c >= a.S || (a.causal && k0c > row_hi);
          if (dead) {
#pragma unroll
            for (int i = 0; i < 16; ++i) sp[16 * cc + i] = NEG_INF2;
            continue;
          }
          uint32_t w[32];
          if constexpr (TPR == 4) {  // register budget (56 at 2 x 576 threads): two 16-column loads
            tmem_ld16(lane_addr + kColS + 32 * c, *reinterpret_cast<uint32_t(*)[16]>(w));
            tmem_ld16(lane_addr + kColS + 32 * c + 16, *reinterpret_cast<uint32_t(*)[16]>(w + 16));
          } else {
            tmem_ld32(lane_addr + kColS + 32 * c, w);
          }
          tmem_wait_ld();
          if (ts && cc == 0) ts[6] = clock64();
          if (k0c + 32 <= a.S && (!a.causal || k0c + 31 <= row_lo)) {  // warp-uniform: no masking
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const uint32_t hv = h2_pack_rn(__uint_as_float(w[2 * i]), __uint_as_float(w[2 * i + 1]));
              sp[16 * cc + i] = hv;
              hm[i & 3] = h2_max(hm[i & 3], hv);
            }
          } else {  // keys j > lim are masked: branch-free selects
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int j = k0c + 2 * i;
              const uint32_t hv = h2_pack_rn(__uint_as_float(w[2 * i]), __uint_as_float(w[2 * i + 1]));
              const uint32_t keep = (j <= key_lim ? 0x0000FFFFu : 0u) | (j + 1 <= key_lim ? 0xFFFF0000u : 0u);
              const uint32_t mv = (hv & keep) | (NEG_INF2 & ~keep);
              sp[16 * cc + i] = mv;
              hm[i & 3] = h2_max(hm[i & 3], mv);
            }
          }
        }
        const uint32_t hmax = h2_max(h2_max(hm[0], hm[1]), h2_max(hm[2], hm[3]));
        if (ts) ts[7] = clock64();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[R_SFREE]);  // the next Q.K^T may overwrite S now
        if (ts) ts[1] = clock64();
        float mnew = 0.0f;  // unstabilised: e = exp(s) (the reference's full_fp16 softmax)
        if (!a.unstab) {
          float h0, h1;
          h2_unpack(hmax, h0, h1);
          float mraw = fmaxf(h0, h1);  // = round16(max acc): round16 is monotone
          if constexpr (TPR > 1) {  // the row's other parts: shared memory + a barrier of the row's warps
            float* rmax = red + (bc & 1) * 512;  // by block parity: a fast group may write the next block's first
            rmax[half * 128 + r] = mraw;
            named_bar_sync(1 + quad, 32 * TPR);
#pragma unroll
            for (int q = 0; q < TPR; ++q) mraw = fmaxf(mraw, rmax[q * 128 + r]);
          }
          const float mblk = mraw == NEG_INF ? NEG_INF : __fmul_rn(mraw, 0.125f);
          mnew = fmaxf(m, mblk);
        }
        constexpr float kLazy = 5.0f;  // see attn_fa_kernel
        const bool rescale = !a.unstab && kb > 0 && __any_sync(0xffffffffu, mnew > m + kLazy);
        const float mold = m;
        if (kb == 0 || rescale) m = mnew;
        // e = exp(s - m), P~ = round16(e), in registers before the wait for the previous P.V
        // (s = round16(acc) * 2^-3, the 2^-3 in the FMA); four independent partial sums
        const float ml = __fmul_rn(m, LOG2E);
        const uint64_t nm = f2_pack(-ml, -ml);
        const uint64_t kl8 = f2_pack(0.125f * LOG2E, 0.125f * LOG2E);
        uint64_t sum2[2] = {f2_pack(0.0f, 0.0f), f2_pack(0.0f, 0.0f)};
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) {
          const int c = static_cast<int>(half) * NC + cc;
          const int k0c = key0 + 32 * c;
          if (k0c >= a.S || (a.causal && k0c > row_hi)) {  // dead chunk: P~ = 0
#pragma unroll
            for (int i = 0; i < 16; ++i) sp[16 * cc + i] = 0u;
            continue;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float s0, s1, x0, x1;
            h2_unpack(sp[16 * cc + i], s0, s1);
            f2_unpack(f2_fma(f2_pack(s0, s1), kl8, nm), x0, x1);
            const float e0 = ex2_approx(x0), e1 = ex2_approx(x1);  // ex2(-inf) = 0: masked keys
            sum2[i & 1] = f2_add(sum2[i & 1], f2_pack(e0, e1));
            sp[16 * cc + i] = h2_pack_rn(e0, e1);  // P~ replaces the score in place
          }
        }
        if (pe.live) epilogue(qc - 1);  // (kb == 0: the previous unit's O, then TFREE)
        if (bc > 0) mbar_wait(&bars[R_PVDONE], (bc - 1) & 1);  // P columns and O free
        tc_fence_after();
        if (ts) ts[2] = clock64();
        if (rescale) {
          const float sc = ex2_approx(__fmul_rn(__fsub_rn(mold, m), LOG2E));
          l = __fmul_rn(l, sc);
          const uint64_t sc2 = f2_pack(sc, sc);
#pragma unroll
          for (int hh = 0; hh < OC / 16; ++hh) {  // this thread's O columns, 16 at a time
            const uint32_t oc = kColO + OC * static_cast<uint32_t>(half) + 16 * hh;
            uint32_t o[16];
            tmem_ld16(lane_addr + oc, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              float x0, x1;
              f2_unpack(f2_mul(f2_pack(__uint_as_float(o[i]), __uint_as_float(o[i + 1])), sc2), x0, x1);
              o[i] = __float_as_uint(x0);
              o[i + 1] = __float_as_uint(x1);
            }
            tmem_st16(lane_addr + oc, o);
          }
        }
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
          tmem_st16(lane_addr + kColP + 16 * (static_cast<uint32_t>(half) * NC + cc), *reinterpret_cast<uint32_t(*)[16]>(sp + 16 * cc));
        float sa, sb, sc_, sd;
        f2_unpack(sum2[0], sa, sb);
        f2_unpack(sum2[1], sc_, sd);
        l = __fadd_rn(l, __fadd_rn(__fadd_rn(sa, sb), __fadd_rn(sc_, sd)));
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars[R_PREADY]);
        if (ts) ts[3] = clock64();
      }
      // epilogue deferred (see Pending): this thread's 64 / TPR columns of the ctx row
      pe.l = l;
      pe.dst = qrow < a.S ? (static_cast<int64_t>(b) * a.S + qrow) * a.ld_ctx + head * 64 + half * OC : -1;
      pe.live = true;
    }
    if (pe.live) epilogue(qc - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (a.dbg && threadIdx.x == 0) a.dbg[257 + 2 * blockIdx.x] = globaltimer();
  if (a.work != nullptr && threadIdx.x == 0) {  // the last CTA out re-arms the counter for the next launch
    __threadfence();
    if (atomicAdd(a.work + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      a.work[0] = 0;
      a.work[1] = 0;
      __threadfence();
    }
  }
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace

bool attn_fa_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PRLAB_ATTN_FA");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

// Balanced static schedule for the persistent grid: units (b, head, q-tile) cost their
// key-block count plus ~half a block of per-unit overhead (the Q load, the epilogue and the
// pipeline refill at a unit boundary); longest-processing-time-first onto the least-loaded
// CTA, each CTA's list heavy first.  The serpentine order it replaces gave C4 CTAs 12-14
// blocks in 5-6 units, and the 14-block / 6-unit CTAs finished 7 us after the rest
// (scripts/fa_phases.py).  Built at plan time, cached per (device, shape, grid).
const int* attn_fa_schedule(int B, int S, int H, int causal) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int>, int*> cache;
  int dev = 0;
  PRLAB_CUDA(cudaGetDevice(&dev));
  const int nqt = (S + 127) / 128, items = B * H, n = items * nqt;
  const int grid = std::min(n, 2 * num_sms());
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, B * H, nqt, causal, grid);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  auto nkb = [&](int u) { const int qt = nqt - 1 - u / items; return causal ? qt + 1 : nqt; };
  std::vector<int> order(n);
  for (int u = 0; u < n; ++u) order[u] = u;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return nkb(x) > nkb(y); });
  using Load = std::pair<double, int>;  // (cost, cta): min-heap, ties to the lower CTA index
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (int c = 0; c < grid; ++c) heap.push({0.0, c});
  std::vector<std::vector<int>> lists(grid);
  for (int u : order) {
    const Load l = heap.top();
    heap.pop();
    lists[l.second].push_back(u);
    heap.push({l.first + nkb(u) + 0.5, l.second});
  }
  std::vector<int> host(grid + 1 + n);
  int o = 0;
  for (int c = 0; c < grid; ++c) {
    host[c] = o;
    for (int u : lists[c]) host[grid + 1 + o++] = u;
  }
  host[grid] = o;
  int* d = nullptr;
  PRLAB_CUDA(cudaMalloc(&d, host.size() * sizeof(int)));
  PRLAB_CUDA(cudaMemcpy(d, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice));
  cache.emplace(key, d);
  return d;
}

void launch_attn_fa(const AttnPlan& p, cudaStream_t st) {
  static std::mutex mu;
  static uint64_t done = 0;
  once_per_device(mu, done, [] {
    PRLAB_CUDA(cudaFuncSetAttribute(attn_fa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kFaSmemBytes)));
    PRLAB_CUDA(cudaFuncSetAttribute(attn_fa_row_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kFaSmemBytes)));
    PRLAB_CUDA(cudaFuncSetAttribute(attn_fa_row_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kFaSmemBytes)));
  });
  static const int row = [] {  // threads per row of the row-owner kernel (0: half-row kernel)
    const char* e = std::getenv("PRLAB_ATTN_ROW");
    return e == nullptr ? 2 : std::atoi(e);
  }();
  FaArgs a;
  a.B = p.B;
  a.S = p.S;
  a.H = p.H;
  a.causal = p.causal;
  a.nqt = (p.S + 127) / 128;
  a.h = p.H * p.hd;
  a.ctx = reinterpret_cast<__half*>(p.ctx);
  a.ld_ctx = p.ld_ctx;
  a.dbg = p.dbg;
  a.unstab = p.unstab;
  const int units = p.B * p.H * a.nqt;
  const int grid = std::min(units, 2 * num_sms());
  a.sched = std::getenv("PRLAB_ATTN_SERPENTINE") ? nullptr : p.fa_sched;
  a.work = (row == 2 || row == 1) && !std::getenv("PRLAB_ATTN_STATIC") ? p.fa_work : nullptr;  // (row kernels only)
  if (row == 2)
    launch_pdl(attn_fa_row_kernel<2>, dim3(grid), dim3(row_threads<2>()), kFaSmemBytes, st, p.tmQKV, a);
  else if (row == 1)
    launch_pdl(attn_fa_row_kernel<1>, dim3(grid), dim3(row_threads<1>()), kFaSmemBytes, st, p.tmQKV, a);
  else
    launch_pdl(attn_fa_kernel, dim3(grid), dim3(kThreads), kFaSmemBytes, st, p.tmQKV, a);
}

}  // namespace prlab_gpu
