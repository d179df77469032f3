// tcgen05 GEMM for the hybrid Linear class (reference matmul + linear_bias,
// src/kernels.cpp:40-83 and src/model.cpp:66-78, under the hybrid config
// {F16E compute, F32 accum}: fp16 operands, fp32 accumulation, one final
// round16, then the bias add on the fp16 lattice).
//
//   out[m, n] = epi( sum_k A[m, k] * Wt[n, k] )      A: [M, K] fp16, Wt: [N, K] fp16
//
// Persistent, warp-specialised kernel, one CTA per SM:
//   warp 0      TMA producer: 128x64 A tile + BNx64 W tile per stage (128B swizzle).
//               The first stages' weight tiles are fetched BEFORE griddepcontrol.wait:
//               weights never depend on the upstream kernel, so with programmatic
//               dependent launch their HBM latency hides under the previous kernel.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 2..5  epilogue: tcgen05.ld (thread = output row), fused bias / GELU /
//               residual, fp16 or fp32 stores
// Two TMEM accumulator stages (2*BN columns) let the epilogue of unit i overlap
// the main loop of unit i+1.
//
// Split-K (small M, e.g. batch-1 latency): a work unit is (tile, k-split).  Each
// unit writes its fp32 partial tile to a workspace; the last unit of a tile to
// arrive (atomic ticket) sums the partials in split order -- deterministic --
// and applies the epilogue, so the rounding points are those of the full sum.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

constexpr int BM = 128, BK = 64;

struct GemmArgs {
  int M, N, K;
  int num_m_blocks, num_n_blocks, num_tiles, num_k_blocks;
  int splits, kb_per_split;
  const float* bias;
  void* out;
  int64_t ldo;
  float* ws;      // split-K partials [tile*splits + split][BM][BN]
  int* tickets;   // per-tile arrival counters (left at zero after every launch)
  int tma_store;  // epilogue through smem staging + TMA store / reduce-add
  int group_m;    // raster band height in m-blocks (A band kept L2-resident)
  int dbg_noload; // debug: after the first fill, skip the TMA loads (MMA/epilogue pacing probe)
  const int32_t* targets;  // EPI_ROWSTAT: target column per row (< 0: none)
  float* tval;             // EPI_ROWSTAT: round16 logit at the target column per row
  long long* dbg; // optional per-CTA %globaltimer stamps [grid][8] (debug), null = off
  int acc16;      // FP16 accumulator (idesc c_format F16; full_fp16 fast path), else FP32
};

// An FP16 accumulator sits in the low half of each 32-bit TMEM cell (probed on B200,
// scripts/ubench/probe_tmem_layout.cu): widen it so the fp32 epilogues apply unchanged
// (exact: every binary16 value is an fp32 value).
__device__ __forceinline__ void acc16_widen(uint32_t (&u)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i)
    u[i] = __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(u[i] & 0xFFFFu))));
}

// LEAN: half-depth pipeline (~100 KB smem) so two CTAs -- this kernel's and the
// next PDL-launched kernel's -- can be co-resident on an SM at batch-1 sizes.
template <int BN, bool LEAN, int EPI = 0>
struct Cfg {
  static constexpr int STAGES0 = (BN == 256 ? 4 : (BN == 128 ? 6 : 8)) / (LEAN ? 2 : 1);
  // epilogue warps: 1, 2 or 4 per TMEM lane quadrant; the erf-heavy GELU epilogue gets
  // the most so it keeps pace with the tensor core
  static constexpr int EPI_WARPS = BN >= 128 ? 8 : 4;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr int COLS_PER_WARP = BN / (EPI_WARPS / 4);
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  // TMA-store epilogue: two 32-row x 128-byte staging buffers per epilogue warp
  static constexpr uint32_t EPI_BYTES = EPI_WARPS * 2 * 4096;
  static constexpr uint32_t BIAS_BYTES = EPI_WARPS * COLS_PER_WARP * 4;
  static constexpr uint32_t SMEM_BUDGET = 227 * 1024 - 1024 - 256 - EPI_BYTES - BIAS_BYTES;
  static constexpr int STAGES = STAGES0 * STAGE_BYTES <= SMEM_BUDGET ? STAGES0 : SMEM_BUDGET / STAGE_BYTES;
  static constexpr uint32_t EPI_OFF = STAGES * STAGE_BYTES;           // 1024-aligned (stage sizes are)
  static constexpr uint32_t BAR_OFF = EPI_OFF + EPI_BYTES;
  static constexpr uint32_t BIAS_OFF = BAR_OFF + 256;                 // per-warp bias slices
  static constexpr size_t SMEM = 1024 + BIAS_OFF + BIAS_BYTES;
};

// epilogues with a bias operand / an fp32 output tile
__host__ __device__ constexpr bool epi_bias(int epi) { return epi != EPI_F16 && epi != EPI_F16_F32; }
__host__ __device__ constexpr bool epi_f32out(int epi) { return epi == EPI_BIAS_RESID_F32 || epi == EPI_F16_F32; }

// Pairs go through the packed pipes: cvt.rn.f16x2 (= round16 of both lanes), then the
// bias add as a binary16 RNE add (= round16(round16(acc) + b) since b is on the lattice).
template <int EPI>
__device__ __forceinline__ uint32_t epilogue_pair(float a0, float a1, float b0, float b1) {
  uint32_t h = h2_pack_rn(a0, a1);
  if (epi_bias(EPI)) {
    h = h2_add_rn(h, h2_pack_rn(b0, b1));  // exact repack: biases are pre-rounded (0 when absent)
    if (EPI == EPI_BIAS_GELU_F16) {
      float x0, x1;
      h2_unpack(h, x0, x1);
      gelu2_fast(x0, x1);
      h = h2_pack_rn(x0, x1);
    }
  }
  return h;
}
template <int EPI>
__device__ __forceinline__ uint32_t epilogue_pair(float a0, float a1, const float* sbias, int i) {
  float b0 = 0.0f, b1 = 0.0f;
  if (epi_bias(EPI) && sbias != nullptr) {
    const float2 b = *reinterpret_cast<const float2*>(sbias + i);
    b0 = b.x;
    b1 = b.y;
  }
  return epilogue_pair<EPI>(a0, a1, b0, b1);
}

// sbias: the 32 (pre-rounded) bias values of columns col0..col0+31 in shared memory, or null.
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const float (&acc)[32], const GemmArgs& g, int row,
                                               int col0, const float* sbias) {
  if (row >= g.M) return;
  const bool full = col0 + 32 <= g.N;
  float v[32];
#pragma unroll
  for (int i = 0; i < 16; ++i)  // round16(acc) [+ conform(b), round16] [GELU, round16]
    h2_unpack(epilogue_pair<EPI>(acc[2 * i], acc[2 * i + 1], sbias, 2 * i), v[2 * i], v[2 * i + 1]);
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
  } else if (EPI == EPI_F16_F32) {
    float* o = reinterpret_cast<float*>(g.out) + static_cast<int64_t>(row) * g.ldo + col0;
    if (full && (g.ldo % 4) == 0) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) o[i] = v[i];
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

// Tile rasterization: bands of up to 16 m-blocks; inside a band the n-blocks
// advance slowest, so the CTAs resident at any moment share one band of A
// (<= 2048 rows) and a few weight tiles -- both stay in L2 (A is read from DRAM once).
__device__ __forceinline__ void tile_coords(const GemmArgs& g, int tile, int& m_blk, int& n_blk) {
  const int GROUP_M = g.group_m;
  const int band = tile / (GROUP_M * g.num_n_blocks);
  const int m0 = band * GROUP_M;
  const int rows = min(GROUP_M, g.num_m_blocks - m0);
  const int local = tile - band * GROUP_M * g.num_n_blocks;
  n_blk = local / rows;
  m_blk = m0 + local % rows;
}

// The Linear-class epilogue numerics on one 32-column chunk of fp32 accumulators:
// round16(acc) [+ round16(b), round16] [GELU, round16]  (kernels.cpp:78, model.cpp:73,
// kernels.cpp:232).  The residual add itself happens in the store path.
// fp16 outputs: 16 packed f16x2 words
template <int EPI>
__device__ __forceinline__ void epilogue_packed(const uint32_t (&u)[32], const float* sbias, uint32_t (&pk)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i)
    pk[i] = epilogue_pair<EPI>(__uint_as_float(u[2 * i]), __uint_as_float(u[2 * i + 1]), sbias, 2 * i);
}

template <int EPI>
__device__ __forceinline__ void epilogue_values(const uint32_t (&u)[32], const float* sbias, float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 16; ++i)
    h2_unpack(epilogue_pair<EPI>(__uint_as_float(u[2 * i]), __uint_as_float(u[2 * i + 1]), sbias, 2 * i),
              v[2 * i], v[2 * i + 1]);
}

__device__ __forceinline__ void unit_range(const GemmArgs& g, int unit, int& tile, int& split,
                                           int& kb0, int& kb1) {
  tile = unit / g.splits;
  split = unit - tile * g.splits;
  kb0 = split * g.kb_per_split;
  kb1 = min(g.num_k_blocks, kb0 + g.kb_per_split);
}

template <int BN, bool LEAN, int EPI>
__global__ void __launch_bounds__(Cfg<BN, LEAN, EPI>::THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const GemmArgs g) {
  using C = Cfg<BN, LEAN, EPI>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int total_units = g.num_tiles * g.splits;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], C::EPI_WARPS);
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
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int pre = 0;
      if (static_cast<int>(blockIdx.x) < total_units) {
        int tile, split, kb0, kb1;
        unit_range(g, blockIdx.x, tile, split, kb0, kb1);
        int m_blk0, n_blk;
        tile_coords(g, tile, m_blk0, n_blk);
        pre = min(C::STAGES, kb1 - kb0);
        for (int i = 0; i < pre; ++i) {  // weights: independent of the upstream kernel
          mbar_expect_tx(&full[i], C::STAGE_BYTES);
          tma_load_2d(sB + i * C::B_BYTES, &tmB, &full[i], (kb0 + i) * BK, n_blk * BN);
        }
      }
      pdl_wait();  // activations below are produced by the upstream kernel
      uint32_t stage = 0, phase = 0;
      bool first = true;
      for (int unit = blockIdx.x; unit < total_units; unit += gridDim.x) {
        int tile, split, kb0, kb1;
        unit_range(g, unit, tile, split, kb0, kb1);
        int m_blk, n_blk;
      tile_coords(g, tile, m_blk, n_blk);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (first && kb - kb0 < pre) {
            tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
            tma_load_2d(sB + stage * C::B_BYTES, &tmB, &full[stage], kb * BK, n_blk * BN);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        first = false;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = idesc_f16_f32(BM, BN, 0, 0) & (g.acc16 ? ~(3u << 4) : ~0u);
    uint32_t stage = 0, phase = 0, t = 0;
    for (int unit = blockIdx.x; unit < total_units; unit += gridDim.x, ++t) {
      int tile, split, kb0, kb1;
      unit_range(g, unit, tile, split, kb0, kb1);
      const uint32_t acc = t & 1, acc_phase = (t >> 1) & 1;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_f16_ss(d_tmem, sw128_desc(a0 + k * 32, 0, 1024), sw128_desc(b0 + k * 32, 0, 1024),
                        idesc, (kb > kb0 || k > 0) ? 1u : 0u);
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
    const uint32_t quad = warp & 3;                     // TMEM lane quadrant this warp may access
    const int cbase = ((warp - 2) >> 2) * C::COLS_PER_WARP;  // this warp's column slice
    const int r = quad * 32 + lane;                     // row within the tile
    const int tid = (warp - 2) * 32 + lane;
    float* sbias = reinterpret_cast<float*>(smem + C::BIAS_OFF) + (warp - 2) * C::COLS_PER_WARP;
    uint32_t t = 0;
    uint32_t store_k = 0;  // TMA-store staging buffer parity (per warp, across tiles)
    for (int unit = blockIdx.x; unit < total_units; unit += gridDim.x, ++t) {
      int tile, split, kb0, kb1;
      unit_range(g, unit, tile, split, kb0, kb1);
      int m_blk, n_blk;
      tile_coords(g, tile, m_blk, n_blk);
      const uint32_t acc = t & 1, acc_phase = (t >> 1) & 1;
      // stage this warp's bias slice while the accumulator is still being produced
      const bool has_bias = epi_bias(EPI) && g.bias != nullptr;
      if (has_bias) {
        __syncwarp();
        for (int c = lane; c < C::COLS_PER_WARP; c += 32) {
          const int col = n_blk * BN + cbase + c;
          sbias[c] = col < g.N ? __ldg(g.bias + col) : 0.0f;
        }
        __syncwarp();
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m_blk * BM + r;
      // (fp32 logits with unaligned rows: staged like the TMA store, written by the warp
      // one row at a time -- 128-byte coalesced rows instead of one row per lane)
      if (g.splits == 1 && (g.tma_store || EPI == EPI_F16_F32)) {
        // fp16 out: 64-column store chunks (2 TMEM loads); fp32 residual: 32-column
        // chunks added into x by the TMA engine (cp.reduce.async.bulk .add.f32)
        constexpr bool F32OUT = epi_f32out(EPI);
        constexpr int SC = F32OUT ? 32 : 64;
        uint8_t* ebuf = smem + C::EPI_OFF + (warp - 2) * 2 * 4096;
#pragma unroll 1
        for (int c = cbase; c < cbase + C::COLS_PER_WARP; c += SC, ++store_k) {
          uint8_t* buf = ebuf + (store_k & 1) * 4096;
          if (lane == 0) bulk_wait_read<1>();  // this buffer's previous store has been read
          __syncwarp();
          uint8_t* rowp = buf + lane * 128;
#pragma unroll
          for (int h = 0; h < SC; h += 32) {
            uint32_t u[32];
            tmem_ld32(tmem_base + ((quad * 32) << 16) + acc * BN + c + h, u);
            tmem_wait_ld();
            if (g.acc16) acc16_widen(u);
            const float* sb = has_bias ? sbias + (c - cbase) + h : nullptr;
            if (F32OUT) {
              float v[32];
              epilogue_values<EPI>(u, sb, v);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                *reinterpret_cast<float4*>(rowp + ((j ^ (lane & 7)) * 16)) =
                    make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            } else {
              uint32_t pk[16];
              epilogue_packed<EPI>(u, sb, pk);
#pragma unroll
              for (int j = 0; j < 4; ++j)
                *reinterpret_cast<uint4*>(rowp + ((((h >> 3) + j) ^ (lane & 7)) * 16)) =
                    make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            }
          }
          if (EPI == EPI_F16_F32 && !g.tma_store) {
            __syncwarp();
            const int col = n_blk * BN + c + static_cast<int>(lane);
            const int row0 = m_blk * BM + static_cast<int>(quad) * 32;
            float* o = reinterpret_cast<float*>(g.out) + static_cast<int64_t>(row0) * g.ldo + col;
#pragma unroll 4
            for (int rr = 0; rr < 32; ++rr)
              if (row0 + rr < g.M && col < g.N)
                o[static_cast<int64_t>(rr) * g.ldo] =
                    *reinterpret_cast<const float*>(buf + rr * 128 + ((((lane >> 2) ^ (rr & 7))) << 4) + (lane & 3) * 4);
            __syncwarp();  // the staging buffer is rewritten by the next chunk
            continue;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (EPI == EPI_BIAS_RESID_F32)
              tma_reduce_add_2d(&tmC, buf, n_blk * BN + c, m_blk * BM + quad * 32);
            else
              tma_store_2d(&tmC, buf, n_blk * BN + c, m_blk * BM + quad * 32);
            bulk_commit();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else if (g.splits == 1) {
#pragma unroll 1
        for (int c = cbase; c < cbase + C::COLS_PER_WARP; c += 32) {
          uint32_t u[32];
          tmem_ld32(tmem_base + ((quad * 32) << 16) + acc * BN + c, u);
          tmem_wait_ld();
          if (g.acc16) acc16_widen(u);
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(u[i]);
          epilogue_chunk<EPI>(v, g, row, n_blk * BN + c, has_bias ? sbias + (c - cbase) : nullptr);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
      } else {
        // partial tile -> workspace (row-contiguous, 16B stores), then release TMEM
        float* wrow = g.ws + (static_cast<int64_t>(unit) * BM + r) * BN;
#pragma unroll 1
        for (int c = cbase; c < cbase + C::COLS_PER_WARP; c += 32) {
          uint32_t u[32];
          tmem_ld32(tmem_base + ((quad * 32) << 16) + acc * BN + c, u);
          tmem_wait_ld();
          if (g.acc16) acc16_widen(u);
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            __stcg(reinterpret_cast<float4*>(wrow + c + i),
                   make_float4(__uint_as_float(u[i]), __uint_as_float(u[i + 1]),
                               __uint_as_float(u[i + 2]), __uint_as_float(u[i + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        __threadfence();
        named_bar_sync(1, 32 * C::EPI_WARPS);
        if (tid == 0) {
          const int prev = atomicAdd(&g.tickets[tile], 1);
          const int last = prev == g.splits - 1;
          if (last) g.tickets[tile] = 0;  // ready for the next launch
          *last_flag = last;
        }
        named_bar_sync(1, 32 * C::EPI_WARPS);
        const int last = *last_flag;
        named_bar_sync(1, 32 * C::EPI_WARPS);  // flag consumed before the next unit overwrites it
        if (last) {
          __threadfence();
          const float* base = g.ws + (static_cast<int64_t>(tile) * g.splits * BM + r) * BN;
#pragma unroll 1
          for (int c = cbase; c < cbase + C::COLS_PER_WARP; c += 32) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.0f;
#pragma unroll 1
            for (int s0 = 0; s0 < g.splits; s0 += 2) {  // fixed split order: deterministic sum
              float4 p[2][8];
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const int s = s0 + j < g.splits ? s0 + j : s0;
                const float4* src = reinterpret_cast<const float4*>(base + static_cast<int64_t>(s) * BM * BN + c);
#pragma unroll
                for (int i = 0; i < 8; ++i) p[j][i] = __ldcg(src + i);
              }
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                if (s0 + j >= g.splits) break;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  v[4 * i] = __fadd_rn(v[4 * i], p[j][i].x);
                  v[4 * i + 1] = __fadd_rn(v[4 * i + 1], p[j][i].y);
                  v[4 * i + 2] = __fadd_rn(v[4 * i + 2], p[j][i].z);
                  v[4 * i + 3] = __fadd_rn(v[4 * i + 3], p[j][i].w);
                }
              }
            }
            epilogue_chunk<EPI>(v, g, row, n_blk * BN + c, has_bias ? sbias + (c - cbase) : nullptr);
          }
        }
      }
    }
    if (lane == 0) bulk_wait<0>();  // TMA stores complete before the CTA retires
    __syncwarp();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}


// ---------------------------------------------------------------------------
// Cluster split-K (small M).  grid = tiles * splits, cluster = (splits, 1, 1):
// the CTAs of one cluster own the k-slices of one output tile.  Each writes its
// fp32 partial tile to its own shared memory; after a cluster barrier every CTA
// reduces 1/splits of the tile's rows across all peers through DSMEM (fixed
// split order -> deterministic) and applies the epilogue.  No global partials,
// no atomics, the reduction is spread over all CTAs of the cluster.
// ---------------------------------------------------------------------------
template <int BN>
struct CCfg {
  static constexpr int STAGES = 4;
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int PSTRIDE = BN + 4;  // partial row stride (floats), skews banks
  static constexpr uint32_t PART_BYTES = BM * PSTRIDE * 4;
  static constexpr uint32_t DATA = STAGES * STAGE_BYTES > PART_BYTES ? STAGES * STAGE_BYTES : PART_BYTES;
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr size_t SMEM = 1024 + DATA + 256;
  static constexpr int THREADS = 192;
};

template <int EPI>
__device__ __forceinline__ void epilogue_vec4(float4 a, const GemmArgs& g, int row, int col) {
  if (row >= g.M || col >= g.N) return;
  float v[4] = {a.x, a.y, a.z, a.w};
  const bool full = col + 4 <= g.N;
  float bb[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) bb[i] = (g.bias != nullptr && col + i < g.N) ? __ldg(g.bias + col + i) : 0.0f;
#pragma unroll
  for (int i = 0; i < 4; i += 2)
    h2_unpack(epilogue_pair<EPI>(v[i], v[i + 1], bb[i], bb[i + 1]), v[i], v[i + 1]);
  if (EPI == EPI_BIAS_RESID_F32) {
    float* o = reinterpret_cast<float*>(g.out) + static_cast<int64_t>(row) * g.ldo + col;
    if (full && (g.ldo % 4) == 0) {
      float4 x = *reinterpret_cast<float4*>(o);
      x.x = __fadd_rn(x.x, v[0]);
      x.y = __fadd_rn(x.y, v[1]);
      x.z = __fadd_rn(x.z, v[2]);
      x.w = __fadd_rn(x.w, v[3]);
      *reinterpret_cast<float4*>(o) = x;
    } else {
      for (int i = 0; i < 4 && col + i < g.N; ++i) o[i] = __fadd_rn(o[i], v[i]);
    }
  } else {
    __half* o = reinterpret_cast<__half*>(g.out) + static_cast<int64_t>(row) * g.ldo + col;
    if (full && (g.ldo % 4) == 0) {
      __half2 h01 = __floats2half2_rn(v[0], v[1]), h23 = __floats2half2_rn(v[2], v[3]);
      *reinterpret_cast<uint2*>(o) = make_uint2(*reinterpret_cast<uint32_t*>(&h01), *reinterpret_cast<uint32_t*>(&h23));
    } else {
      for (int i = 0; i < 4 && col + i < g.N; ++i) o[i] = __float2half_rn(v[i]);
    }
  }
}

// full-width quad with the bias and residual already in registers
template <int EPI>
__device__ __forceinline__ void epilogue_vec4_fast(float4 a, float4 b, float4 x, const GemmArgs& g, int row,
                                                   int col) {
  float v[4] = {a.x, a.y, a.z, a.w};
  const float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
  for (int i = 0; i < 4; i += 2)
    h2_unpack(epilogue_pair<EPI>(v[i], v[i + 1], bb[i], bb[i + 1]), v[i], v[i + 1]);
  if (EPI == EPI_BIAS_RESID_F32) {
    float* o = reinterpret_cast<float*>(g.out) + static_cast<int64_t>(row) * g.ldo + col;
    *reinterpret_cast<float4*>(o) =
        make_float4(__fadd_rn(x.x, v[0]), __fadd_rn(x.y, v[1]), __fadd_rn(x.z, v[2]), __fadd_rn(x.w, v[3]));
  } else {
    __half* o = reinterpret_cast<__half*>(g.out) + static_cast<int64_t>(row) * g.ldo + col;
    __half2 h01 = __floats2half2_rn(v[0], v[1]), h23 = __floats2half2_rn(v[2], v[3]);
    if ((g.ldo % 4) == 0)
      *reinterpret_cast<uint2*>(o) = make_uint2(*reinterpret_cast<uint32_t*>(&h01), *reinterpret_cast<uint32_t*>(&h23));
    else {
      o[0] = __low2half(h01);
      o[1] = __high2half(h01);
      o[2] = __low2half(h23);
      o[3] = __high2half(h23);
    }
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(CCfg<BN>::THREADS, 1)
    gemm_splitk_cluster_kernel(const __grid_constant__ CUtensorMap tmA,
                               const __grid_constant__ CUtensorMap tmB, const GemmArgs g) {
  using C = CCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  float* part = reinterpret_cast<float*>(smem);  // reuses the stage buffers after the MMAs
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::DATA);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const uint32_t warp = warp_id(), lane = lane_id();
  long long* dbg = g.dbg ? g.dbg + static_cast<int64_t>(blockIdx.x) * 8 : nullptr;
  if (dbg && threadIdx.x == 0) dbg[0] = globaltimer();
  const int split = static_cast<int>(cluster_ctarank());
  const int tile = blockIdx.x / g.splits;
  const int kb0 = split * g.kb_per_split;
  const int kb1 = min(g.num_k_blocks, kb0 + g.kb_per_split);
  int m_blk, n_blk;
      tile_coords(g, tile, m_blk, n_blk);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;
  if (dbg && threadIdx.x == 0) dbg[1] = globaltimer();

  if (warp == 0) {
    if (lane == 0) {
      const int pre = min(C::STAGES, kb1 - kb0);
      for (int i = 0; i < pre; ++i) {  // weights first: independent of the upstream kernel
        mbar_expect_tx(&full[i], C::STAGE_BYTES);
        tma_load_2d(sB + i * C::B_BYTES, &tmB, &full[i], (kb0 + i) * BK, n_blk * BN);
      }
      pdl_wait();
      if (dbg) dbg[2] = globaltimer();
      uint32_t stage = 0, phase = 0;
      for (int kb = kb0; kb < kb1; ++kb) {
        if (kb - kb0 < pre) {
          tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
        } else {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
          tma_load_2d(sB + stage * C::B_BYTES, &tmB, &full[stage], kb * BK, n_blk * BN);
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    const uint32_t idesc = idesc_f16_f32(BM, BN, 0, 0) & (g.acc16 ? ~(3u << 4) : ~0u);
    uint32_t stage = 0, phase = 0;
    for (int kb = kb0; kb < kb1; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sA + stage * C::A_BYTES);
        const uint32_t b0 = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          umma_f16_ss(tmem_base, sw128_desc(a0 + k * 32, 0, 1024), sw128_desc(b0 + k * 32, 0, 1024), idesc,
                      (kb > kb0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[stage]);
      }
      __syncwarp();
      if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
    }
    if (lane == 0) umma_commit(tfull);
    __syncwarp();
  } else {
    // accumulator -> own shared memory (row r, padded stride)
    const uint32_t quad = warp & 3;
    const int r = quad * 32 + lane;
    mbar_wait(tfull, 0);
    tc_fence_after();
    if (dbg && warp == 2 && lane == 0) dbg[3] = globaltimer();
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t u[32];
      tmem_ld32(tmem_base + ((quad * 32) << 16) + c, u);
      tmem_wait_ld();
      if (g.acc16) acc16_widen(u);
      float* dst = part + r * C::PSTRIDE + c;
#pragma unroll
      for (int i = 0; i < 32; i += 4)
        *reinterpret_cast<float4*>(dst + i) = make_float4(__uint_as_float(u[i]), __uint_as_float(u[i + 1]),
                                                          __uint_as_float(u[i + 2]), __uint_as_float(u[i + 3]));
    }
    tc_fence_before();
  }
  // Hoist this thread's global reads (bias quad, residual x) above the cluster
  // barrier: their latency overlaps the wait instead of serialising the reduce.
  constexpr int C4 = BN / 4;
  constexpr int MAXIT = 8;  // (rows_per * C4) / 128 <= 8 for splits >= 2 at BN 64, >= 4 at BN 128
  const int tid = static_cast<int>(threadIdx.x) - 64;
  const int rows_per = (BM + g.splits - 1) / g.splits;
  const int r0 = split * rows_per, r1 = min(BM, r0 + rows_per);
  const int c4 = (tid >= 0 ? tid : 0) % C4;  // each thread's column quad is fixed (128 % C4 == 0)
  const int col = n_blk * BN + c4 * 4;
  const int nit = tid >= 0 ? ((r1 - r0) * C4 - tid + 127) / 128 : 0;
  float4 bias4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 xres[MAXIT];
  if (warp >= 2) {
    if (EPI != EPI_F16 && g.bias != nullptr && col + 4 <= g.N) bias4 = __ldg(reinterpret_cast<const float4*>(g.bias + col));
    if (EPI == EPI_BIAS_RESID_F32) {
#pragma unroll
      for (int it = 0; it < MAXIT; ++it) {
        const int rr = r0 + (tid + it * 128) / C4;
        const int row = m_blk * BM + rr;
        xres[it] = (it < nit && row < g.M && col + 4 <= g.N && (g.ldo % 4) == 0)
                       ? *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(g.out) +
                                                          static_cast<int64_t>(row) * g.ldo + col)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  if (dbg && threadIdx.x == 64) dbg[4] = globaltimer();
  cluster_sync_all();  // every CTA's partial is complete and visible cluster-wide
  if (dbg && threadIdx.x == 64) dbg[5] = globaltimer();
  if (warp >= 2) {
    const uint32_t base = smem_u32(part);
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      if (it >= nit) break;
      const int e = tid + it * 128;
      const int rr = r0 + e / C4;
      const uint32_t off = static_cast<uint32_t>((rr * C::PSTRIDE + c4 * 4) * 4);
      float4 p[8];
#pragma unroll
      for (int s = 0; s < 8; ++s)  // all peer loads in flight before the (ordered) sum
        if (s < g.splits) p[s] = ld_dsmem_f4(mapa_shared(base + off, static_cast<uint32_t>(s)));
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int s = 0; s < 8; ++s) {  // fixed order: deterministic
        if (s < g.splits) {
          acc.x = __fadd_rn(acc.x, p[s].x);
          acc.y = __fadd_rn(acc.y, p[s].y);
          acc.z = __fadd_rn(acc.z, p[s].z);
          acc.w = __fadd_rn(acc.w, p[s].w);
        }
      }
      const int row = m_blk * BM + rr;
      if (col + 4 <= g.N && row < g.M && (EPI != EPI_BIAS_RESID_F32 || (g.ldo % 4) == 0)) {
        epilogue_vec4_fast<EPI>(acc, bias4, xres[it], g, row, col);
      } else {
        epilogue_vec4<EPI>(acc, g, row, col);
      }
    }
    for (int it = MAXIT; it < nit; ++it) {  // tall slices (few splits, wide tiles): no prefetch
      const int rr = r0 + (tid + it * 128) / C4;
      const uint32_t off = static_cast<uint32_t>((rr * C::PSTRIDE + c4 * 4) * 4);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s = 0; s < g.splits; ++s) {
        const float4 p = ld_dsmem_f4(mapa_shared(base + off, static_cast<uint32_t>(s)));
        acc.x = __fadd_rn(acc.x, p.x);
        acc.y = __fadd_rn(acc.y, p.y);
        acc.z = __fadd_rn(acc.z, p.z);
        acc.w = __fadd_rn(acc.w, p.w);
      }
      epilogue_vec4<EPI>(acc, g, m_blk * BM + rr, col);
    }
  }
  if (dbg && threadIdx.x == 64) dbg[6] = globaltimer();
  cluster_sync_all();  // peers are done reading this CTA's shared memory
  if (dbg && threadIdx.x == 64) dbg[7] = globaltimer();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int BN, int EPI>
void configure_cluster_one() {
  auto k = gemm_splitk_cluster_kernel<BN, EPI>;
  PRLAB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(CCfg<BN>::SMEM)));
  PRLAB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

template <int BN>
void configure_cluster_bn() {
  configure_cluster_one<BN, EPI_BIAS_F16>();
  configure_cluster_one<BN, EPI_BIAS_GELU_F16>();
  configure_cluster_one<BN, EPI_BIAS_RESID_F32>();
  configure_cluster_one<BN, EPI_F16>();
}

template <int BN, int EPI>
void launch_cluster_one(const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(CCfg<BN>::THREADS);
  cfg.dynamicSmemBytes = CCfg<BN>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.splits;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  PRLAB_CUDA(cudaLaunchKernelEx(&cfg, gemm_splitk_cluster_kernel<BN, EPI>, p.tmA, p.tmB, g));
}

template <int BN>
void launch_cluster_bn(const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
  switch (p.epi) {
    case EPI_BIAS_F16: launch_cluster_one<BN, EPI_BIAS_F16>(p, g, st); break;
    case EPI_BIAS_GELU_F16: launch_cluster_one<BN, EPI_BIAS_GELU_F16>(p, g, st); break;
    case EPI_BIAS_RESID_F32: launch_cluster_one<BN, EPI_BIAS_RESID_F32>(p, g, st); break;
    case EPI_F16: launch_cluster_one<BN, EPI_F16>(p, g, st); break;
    default: throw std::invalid_argument("unknown gemm epilogue");
  }
}


// ---------------------------------------------------------------------------
// CTA-pair GEMM (large M): a cluster of 2 CTAs computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 (M = 256).  CTA r loads its own 128 rows of A and
// half of the B tile (BN/2 weight rows) -- per CTA and k-block that is 16 KB
// + BN*64 B instead of 16 KB + BN*128 B, which cuts the L2->SM traffic per
// FLOP by a third at BN = 256.  Only the leader (rank 0) issues MMAs; its
// commits are multicast to both CTAs' barriers; both CTAs run their own
// epilogue on their own TMEM rows (TMA-store / reduce-add as in gemm_tc_kernel).
// Barriers: full (leader; 2 arrivals + both CTAs' transaction bytes), empty and
// tfull (per CTA, multicast commits), tempty (leader; all epilogue warps of both).
// ---------------------------------------------------------------------------
template <int BN, int EPI = 0>
struct Cfg2 {
  // the erf-heavy GELU epilogue gets 4 warps per TMEM lane quadrant (one staging
  // buffer each); the others 2 warps per quadrant with double-buffered staging
  static constexpr int EPI_WARPS = (EPI == EPI_BIAS_GELU_F16 && BN == 256) ? 16 : 8;
  static constexpr int NBUF = EPI_WARPS == 16 ? 1 : 2;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr int COLS_PER_WARP = BN / (EPI_WARPS / 4);
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = (BN / 2) * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr uint32_t EPI_BYTES = EPI_WARPS * NBUF * 4096;
  static constexpr uint32_t BIAS_BYTES = EPI_WARPS * COLS_PER_WARP * 4;
  static constexpr uint32_t SMEM_BUDGET = 227 * 1024 - 1024 - 256 - EPI_BYTES - BIAS_BYTES;
  static constexpr int STAGES = SMEM_BUDGET / STAGE_BYTES > 6 ? 6 : SMEM_BUDGET / STAGE_BYTES;
  static constexpr uint32_t EPI_OFF = STAGES * STAGE_BYTES;
  static constexpr uint32_t BAR_OFF = EPI_OFF + EPI_BYTES;
  static constexpr uint32_t BIAS_OFF = BAR_OFF + 256;
  static constexpr size_t SMEM = 1024 + BIAS_OFF + BIAS_BYTES;
};

// MC: clusters of 4 = two CTA pairs on adjacent m-pairs of the same n-block; each CTA
// loads a quarter of the weight tile and multicasts it to the matching CTA of the other
// pair, so the per-CTA weight traffic from L2 halves (the main loop is L2-feed bound:
// scripts/gemm_probe.py).  Stage release (empty) then needs both pairs' MMA commits.
template <int BN, int EPI, bool MC = false>
__global__ void __launch_bounds__(Cfg2<BN, EPI>::THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmC, const GemmArgs g) {
  using C = Cfg2<BN, EPI>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1;           // rank inside the pair
  const uint32_t pp = MC ? (crank >> 1) : 0; // pair inside the cluster
  const bool leader = rank == 0;
  // work unit = (pair of m-blocks, n-block) -- with MC (quad of m-blocks, n-block), the
  // cluster's two pairs taking the two m-pairs; units stride by the number of clusters
  const int csize = MC ? 4 : 2;
  const int pair = blockIdx.x / csize, npairs = gridDim.x / csize;
  const int m_pairs = (g.num_m_blocks + 1) / 2;
  const int m_units = MC ? (m_pairs + 1) / 2 : m_pairs;
  const int total_units = m_units * g.num_n_blocks;
  const uint16_t pair_mask = static_cast<uint16_t>(3u << (2 * pp));
  const uint16_t all_mask = MC ? 0xF : 3;
  const uint16_t mc_mask = static_cast<uint16_t>((1u << rank) | (1u << (2 + rank)));

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (g.tma_store && EPI != EPI_ROWSTAT) tma_prefetch_desc(&tmC);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], MC ? 2 : 1);  // MC: both pairs' MMAs read this stage's weights
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * C::EPI_WARPS);
    }
    fence_barrier_init();
  }
  cluster_sync_all();  // barriers of both CTAs initialised before any cross-CTA traffic
  if (warp == 1) {
    tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;

  auto coords = [&](int unit, int& mp, int& n_blk) {
    // bands of group_m/2 m-pairs (group_m/4 m-quads); n-blocks advance slowest inside a band
    const int GROUP = MC ? max(1, g.group_m >> 2) : (g.group_m >> 1);
    const int band = unit / (GROUP * g.num_n_blocks);
    const int m0 = band * GROUP;
    const int rows = min(GROUP, m_units - m0);
    const int local = unit - band * GROUP * g.num_n_blocks;
    n_blk = local / rows;
    mp = m0 + local % rows;
    if (MC) mp = 2 * mp + static_cast<int>(pp);
  };
  // this CTA's weight rows: its half of the pair's tile (MC: a quarter, multicast)
  auto load_b = [&](int stage, int kb, int n_blk) {
    if (MC)
      tma_load_2d_pair_mc(sB + stage * C::B_BYTES + pp * (C::B_BYTES / 2), &tmB, &full[stage], kb * BK,
                          n_blk * BN + rank * (BN / 2) + pp * (BN / 4), mc_mask);
    else
      tma_load_2d_pair(sB + stage * C::B_BYTES, &tmB, &full[stage], kb * BK, n_blk * BN + rank * (BN / 2));
  };

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (lane == 0) {
      int pre = 0;
      if (pair < total_units) {
        int mp, n_blk;
        coords(pair, mp, n_blk);
        pre = min(C::STAGES, g.num_k_blocks);
        for (int i = 0; i < pre; ++i) {  // weight halves first (independent of the upstream kernel)
          if (leader) mbar_expect_tx(&full[i], 2 * C::STAGE_BYTES);
          load_b(i, i, n_blk);
        }
      }
      pdl_wait();
      uint32_t stage = 0, phase = 0;
      bool first = true;
      for (int unit = pair; unit < total_units; unit += npairs) {
        int mp, n_blk;
        coords(unit, mp, n_blk);
        const int m_blk = 2 * mp + static_cast<int>(rank);
        for (int kb = 0; kb < g.num_k_blocks; ++kb) {
          if (first && kb < pre) {
            tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
          } else if (g.dbg_noload) {  // debug probe: 3 = no operand loads, 1 = no A, 2 = no B
            mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t bytes = ((g.dbg_noload & 1) ? 0u : C::A_BYTES) + ((g.dbg_noload & 2) ? 0u : C::B_BYTES);
            if (leader) {
              if (bytes) mbar_expect_tx(&full[stage], 2 * bytes);
              else mbar_arrive(&full[stage]);
            }
            if (!(g.dbg_noload & 1)) tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
            if (!(g.dbg_noload & 2)) load_b(stage, kb, n_blk);
          } else {
            mbar_wait(&empty[stage], phase ^ 1);
            if (leader) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m_blk * BM);
            load_b(stage, kb, n_blk);
          }
          if (!leader) mbar_arrive_cluster(to_leader(smem_u32(&full[stage])));
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        first = false;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only) ----------------
    if (leader) {
      const uint32_t idesc = idesc_f16_f32(256, BN, 0, 0) & (g.acc16 ? ~(3u << 4) : ~0u);
      uint32_t stage = 0, phase = 0, t = 0;
      for (int unit = pair; unit < total_units; unit += npairs, ++t) {
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
              umma_f16_ss_pair(d_tmem, sw128_desc(a0 + k * 32, 0, 1024), sw128_desc(b0 + k * 32, 0, 1024), idesc,
                               (kb > 0 || k > 0) ? 1u : 0u);
            umma_commit_pair(&empty[stage], all_mask);
          }
          __syncwarp();
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) umma_commit_pair(&tfull[acc], pair_mask);
        __syncwarp();
      }
      // the peer's last tempty arrivals must land before the leader retires
      if (t > 0) mbar_wait(&tempty[(t - 1) & 1], ((t - 1) >> 1) & 1);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (both CTAs, own TMEM rows) ----------------
    const uint32_t quad = warp & 3;
    const int cbase = ((warp - 2) >> 2) * C::COLS_PER_WARP;
    float* sbias = reinterpret_cast<float*>(smem + C::BIAS_OFF) + (warp - 2) * C::COLS_PER_WARP;
    const uint32_t tempty_leader = to_leader(smem_u32(&tempty[0]));
    uint8_t* ebuf = smem + C::EPI_OFF + (warp - 2) * C::NBUF * 4096;
    constexpr bool F32OUT = epi_f32out(EPI);
    constexpr int SC = F32OUT ? 32 : 64;
    uint32_t t = 0, store_k = 0;
    for (int unit = pair; unit < total_units; unit += npairs, ++t) {
      int mp, n_blk;
      coords(unit, mp, n_blk);
      const int m_blk = 2 * mp + static_cast<int>(rank);
      const uint32_t acc = t & 1, acc_phase = (t >> 1) & 1;
      const bool has_bias = epi_bias(EPI) && g.bias != nullptr;
      if (has_bias) {
        __syncwarp();
        for (int c = lane; c < C::COLS_PER_WARP; c += 32) {
          const int col = n_blk * BN + cbase + c;
          sbias[c] = col < g.N ? __ldg(g.bias + col) : 0.0f;
        }
        __syncwarp();
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if constexpr (EPI == EPI_ROWSTAT) {
        // Fused log-softmax statistics of this thread's row over the warp's columns
        // (logits v = round16(acc), exactly the values EPI_F16 would store): running max
        // with a rescaled fp32 sum of 2^((v - max) log2 e) (ex2.approx, packed fp32x2
        // subtract/scale), the first column of the maximum (strict >, ascending columns:
        // the chunk is rescanned only when its max is a new record), the target's value.
        // Non-finite rows: a NaN anywhere reaches the sum, +inf the max.  ~8 issue slots per
        // element (the per-element argmax / NaN / target tests cost ~20).
        const int row = m_blk * BM + static_cast<int>(quad) * 32 + static_cast<int>(lane);
        const int32_t tgt = (g.targets != nullptr && row < g.M) ? g.targets[row] : -1;
        const float ninf = __int_as_float(0xff800000);
        constexpr float L2E = 1.4426950408889634f;
        constexpr int NCH = C::COLS_PER_WARP / 32;
        float mx = ninf, sum = 0.0f;
        int bidx = 0x7fffffff;
        bool nan_seen = false;
        const uint32_t tbase = tmem_base + ((quad * 32) << 16) + acc * BN;
        auto load_chunk = [&](int k, float (&v)[32]) {
          uint32_t u[32];
          tmem_ld32(tbase + cbase + k * 32, u);
          tmem_wait_ld();
          if (g.acc16) acc16_widen(u);
#pragma unroll
          for (int q = 0; q < 16; ++q)
            h2_unpack(h2_pack_rn(__uint_as_float(u[2 * q]), __uint_as_float(u[2 * q + 1])), v[2 * q], v[2 * q + 1]);
          const int col0 = n_blk * BN + cbase + k * 32;
          if (col0 + 32 > g.N) {  // (warp-uniform: the vocabulary tail)
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (col0 + q >= g.N) v[q] = ninf;
          }
        };
#pragma unroll
        for (int k = 0; k < NCH; ++k) {
          float v[32];
          load_chunk(k, v);
          const int col0 = n_blk * BN + cbase + k * 32;
          float m4[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
          for (int q = 4; q < 32; ++q) m4[q & 3] = fmaxf(m4[q & 3], v[q]);
          const float cm = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
          const unsigned kt = static_cast<unsigned>(tgt - col0);
          if (kt < 32u) {
            float tv = v[0];
#pragma unroll
            for (int q = 1; q < 32; ++q) tv = kt == static_cast<unsigned>(q) ? v[q] : tv;
            g.tval[row] = tv;
          }
          if (cm > mx) {
            int jj = 31;
#pragma unroll
            for (int q = 31; q >= 0; --q) jj = v[q] == cm ? q : jj;
            bidx = col0 + jj;
            sum = mx == ninf ? 0.0f : sum * ex2_approx(__fmul_rn(__fsub_rn(mx, cm), L2E));
            mx = cm;
          }
          if (mx != ninf) {
            const uint64_t nm = f2_pack(-mx, -mx), l2 = f2_pack(L2E, L2E);
            float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              float d0, d1;
              f2_unpack(f2_mul(f2_add(f2_pack(v[2 * q], v[2 * q + 1]), nm), l2), d0, d1);
              s4[(2 * q) & 3] += ex2_approx(d0);
              s4[(2 * q + 1) & 3] += ex2_approx(d1);
            }
            sum += (s4[0] + s4[1]) + (s4[2] + s4[3]);
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) nan_seen |= v[q] != v[q];
          }
        }
        bool bad = nan_seen || sum != sum || mx == __int_as_float(0x7f800000);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
        // the two column groups of a TMEM lane quadrant (warps q and q + 4) merge through
        // shared memory (double-buffered by tile parity: one barrier per tile), so the head
        // writes one slot per n-block and row: half the bytes for the fold kernel
        static_assert(C::EPI_WARPS == 8, "row statistics: two column groups per quadrant");
        const int grp = (static_cast<int>(warp) - 2) >> 2;
        float4* xch = reinterpret_cast<float4*>(smem + C::EPI_OFF) + ((t & 1) * 4 + quad) * 32;
        if (grp == 1) xch[lane] = make_float4(mx, sum, __int_as_float(bidx), bad ? 1.0f : 0.0f);
        named_bar_sync(8 + quad, 64);
        if (grp == 1) continue;
        const float4 o = xch[lane];
        if (o.x > mx) {  // (ties keep group 0: its columns come first)
          sum = (mx == ninf ? 0.0f : sum * ex2_approx(__fmul_rn(__fsub_rn(mx, o.x), L2E))) + o.y;
          mx = o.x;
          bidx = __float_as_int(o.z);
        } else if (o.x != ninf) {
          sum += o.y * ex2_approx(__fmul_rn(__fsub_rn(o.x, mx), L2E));
        }
        bad |= o.w != 0.0f || sum != sum;
        if (row < g.M)
          reinterpret_cast<float4*>(g.out)[static_cast<int64_t>(n_blk) * g.M + row] =
              make_float4(mx, sum, __int_as_float(bidx), bad ? 1.0f : 0.0f);
        continue;
      }
#pragma unroll 1
      for (int c = cbase; c < cbase + C::COLS_PER_WARP; c += SC, ++store_k) {
        uint8_t* buf = ebuf + (C::NBUF == 2 ? (store_k & 1) * 4096 : 0);
        if (lane == 0) {
          if (C::NBUF == 2)
            bulk_wait_read<1>();
          else
            bulk_wait_read<0>();
        }
        __syncwarp();
        uint8_t* rowp = buf + lane * 128;
#pragma unroll
        for (int h = 0; h < SC; h += 32) {
          uint32_t u[32];
          tmem_ld32(tmem_base + ((quad * 32) << 16) + acc * BN + c + h, u);
          tmem_wait_ld();
          if (g.acc16) acc16_widen(u);
          const float* sb = has_bias ? sbias + (c - cbase) + h : nullptr;
          if (F32OUT) {
            float v[32];
            epilogue_values<EPI>(u, sb, v);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(rowp + ((j ^ (lane & 7)) * 16)) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
            uint32_t pk[16];
            epilogue_packed<EPI>(u, sb, pk);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(rowp + ((((h >> 3) + j) ^ (lane & 7)) * 16)) =
                  make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (EPI == EPI_BIAS_RESID_F32)
            tma_reduce_add_2d(&tmC, buf, n_blk * BN + c, m_blk * BM + quad * 32);
          else
            tma_store_2d(&tmC, buf, n_blk * BN + c, m_blk * BM + quad * 32);
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  cluster_sync_all();  // all MMAs / TMEM reads of both CTAs done
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
  }
}

template <int BN, int EPI>
void configure_pair_one() {
  for (auto k : {gemm_tc2_kernel<BN, EPI, false>, gemm_tc2_kernel<BN, EPI, true>}) {
    PRLAB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(Cfg2<BN, EPI>::SMEM)));
  }
}

template <int BN>
void configure_pair_bn() {
  configure_pair_one<BN, EPI_BIAS_F16>();
  configure_pair_one<BN, EPI_BIAS_GELU_F16>();
  configure_pair_one<BN, EPI_BIAS_RESID_F32>();
  configure_pair_one<BN, EPI_F16>();
  configure_pair_one<BN, EPI_ROWSTAT>();
  configure_pair_one<BN, EPI_F16_F32>();
}

template <int BN, int EPI>
void launch_pair_one(const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(Cfg2<BN, EPI>::THREADS);
  cfg.dynamicSmemBytes = Cfg2<BN, EPI>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.pair_mc ? 4 : 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (p.pair_mc)
    PRLAB_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc2_kernel<BN, EPI, true>, p.tmA, p.tmB, p.tmC, g));
  else
    PRLAB_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc2_kernel<BN, EPI, false>, p.tmA, p.tmB, p.tmC, g));
}

template <int BN>
void launch_pair_bn(const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
  switch (p.epi) {
    case EPI_BIAS_F16: launch_pair_one<BN, EPI_BIAS_F16>(p, g, st); break;
    case EPI_BIAS_GELU_F16: launch_pair_one<BN, EPI_BIAS_GELU_F16>(p, g, st); break;
    case EPI_BIAS_RESID_F32: launch_pair_one<BN, EPI_BIAS_RESID_F32>(p, g, st); break;
    case EPI_F16: launch_pair_one<BN, EPI_F16>(p, g, st); break;
    case EPI_ROWSTAT: launch_pair_one<BN, EPI_ROWSTAT>(p, g, st); break;
    case EPI_F16_F32: launch_pair_one<BN, EPI_F16_F32>(p, g, st); break;
    default: throw std::invalid_argument("unknown gemm epilogue");
  }
}

template <int BN, bool LEAN, int EPI>
void configure_one() {
  PRLAB_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, LEAN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(Cfg<BN, LEAN, EPI>::SMEM)));
}

template <int BN, bool LEAN>
void configure_bn() {
  configure_one<BN, LEAN, EPI_BIAS_F16>();
  configure_one<BN, LEAN, EPI_BIAS_GELU_F16>();
  configure_one<BN, LEAN, EPI_BIAS_RESID_F32>();
  configure_one<BN, LEAN, EPI_F16>();
  configure_one<BN, LEAN, EPI_F16_F32>();
}

template <int BN, bool LEAN, int EPI>
void launch_one(const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
  using C = Cfg<BN, LEAN, EPI>;
  launch_pdl(gemm_tc_kernel<BN, LEAN, EPI>, dim3(p.grid), dim3(C::THREADS), C::SMEM, st, p.tmA, p.tmB, p.tmC, g);
}

template <int BN, bool LEAN>
void launch_bn(const GemmPlan& p, const GemmArgs& g, cudaStream_t st) {
  switch (p.epi) {
    case EPI_BIAS_F16: launch_one<BN, LEAN, EPI_BIAS_F16>(p, g, st); break;
    case EPI_BIAS_GELU_F16: launch_one<BN, LEAN, EPI_BIAS_GELU_F16>(p, g, st); break;
    case EPI_BIAS_RESID_F32: launch_one<BN, LEAN, EPI_BIAS_RESID_F32>(p, g, st); break;
    case EPI_F16: launch_one<BN, LEAN, EPI_F16>(p, g, st); break;
    case EPI_F16_F32: launch_one<BN, LEAN, EPI_F16_F32>(p, g, st); break;
    default: throw std::invalid_argument("unknown gemm epilogue");
  }
}

}  // namespace

long long*& debug_stamps() {
  static long long* p = nullptr;
  return p;
}

SplitScratch& global_split_scratch() {
  static SplitScratch s;
  if (!s.ws) {
    s.ws_floats = static_cast<size_t>(2 * num_sms()) * BM * 128;
    PRLAB_CUDA(cudaMalloc(&s.ws, s.ws_floats * sizeof(float)));
    s.n_tickets = 4096;
    PRLAB_CUDA(cudaMalloc(&s.tickets, s.n_tickets * sizeof(int)));
    PRLAB_CUDA(cudaMemset(s.tickets, 0, s.n_tickets * sizeof(int)));
  }
  return s;
}

// co-resident 4-CTA clusters of the ~200 KB pair kernel (GPC packing leaves SMs idle)
int max_active_clusters4() {
  static int n_dev[64] = {};
  int& n = n_dev[current_device() & 63];
  if (n == 0) {
    configure_gemm_tc();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4 * 64);
    cfg.blockDim = dim3(Cfg2<256, EPI_BIAS_F16>::THREADS);
    cfg.dynamicSmemBytes = Cfg2<256, EPI_BIAS_F16>::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 4;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PRLAB_CUDA(cudaOccupancyMaxActiveClusters(&n, gemm_tc2_kernel<256, EPI_BIAS_F16, true>, &cfg));
    n = std::max(n, 1);
  }
  return n;
}

GemmPlan plan_gemm_tc(const void* A, int64_t lda, const void* Wt, int64_t ldw, const float* bias,
                      void* out, int64_t ldo, int M, int N, int K, int epi, const SplitScratch* scratch,
                      int force_bn, int force_splits, int force_lean) {
  if (M < 1 || N < 1 || K < 1) throw std::invalid_argument("tc gemm: empty extent");
  if (K % 8 != 0 || lda % 8 != 0 || ldw % 8 != 0)
    throw std::invalid_argument("tc gemm: K and row pitches must be multiples of 8");
  GemmPlan p{};
  const int sms = num_sms();
  const int mb = (M + BM - 1) / BM;
  const int nkb = (K + BK - 1) / BK;
  // Widest N tile that still gives at least 0.6 of the SMs work; narrower tiles stream
  // the weights through more SMs when M is small (weight-bandwidth bound).  Measured over
  // the forward's shapes (M 128..4096 x QKV / Wo / FFN / heads, profiles/r02/bn_rule.jsonl):
  // one wave of 96-144 wide tiles beats two waves of half-width ones by 20-40 %.
  int bn = 256;
  while (bn > 64 && static_cast<int64_t>(mb) * ((N + bn - 1) / bn) * 5 < static_cast<int64_t>(sms) * 3) bn /= 2;
  if (force_bn) bn = force_bn;
  const int tiles = mb * ((N + bn - 1) / bn);
  // Split K while the grid is far below one wave (batch-1 latency shapes): the
  // cluster split-K kernel reduces partials through DSMEM (cluster <= 8 CTAs).
  int splits = 1;
  bool cluster = false;
  if (bn <= 128 && tiles * 2 <= sms && nkb > 1) {
    splits = std::min(std::min(nkb, 8), std::max(1, sms / tiles));
    cluster = splits > 1;
  }
  if (force_splits) {
    splits = std::min(std::abs(force_splits), nkb);
    cluster = force_splits > 0 && splits > 1;  // negative: the global-workspace split-K path
  }
  if (epi == EPI_F16_F32) cluster = false;  // (the cluster split-K kernel has no fp32-widening epilogue)
  if (splits > 1) {
    const int kps = (nkb + splits - 1) / splits;
    splits = (nkb + kps - 1) / kps;
    if (splits == 1) cluster = false;
  }
  if (!cluster && splits > 1 &&
      (!scratch || static_cast<size_t>(tiles) * splits * BM * bn > scratch->ws_floats || tiles > scratch->n_tickets))
    splits = 1;
  // lean pipelines when the whole grid fits in one wave: every CTA then runs a
  // single short unit and the next kernel's CTAs can share its SM (PDL overlap)
  p.lean = (tiles * splits <= sms);
  if (force_lean) p.lean = force_lean > 0;
  p.cluster = cluster;
  // CTA pairs (cta_group::2) once there are several waves of 256-row tiles
  p.pair = !cluster && splits == 1 && (bn == 256 || bn == 128) && mb >= 4 &&
           static_cast<int64_t>((mb + 1) / 2) * ((N + bn - 1) / bn) >= sms / 2 && !std::getenv("PRLAB_NO_PAIR");
  if (force_lean < -1) p.pair = false;  // tuning: -2 forces the 1-CTA kernel
  if (force_lean > 1) p.pair = (bn == 256 || bn == 128);  // tuning: 2 forces the pair kernel
  // Raster band: inside a band the n-blocks advance slowest, so the band's rows of A
  // are re-read from L2 once per n-block and each weight tile is fetched once per band.
  // When all of A fits comfortably in L2 (e.g. the LM head: A 25 MB, E 77 MB at C4)
  // one band covers every m-block and the weights stream from DRAM exactly once;
  // otherwise bands of 16 m-blocks (2048 rows).
  {
    const int64_t a_bytes = static_cast<int64_t>(M) * K * 2;
    const int64_t w_bytes = static_cast<int64_t>(N) * K * 2;
    int grp = 16;
    if (a_bytes <= (48ll << 20) && w_bytes > a_bytes) grp = mb;
    grp = std::max(2, (grp + 1) / 2 * 2);  // the pair kernel bands by m-pairs
    p.group_m = grp;
  }
  p.M = M;
  p.N = N;
  p.K = K;
  p.bn = bn;
  p.epi = epi;
  p.bias = bias;
  p.out = out;
  p.ldo = ldo;
  p.splits = splits;
  p.kb_per_split = (nkb + splits - 1) / splits;
  p.splits = (nkb + p.kb_per_split - 1) / p.kb_per_split;
  if (p.splits > 1 && !p.cluster) {
    if (!scratch || static_cast<size_t>(tiles) * p.splits * BM * bn > scratch->ws_floats ||
        tiles > scratch->n_tickets)
      throw std::invalid_argument("tc gemm: split-K workspace too small");
    p.ws = scratch->ws;
    p.tickets = scratch->tickets;
  }
  p.tmA = make_tmap_f16_2d(A, M, K, lda, BM, BK);
  // TMA-store epilogue when the output rows are 16-byte aligned (TMA clips the M/N tails)
  const bool f32out = epi_f32out(epi);
  const int64_t row_bytes = ldo * (f32out ? 4 : 2);
  p.tma_store = !std::getenv("PRLAB_NO_TMA_STORE") && (row_bytes % 16 == 0) &&
                (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  if (epi == EPI_ROWSTAT) {  // no output tile: the pair kernel writes row statistics
    if (!p.pair) throw std::invalid_argument("tc gemm: row statistics need the CTA-pair kernel");
    p.tma_store = true;
  } else if (p.tma_store)
    p.tmC = f32out ? make_tmap_f32_2d(out, M, N, ldo, 32, 32) : make_tmap_f16_2d(out, M, N, ldo, 32, 64);
  const int units = tiles * p.splits;
  p.grid = p.cluster ? units : (units < sms ? units : sms);
  if (p.pair) {
    if (!p.tma_store) p.pair = false;  // the pair kernel only has the TMA-store epilogue
  }
  if (p.pair) {
    // two pairs per cluster sharing the weight tile (multicast) once there are >= 2 m-pairs
    const int m_pairs = (mb + 1) / 2;
    // Off by default: 4-CTA clusters only tile 132 of the 148 SMs (33 co-resident
    // clusters, scripts/ubench/cluster_occ.cu), which costs more than the halved weight
    // traffic saves (profiles/r01/gemm_probe_mc.jsonl).  PRLAB_GEMM_MC=1 enables it.
    p.pair_mc = m_pairs >= 2 && std::getenv("PRLAB_GEMM_MC") != nullptr;
    if (p.pair_mc) {
      const int units = ((m_pairs + 1) / 2) * ((N + bn - 1) / bn);
      p.grid = 4 * std::min(units, max_active_clusters4());
      p.tmB = make_tmap_f16_2d(Wt, N, K, ldw, bn / 4, BK);
    } else {
      const int pair_units = m_pairs * ((N + bn - 1) / bn);
      p.grid = 2 * std::min(pair_units, sms / 2);
      p.tmB = make_tmap_f16_2d(Wt, N, K, ldw, bn / 2, BK);
    }
  } else {
    p.tmB = make_tmap_f16_2d(Wt, N, K, ldw, bn, BK);
  }
  return p;
}

void configure_gemm_tc() {
  static std::mutex mu;
  static uint64_t done = 0;
  once_per_device(mu, done, [] {
    configure_bn<256, false>();
    configure_bn<128, false>();
    configure_bn<64, false>();
    configure_bn<256, true>();
    configure_bn<128, true>();
    configure_bn<64, true>();
    configure_cluster_bn<64>();
    configure_cluster_bn<128>();
    configure_pair_bn<128>();
    configure_pair_bn<256>();
  });
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
  g.splits = p.splits;
  g.kb_per_split = p.kb_per_split;
  g.bias = p.bias;
  g.out = p.out;
  g.ldo = p.ldo;
  g.ws = p.ws;
  g.tickets = p.tickets;
  g.tma_store = p.tma_store ? 1 : 0;
  g.group_m = p.group_m;
  g.dbg_noload = std::getenv("PRLAB_DBG_GEMM_NOLOAD") ? std::atoi(std::getenv("PRLAB_DBG_GEMM_NOLOAD")) : 0;
  g.dbg = debug_stamps();
  g.targets = p.targets;
  g.tval = p.tval;
  g.acc16 = p.acc16 ? 1 : 0;
  if (p.pair) {
    if (p.bn == 256)
      launch_pair_bn<256>(p, g, st);
    else
      launch_pair_bn<128>(p, g, st);
    return;
  }
  if (p.cluster) {
    if (p.bn == 64)
      launch_cluster_bn<64>(p, g, st);
    else if (p.bn == 128)
      launch_cluster_bn<128>(p, g, st);
    else
      throw std::invalid_argument("cluster split-K supports tile widths 64 and 128");
    return;
  }
  switch (p.bn * 2 + (p.lean ? 1 : 0)) {
    case 512: launch_bn<256, false>(p, g, st); break;
    case 256: launch_bn<128, false>(p, g, st); break;
    case 128: launch_bn<64, false>(p, g, st); break;
    case 513: launch_bn<256, true>(p, g, st); break;
    case 257: launch_bn<128, true>(p, g, st); break;
    case 129: launch_bn<64, true>(p, g, st); break;
    default: throw std::invalid_argument("bad tile width");
  }
}

}  // namespace prlab_gpu
