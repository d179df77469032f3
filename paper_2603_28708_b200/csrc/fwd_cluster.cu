// Batch-1 forward_hidden (hybrid policy, M = B*S <= 128 rows, S <= 128, h = 768, 12 heads of
// 64, ffn 3072 -- GPT-2 small / BERT-base) on thread-block CLUSTERS that each own a block of
// 32 token rows (src/model.cpp:350-452).
//
// Why (measured on B200): the one-CTA-per-SM persistent kernel
// (fwd_small.cu) runs 6 grid-wide stages per layer; a grid barrier costs ~2 400 cycles
// (+1 700 with stores in flight, scripts/ubench/ubench_gridbar2.cu) and every GEMM stage
// re-streams the whole 128-row activation into every SM.  Everything in a transformer
// layer except attention is row-local, so here a 16-CTA cluster owns 32 rows for the whole
// forward: its CTAs split every weight matrix by output features (each CTA streams ~1/16 of
// each layer's fp16 weights through its own TMA ring, ahead of use), exchange activations
// inside the cluster, and synchronise with per-CTA mbarrier arrivals in distributed shared
// memory instead of grid barriers.  Clusters meet only where attention needs keys/values of
// earlier row blocks (per (layer, block, head) release/acquire flags).
//
// Per layer, cluster r (rows 32r..32r+31), CTA c (0..15):
//   LN1   every CTA: the block's x rows (fp32, gathered in L2) -> round16(LN(x)) as the
//         B operand [32 tokens x 768] in its shared memory (SW128 K-major)
//   QKV   CTAs 0..11 = heads: D = [Wq_c; Wk_c] (M=128) and Wv_c (M=64) x xn^T (N = 32 tokens)
//         on tcgen05 (swap-AB: weights are the M operand), epilogue round16(round16(acc)+b)
//   ATTN  head c: q . k^T * 0.125 (causal / batch mask), exact two-pass softmax, P . V on
//         warp-level tensor-core tiles (mma.sync); k/v of earlier blocks from the clusters
//         that own them -> ctx_c
//   Wo    every CTA: its 48 output features (M=64 tile) x ctx^T (all heads, TMA from L2)
//         -> x[:, 48c..] += round16(round16(acc)+bo), kept in shared memory
//   LN2   as LN1
//   FFN1  its 192 hidden features (M=128 + M=64) -> round16(gelu(round16(round16(acc)+b1)))
//         into shared memory as the B operand of
//   FFN2  split-K over the hidden dim: W2[:, 192c..] (6 x M=128) -> fp32 partial [768 x 32];
//         CTA c then sums the 16 partials of its 48 features in fixed order:
//         x += round16(round16(sum) + b2)
// Rounding points are the hybrid path's; fp32 summation orders differ
// (per-CTA K slices, tensor-core accumulation), as everywhere on the tensor-core path.
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

constexpr int kH = 768, kF = 3072, kHeads = 12;
constexpr int kRB = 32;                 // token rows per cluster
constexpr int kCS = 16;                 // CTAs per cluster
constexpr int kXS = kH / kCS;           // 48: x / Wo / FFN2-output features owned per CTA
constexpr int kFS = kF / kCS;           // 192: hidden features per CTA
constexpr int kKB = kH / 64;            // 12 k-blocks over the hidden dim
constexpr int kCompute = 256;           // warps 0..7: MMA issue (warp 0 lane 0), epilogues, rows
constexpr int kThreads = kCompute + 32; // warp 8: weight producer (TMA ring)
constexpr int kRing = 4;
constexpr uint32_t kUnit = 16384;       // one weight unit: 128 rows x 64 k, or 2 k-blocks x 64 rows (fp16)
constexpr uint32_t kSlot = 2 * kUnit;   // one bulk copy / ring slot: two units
// per layer, per CTA: QKV 18 units (heads only), Wo 6, FFN1 18, FFN2 18
constexpr int kUnitsHead = 60, kUnitsOther = 42;
constexpr int kUnitsLayer = kHeads * kUnitsHead + (kCS - kHeads) * kUnitsOther;  // 888
constexpr int kMaxL = 48;
constexpr int kRowH = 72, kRowP = 136, kRowS = 132;  // padded smem rows (conflict-free ldmatrix)

struct Sm {
  static constexpr uint32_t RING = 0;                         // kRing x 32 KB weight slots
  static constexpr uint32_t BOP = RING + kRing * kSlot;       // [12 kb][32 tokens][128 B] xn16 / ctx
  static constexpr uint32_t FF = BOP + kKB * 4096;            // [3 kb][32][128 B] this CTA's ff slice
  // attention scratch, aliasing BOP + FF: xn16 is dead once QKV's MMAs completed, the ff slice
  // once the previous layer's FFN2 did; ctx overwrites it only after every head finished
  static constexpr uint32_t Q = BOP;                          // [32][72] fp16
  static constexpr uint32_t K = Q + kRB * kRowH * 2;          // [128][72]
  static constexpr uint32_t V = K + 128 * kRowH * 2;          // [128][72]
  static constexpr uint32_t P = V + 128 * kRowH * 2;          // [32][136] fp16
  static constexpr uint32_t S = FF + 3 * 4096;                // [32][132] fp32
  static constexpr uint32_t XS = S + kRB * kRowS * 4;         // [32][48] fp32: this CTA's x slice
  static constexpr uint32_t BAR = XS + kRB * kXS * 4;
  static constexpr uint32_t TOTAL = BAR + 256;
};
static_assert(Sm::P + kRB * kRowP * 2 <= Sm::S, "attention scratch must fit in BOP + FF");
constexpr size_t kSmem = 1024 + Sm::TOTAL;
static_assert(kSmem <= 227 * 1024, "fwd_cluster smem");

enum : int { B_FULL = 0, B_EMPTY = kRing, B_ACC = 2 * kRing, B_BOP, B_CS0, B_CS1, B_COUNT };

struct ClLayer {
  const float *ln1g, *ln1b, *ln2g, *ln2b;
  const float *bqkv, *bo, *b1, *b2;  // pre-rounded onto the fp16 lattice
};

struct ClArgs {
  CUtensorMap ctx_map;  // ctx rows as [12 kb][128 rows][64] (box: the block's 32 rows x 12 kb)
  const uint8_t* wstream;  // [L][888 units of 16 KB]: every CTA's weights in consumption order
  ClLayer lw[kMaxL];
  int M, S, L, V, causal;
  int embed_only;      // debug / parity: stop after the embedding gather (xg = tok + pos)
  const float *tok, *pos, *lnfg, *lnfb;
  const int32_t* ids;
  int* err;
  float* xg;           // [128][768] fp32: x rows gathered for the LayerNorms
  __half* ctxg;        // [128][768] fp16: attention outputs (TMA source of Wo's B operand)
  __half* kvg;         // [L][128][1536] fp16: k | v of every row (cross-cluster attention)
  float* part;         // [4 clusters][16][768][32] fp32: FFN2 split-K partials
  unsigned* flags;     // [L][4][16]: k/v of (layer, block, head) published (zeroed per launch)
  long long* dbg;      // optional %globaltimer phase stamps [cluster][2: CTA 0 / 15][L][16] (debug)
  __half* xn16;        // [M][768] out: round16(final LN) for the tied head
};

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_trans(uint32_t addr, uint32_t (&r)[2]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void compute_sync() { named_bar_sync(1, kCompute); }

// mbarrier wait with cluster-scope acquire (the arrivals come from other CTAs' threads)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  const long long t0 = clock64();
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (!ok && clock64() - t0 > (1ll << 31)) {
      printf("prlab_gpu watchdog: cluster sync timeout block %d\n", blockIdx.x);
      __trap();
    }
  }
  asm volatile("fence.acq_rel.cluster;" ::: "memory");  // acquire side of the arrivals' release fences
}

// Cluster-wide barrier of the compute warps (the producer warp keeps streaming weights):
// thread 0 of every CTA arrives (release, cluster scope) on the same-parity mbarrier of all
// 16 CTAs; every compute thread waits for its own CTA's barrier (acquire).  Two barriers
// alternate so an early arrival for the next sync never lands in the current phase.
__device__ __forceinline__ void cluster_sync_compute(uint64_t* bars, uint32_t& n) {
  compute_sync();
  uint64_t* b = bars + B_CS0 + (n & 1);
  if (threadIdx.x == 0) {
    // one cluster-scope release fence (cumulative over the CTA's writes, ordered by the
    // named barrier above), then 16 relaxed arrivals: a release per arrival costs a fence each
    asm volatile("fence.acq_rel.cluster;" ::: "memory");
    const uint32_t a = smem_u32(b);
#pragma unroll
    for (uint32_t p = 0; p < kCS; ++p)
      asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(a, p))
                   : "memory");
  }
  if (threadIdx.x == 0) mbar_wait_cluster(b, (n >> 1) & 1);  // one waiter + fence, then the CTA
  compute_sync();
  ++n;
}

// ---- the weight stream: per layer and CTA rank c, the units the CTA's MMAs consume, in
// order, as SW128 K-major images (built once by build_cluster_stream_kernel) ----
__device__ __forceinline__ int stream_units(int c) { return c < kHeads ? kUnitsHead : kUnitsOther; }
__device__ __forceinline__ int64_t stream_base(int l, int c) {  // in units
  return static_cast<int64_t>(l) * kUnitsLayer + (c < kHeads ? kUnitsHead * c : kHeads * kUnitsHead + kUnitsOther * (c - kHeads));
}

// ---- row LayerNorm of the block's 32 rows (all 768 features) from the gathered x ----
// y = round16(gamma * ((x - mean) * inv) + beta), two-pass fp32 statistics like
// layernorm_lastdim (src/kernels.cpp:170-219), written as the SW128 K-major B operand.
// out16 (optional): rows of the final LN for the head, this CTA's 48 columns.
__device__ void block_layernorm(const ClArgs& a, int r, int nrows, const float* g, const float* bta, uint8_t* bop,
                                __half* out16, int c) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4 vv[4][6];  // the warp's 4 rows in flight at once (one L2 round trip, not four)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int t = warp * 4 + q;
    const float* xr = a.xg + static_cast<int64_t>(kRB * r + t) * kH;
#pragma unroll
    for (int j = 0; j < 6; ++j) vv[q][j] = t < nrows ? ldcg4(xr + lane * 4 + 128 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // the 4 rows' statistics interleaved: independent shuffle / divide chains overlap
  float mean[4], inv[4];
  {
    float sv[4];
#pragma unroll
    for (int rq = 0; rq < 4; ++rq) {
      float s = 0.0f;
#pragma unroll
      for (int j = 0; j < 6; ++j) s += (vv[rq][j].x + vv[rq][j].y) + (vv[rq][j].z + vv[rq][j].w);
      sv[rq] = s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int rq = 0; rq < 4; ++rq) sv[rq] += __shfl_xor_sync(0xffffffffu, sv[rq], o);
#pragma unroll
    for (int rq = 0; rq < 4; ++rq) mean[rq] = __fdiv_rn(sv[rq], static_cast<float>(kH));
#pragma unroll
    for (int rq = 0; rq < 4; ++rq) {
      float q = 0.0f;
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        const float d0 = __fsub_rn(vv[rq][j].x, mean[rq]), d1 = __fsub_rn(vv[rq][j].y, mean[rq]),
                    d2 = __fsub_rn(vv[rq][j].z, mean[rq]), d3 = __fsub_rn(vv[rq][j].w, mean[rq]);
        q += (__fmul_rn(d0, d0) + __fmul_rn(d1, d1)) + (__fmul_rn(d2, d2) + __fmul_rn(d3, d3));
      }
      sv[rq] = q;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int rq = 0; rq < 4; ++rq) sv[rq] += __shfl_xor_sync(0xffffffffu, sv[rq], o);
#pragma unroll
    for (int rq = 0; rq < 4; ++rq)
      inv[rq] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(sv[rq], static_cast<float>(kH)), 1e-5f)));
  }
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    const int k = lane * 4 + 128 * j;
    const float4 gg = __ldg(reinterpret_cast<const float4*>(g + k)), bb = __ldg(reinterpret_cast<const float4*>(bta + k));
    const int kb = k >> 6, chunk = (k & 63) >> 3;
#pragma unroll
    for (int rq = 0; rq < 4; ++rq) {
      const int t = warp * 4 + rq;
      const float4 v = vv[rq][j];
      const float m = mean[rq], iv = inv[rq];
      const uint32_t lo = h2_pack_rn(__fadd_rn(__fmul_rn(gg.x, __fmul_rn(__fsub_rn(v.x, m), iv)), bb.x),
                                     __fadd_rn(__fmul_rn(gg.y, __fmul_rn(__fsub_rn(v.y, m), iv)), bb.y));
      const uint32_t hi = h2_pack_rn(__fadd_rn(__fmul_rn(gg.z, __fmul_rn(__fsub_rn(v.z, m), iv)), bb.z),
                                     __fadd_rn(__fmul_rn(gg.w, __fmul_rn(__fsub_rn(v.w, m), iv)), bb.w));
      *reinterpret_cast<uint2*>(bop + kb * 4096 + t * 128 + ((chunk ^ (t & 7)) << 4) + (k & 7) * 2) = make_uint2(lo, hi);
      if (out16 && t < nrows && k >= kXS * c && k < kXS * (c + 1))
        *reinterpret_cast<uint2*>(out16 + static_cast<int64_t>(kRB * r + t) * kH + k) = make_uint2(lo, hi);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> MMA operand reads
}

// this CTA's x slice (smem, [32][48] fp32) -> the cluster's gathered rows in L2
__device__ __forceinline__ void publish_x(const ClArgs& a, int r, int nrows, int c, const float* xs) {
  for (int e = threadIdx.x; e < kRB * (kXS / 4); e += kCompute) {
    const int t = e / (kXS / 4), j = e % (kXS / 4);
    if (t < nrows)
      *reinterpret_cast<float4*>(a.xg + static_cast<int64_t>(kRB * r + t) * kH + kXS * c + 4 * j) =
          *reinterpret_cast<const float4*>(xs + t * kXS + 4 * j);
  }
}

__global__ void __cluster_dims__(kCS, 1, 1) __launch_bounds__(kThreads, 1) fwd_cluster_kernel(const __grid_constant__ ClArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Sm::BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + B_COUNT);
  const int c = static_cast<int>(cluster_ctarank());
  const int r = static_cast<int>(blockIdx.x) / kCS;
  const int nrows = min(kRB, a.M - kRB * r);
  const uint32_t warp = warp_id(), lane = lane_id();
  uint8_t* bop = smem + Sm::BOP;
  uint8_t* ffb = smem + Sm::FF;
  __half* sQ = reinterpret_cast<__half*>(smem + Sm::Q);
  __half* sK = reinterpret_cast<__half*>(smem + Sm::K);
  __half* sV = reinterpret_cast<__half*>(smem + Sm::V);
  float* sS = reinterpret_cast<float*>(smem + Sm::S);
  __half* sP = reinterpret_cast<__half*>(smem + Sm::P);
  float* xs = reinterpret_cast<float*>(smem + Sm::XS);

  if (threadIdx.x == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&bars[B_FULL + i], 1);
      mbar_init(&bars[B_EMPTY + i], 1);
    }
    mbar_init(&bars[B_ACC], 1);
    mbar_init(&bars[B_BOP], 1);
    mbar_init(&bars[B_CS0], kCS);
    mbar_init(&bars[B_CS1], kCS);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(tslot, 256);
    tmem_relinquish();
  }
  if (warp == 8 && lane == 0) tma_prefetch_desc(&a.ctx_map);
  tc_fence_before();
  cluster_sync_all();  // barrier inits visible to the whole cluster before any remote arrival
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 8) {
    // ---------------- weight producer: the CTA's whole weight stream, 32 KB bulk copies,
    // kRing slots ahead of the MMAs (the stream is contiguous per layer and rank)
    if (lane == 0) {
      uint32_t ch = 0;
      for (int l = 0; l < (a.embed_only ? 0 : a.L); ++l) {
        const uint8_t* src = a.wstream + stream_base(l, c) * kUnit;
        const int n = stream_units(c) / 2;
        for (int i = 0; i < n; ++i, ++ch) {
          const uint32_t sl = ch % kRing;
          mbar_wait(&bars[B_EMPTY + sl], ((ch / kRing) & 1) ^ 1);
          mbar_expect_tx(&bars[B_FULL + sl], kSlot);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(smem + Sm::RING + sl * kSlot)),
              "l"(src + static_cast<int64_t>(i) * kSlot), "r"(kSlot), "r"(smem_u32(&bars[B_FULL + sl]))
              : "memory");
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- compute warps
    uint32_t csn = 0;       // cluster syncs done
    uint32_t it = 0;        // weight items consumed (MMA thread)
    uint32_t accn = 0;      // accumulator-ready phases
    uint32_t bopn = 0;      // ctx TMA phases
    const uint32_t quad = warp & 3, half = warp >> 2;
    const uint32_t lane_base = tmem + ((quad * 32) << 16);
    constexpr uint32_t id128 = idesc_f16_f32(128, 32, 0, 0);
    constexpr uint32_t id64 = idesc_f16_f32(64, 32, 0, 0);
    long long wait_cyc = 0;  // MMA thread: cycles spent waiting for weight units (debug)
    // MMA thread: shared address of the next weight unit (waits for its slot); units come in
    // pairs per slot, the slot is released after the pair's MMAs (unit_done)
    auto next_unit = [&]() -> uint32_t {
      const uint32_t ch = it >> 1, sl = ch % kRing;
      if ((it & 1) == 0) {
        const long long w0 = clock64();
        mbar_wait(&bars[B_FULL + sl], (ch / kRing) & 1);
        wait_cyc += clock64() - w0;
        tc_fence_after();
      }
      return smem_u32(smem + Sm::RING + sl * kSlot + (it & 1) * kUnit);
    };
    auto unit_done = [&]() {
      if (it & 1) umma_commit(&bars[B_EMPTY + (it >> 1) % kRing]);
      ++it;
    };
    // one unit of A: 4 k-steps of 16 against the B k-block at b0
    auto mma4 = [&](uint32_t d, uint32_t a0, uint32_t b0, uint32_t idesc, bool first) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_f16_ss(d, sw128_desc(a0 + kk * 32, 0, 1024), sw128_desc(b0 + kk * 32, 0, 1024), idesc, !first || kk != 0);
    };
    // the [128 rows | 2 x 64 rows] pattern of QKV and FFN1: per k-block pair, two M=128 units
    // (one k-block each) into TMEM columns [0, 32) and one unit holding both k-blocks of the
    // 64-row tail (M=64) into [32, 64)
    auto gemm_128_64 = [&](uint32_t bbase) {
      for (int kp = 0; kp < kKB / 2; ++kp) {
        for (int s2 = 0; s2 < 2; ++s2) {
          const int kb = 2 * kp + s2;
          mma4(tmem, next_unit(), smem_u32(smem + bbase + kb * 4096), id128, kb == 0);
          unit_done();
        }
        const uint32_t a0 = next_unit();
        for (int s2 = 0; s2 < 2; ++s2) {
          const int kb = 2 * kp + s2;
          mma4(tmem + 32, a0 + s2 * 8192, smem_u32(smem + bbase + kb * 4096), id64, kb == 0);
        }
        unit_done();
      }
      umma_commit(&bars[B_ACC]);
    };
    auto acc_wait = [&]() {
      mbar_wait(&bars[B_ACC], accn & 1);
      ++accn;
      tc_fence_after();
    };
    // M=64 accumulator layout (probed, scripts/ubench/probe_tmem_layout.cu): row m sits in
    // TMEM lane 32 * (m / 16) + m % 16 -- lanes 0..15 of each quadrant

    // ---- embedding gather (bit-exact fp32 tok + pos, kernels.cpp:288-290) into the x slice
    for (int e = threadIdx.x; e < kRB * kXS; e += kCompute) {
      const int t = e / kXS, j = e % kXS, row = kRB * r + t;
      float v = 0.0f;
      if (t < nrows) {
        const int id = a.ids[row];
        const bool ok = id >= 0 && id < a.V;
        if (!ok) atomicExch(a.err, 1);
        const int col = kXS * c + j;
        v = __fadd_rn(ok ? a.tok[static_cast<int64_t>(id) * kH + col] : 0.0f,
                      a.pos[static_cast<int64_t>(row % a.S) * kH + col]);
      }
      xs[t * kXS + j] = v;
    }
    compute_sync();
    publish_x(a, r, nrows, c, xs);
    cluster_sync_compute(bars, csn);

    for (int l = 0; l < (a.embed_only ? 0 : a.L); ++l) {
      const ClLayer& w = a.lw[l];
      long long* dbs = (a.dbg && threadIdx.x == 0 && (c == 0 || c == kCS - 1))
                           ? a.dbg + ((static_cast<int64_t>(r) * 2 + (c != 0)) * a.L + l) * 16 : nullptr;
#define STAMP(k) \
  if (dbs) dbs[k] = globaltimer()
      STAMP(0);
      // ---------------- LN1 -> B operand
      block_layernorm(a, r, nrows, w.ln1g, w.ln1b, bop, nullptr, c);
      tc_fence_before();
      compute_sync();
      STAMP(1);
      if (c < kHeads) {
        // ---------------- QKV of head c (swap-AB: weights M, tokens N = 32)
        if (threadIdx.x == 0) {
          tc_fence_after();
          gemm_128_64(Sm::BOP);
        }
        __syncwarp();
        // key range of the block's queries: their sequences, causal up to the block's end
        const int R0 = kRB * r, R1 = R0 + nrows;
        const int klo = (R0 / a.S) * a.S;
        const int khi = a.causal ? R1 : min(a.M, ((R1 - 1) / a.S + 1) * a.S);
        const int nkeys = khi - klo, kvp = (nkeys + 15) & ~15;
        acc_wait();
        STAMP(2);
        {
          // q (lanes 0..63) / k (lanes 64..127) of D1, v from the M=64 D2
          uint32_t u[16];
          tmem_ld16(lane_base + 16 * half, u);
          tmem_wait_ld();
          const int m = static_cast<int>(quad * 32 + lane);
          const float bias = m < 64 ? w.bqkv[64 * c + m] : w.bqkv[kH + 64 * c + (m - 64)];
          for (int j = 0; j < 16; ++j) {
            const int t = static_cast<int>(16 * half) + j;
            const __half hv = __float2half_rn(__fadd_rn(r16(__uint_as_float(u[j])), bias));
            if (m < 64)
              sQ[t * kRowH + m] = hv;
            else
              sK[(R0 + t - klo) * kRowH + (m - 64)] = hv;
          }
          uint32_t v[16];
          tmem_ld16(lane_base + 32 + 16 * half, v);
          tmem_wait_ld();
          if (lane < 16) {
            const int f = static_cast<int>(quad * 16 + lane);
            const float bv = w.bqkv[2 * kH + 64 * c + f];
            for (int j = 0; j < 16; ++j) {
              const int t = static_cast<int>(16 * half) + j;
              sV[(R0 + t - klo) * kRowH + f] = __float2half_rn(__fadd_rn(r16(__uint_as_float(v[j])), bv));
            }
          }
        }
        tc_fence_before();
        compute_sync();
        // publish this block's k / v of head c (rows R0..R1) for the clusters after it
        {
          __half* kvl = a.kvg + static_cast<int64_t>(l) * 128 * 2 * kH;
          for (int e = threadIdx.x; e < nrows * 16; e += kCompute) {
            const int t = e >> 4, part = (e >> 3) & 1, ch = e & 7;
            const __half* src = (part ? sV : sK) + (R0 + t - klo) * kRowH + ch * 8;
            *reinterpret_cast<uint4*>(kvl + static_cast<int64_t>(R0 + t) * 2 * kH + part * kH + 64 * c + ch * 8) =
                *reinterpret_cast<const uint4*>(src);
          }
          compute_sync();
          if (threadIdx.x == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.flags + (l * 4 + r) * 16 + c), "r"(1u)
                         : "memory");
          STAMP(3);
        }
        // ---------------- attention of head c for the block's 32 queries
        {
          // keys of other blocks: wait for their owners' flags, then load
          const int rlo = klo / kRB, rhi = (khi - 1) / kRB;
          if (threadIdx.x == 0) {
            for (int rb = rlo; rb <= rhi; ++rb) {
              if (rb == r) continue;
              const unsigned* f = a.flags + (l * 4 + rb) * 16 + c;
              const long long t0 = clock64();
              while (ld_acquire_gpu(f) == 0u) {
                if (clock64() - t0 > (1ll << 31)) {
                  printf("prlab_gpu watchdog: k/v flag timeout block %d layer %d src %d\n", blockIdx.x, l, rb);
                  __trap();
                }
              }
            }
          }
          compute_sync();
          STAMP(4);
          const __half* kvl = a.kvg + static_cast<int64_t>(l) * 128 * 2 * kH;
          for (int e = threadIdx.x; e < kvp * 16; e += kCompute) {
            const int kj = e >> 4, part = (e >> 3) & 1, ch = e & 7;
            const int row = klo + kj;
            __half* dst = (part ? sV : sK) + kj * kRowH + ch * 8;
            if (kj >= nkeys)
              *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
            else if (row < R0 || row >= R1)
              *reinterpret_cast<uint4*>(dst) =
                  __ldcg(reinterpret_cast<const uint4*>(kvl + static_cast<int64_t>(row) * 2 * kH + part * kH + 64 * c + ch * 8));
          }
          compute_sync();
          const int g8 = static_cast<int>(lane >> 2), t4 = static_cast<int>(lane & 3);
          // scores: warp w -> keys [16w, 16w + 16), both 16-query halves
          if (static_cast<int>(warp) * 16 < kvp) {
#pragma unroll
            for (int mq = 0; mq < 2; ++mq) {
              float acc[2][4] = {};
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
                uint32_t af[4], bf[4];
                ldsm_x4(smem_u32(sQ + (mq * 16 + (lane & 15)) * kRowH + ks * 16 + (lane >> 4) * 8), af);
                ldsm_x4(smem_u32(sK + (warp * 16 + (lane & 7) + (lane >> 4) * 8) * kRowH + ks * 16 + ((lane >> 3) & 1) * 8), bf);
                mma16816(acc[0], af, bf[0], bf[1]);
                mma16816(acc[1], af, bf[2], bf[3]);
              }
#pragma unroll
              for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int t = mq * 16 + g8 + (e >> 1) * 8, kj = static_cast<int>(warp) * 16 + nt * 8 + 2 * t4 + (e & 1);
                  const int qrow = R0 + t, krow = klo + kj;
                  const bool valid = t < nrows && kj < nkeys && krow / a.S == qrow / a.S && (!a.causal || krow <= qrow);
                  sS[t * kRowS + kj] = valid ? r16(__fmul_rn(acc[nt][e], 0.125f)) : __int_as_float(0xff800000);
                }
            }
          }
          compute_sync();
          // exact two-pass softmax (kernels.cpp:127-168): warp w -> rows 4w .. 4w + 3
          {
            constexpr float LOG2E = 1.4426950408889634f;
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
              const int t = static_cast<int>(warp) * 4 + rr;
              float sc[4], e[4], mx = __int_as_float(0xff800000);
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const int j = c4 * 32 + static_cast<int>(lane);
                sc[c4] = j < kvp ? sS[t * kRowS + j] : __int_as_float(0xff800000);
                mx = fmaxf(mx, sc[c4]);
              }
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
              const bool live = mx != __int_as_float(0xff800000);
              const float mxl = live ? __fmul_rn(mx, LOG2E) : 0.0f;
              float sum = 0.0f;
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                e[c4] = live ? ex2_approx(__fmaf_rn(sc[c4], LOG2E, -mxl)) : 0.0f;
                sum = __fadd_rn(sum, e[c4]);
              }
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) sum = __fadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
              const float inv = live ? __frcp_rn(sum) : 0.0f;
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const int j = c4 * 32 + static_cast<int>(lane);
                if (j < kvp) sP[t * kRowP + j] = __float2half_rn(__fmul_rn(e[c4], inv));
              }
            }
          }
          compute_sync();
          // ctx = round16(P . V): warp w -> dims [8w, 8w + 8), both query halves -> L2
#pragma unroll
          for (int mq = 0; mq < 2; ++mq) {
            float o[4] = {};
            for (int ks = 0; ks < kvp / 16; ++ks) {
              uint32_t af[4], bf[2];
              ldsm_x4(smem_u32(sP + (mq * 16 + (lane & 15)) * kRowP + ks * 16 + (lane >> 4) * 8), af);
              ldsm_x2_trans(smem_u32(sV + (ks * 16 + (lane & 15)) * kRowH + warp * 8), bf);
              mma16816(o, af, bf[0], bf[1]);
            }
            const int t0 = mq * 16 + g8;
            __half* base = a.ctxg + static_cast<int64_t>(R0) * kH + 64 * c + warp * 8 + 2 * t4;
            *reinterpret_cast<__half2*>(base + static_cast<int64_t>(t0) * kH) = __floats2half2_rn(o[0], o[1]);
            *reinterpret_cast<__half2*>(base + static_cast<int64_t>(t0 + 8) * kH) = __floats2half2_rn(o[2], o[3]);
          }
        }
      }
      STAMP(5);
      cluster_sync_compute(bars, csn);  // every head's ctx of the block is in L2
      STAMP(6);
      // ---------------- Wo: this CTA's 48 output features x all heads' ctx (TMA from L2)
      if (threadIdx.x == 0) {
        // generic reads of the attention scratch (aliasing BOP) were ordered by the sync
        // above; order them against the async-proxy write that reuses the bytes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
        mbar_expect_tx(&bars[B_BOP], kKB * 4096);
        tma_load_3d(bop, &a.ctx_map, &bars[B_BOP], 0, kRB * r, 0);
        mbar_wait(&bars[B_BOP], bopn & 1);
        tc_fence_after();
        for (int kp = 0; kp < kKB / 2; ++kp) {  // Wo rows 48c.. padded to 64: one unit per k-block pair
          const uint32_t a0 = next_unit();
          for (int s2 = 0; s2 < 2; ++s2) {
            const int kb = 2 * kp + s2;
            mma4(tmem, a0 + s2 * 8192, smem_u32(bop + kb * 4096), id64, kb == 0);
          }
          unit_done();
        }
        umma_commit(&bars[B_ACC]);
      }
      ++bopn;
      __syncwarp();
      acc_wait();
      STAMP(7);
      {
        uint32_t u[16];
        tmem_ld16(lane_base + 16 * half, u);
        tmem_wait_ld();
        const int m = static_cast<int>(quad * 16 + lane);
        if (lane < 16 && m < kXS) {
          const float bo = w.bo[kXS * c + m];
          for (int j = 0; j < 16; ++j) {
            const int t = static_cast<int>(16 * half) + j;
            float& xv = xs[t * kXS + m];
            xv = __fadd_rn(xv, r16(__fadd_rn(r16(__uint_as_float(u[j])), bo)));
          }
        }
      }
      tc_fence_before();
      compute_sync();
      publish_x(a, r, nrows, c, xs);
      cluster_sync_compute(bars, csn);
      STAMP(8);
      // ---------------- LN2 -> B operand; FFN1 (+GELU) -> ff slice in shared memory
      block_layernorm(a, r, nrows, w.ln2g, w.ln2b, bop, nullptr, c);
      tc_fence_before();
      compute_sync();
      STAMP(9);
      if (threadIdx.x == 0) {
        tc_fence_after();
        gemm_128_64(Sm::BOP);
      }
      __syncwarp();
      acc_wait();
      STAMP(10);
      {
        auto put_ff = [&](int k, int t, float v) {  // ff[token t][local hidden k] in the SW128 K-major layout
          *reinterpret_cast<__half*>(ffb + (k >> 6) * 4096 + t * 128 + ((((k & 63) >> 3) ^ (t & 7)) << 4) + (k & 7) * 2) =
              __float2half_rn(v);
        };
        uint32_t u[16];
        tmem_ld16(lane_base + 16 * half, u);
        tmem_wait_ld();
        {
          const int k = static_cast<int>(quad * 32 + lane);
          const float b1 = w.b1[kFS * c + k];
          for (int j = 0; j < 16; j += 2) {
            float x0 = r16(__fadd_rn(r16(__uint_as_float(u[j])), b1)), x1 = r16(__fadd_rn(r16(__uint_as_float(u[j + 1])), b1));
            gelu2_fast(x0, x1);
            put_ff(k, static_cast<int>(16 * half) + j, x0);
            put_ff(k, static_cast<int>(16 * half) + j + 1, x1);
          }
        }
        tmem_ld16(lane_base + 32 + 16 * half, u);
        tmem_wait_ld();
        if (lane < 16) {
          const int k = 128 + static_cast<int>(quad * 16 + lane);
          const float b1 = w.b1[kFS * c + k];
          for (int j = 0; j < 16; j += 2) {
            float x0 = r16(__fadd_rn(r16(__uint_as_float(u[j])), b1)), x1 = r16(__fadd_rn(r16(__uint_as_float(u[j + 1])), b1));
            gelu2_fast(x0, x1);
            put_ff(k, static_cast<int>(16 * half) + j, x0);
            put_ff(k, static_cast<int>(16 * half) + j + 1, x1);
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      compute_sync();
      // ---------------- FFN2 split-K: W2[:, 192c ..] x ff_c^T -> fp32 partial [768][32] in L2
      if (threadIdx.x == 0) {
        tc_fence_after();
        for (int mt = 0; mt < 6; ++mt)
          for (int kbx = 0; kbx < 3; ++kbx) {
            mma4(tmem + 32 * mt, next_unit(), smem_u32(ffb + kbx * 4096), id128, kbx == 0);
            unit_done();
          }
        umma_commit(&bars[B_ACC]);
      }
      __syncwarp();
      acc_wait();
      STAMP(11);
      {
        float* pbase = a.part + (static_cast<int64_t>(r) * kCS + c) * kH * kRB;
        for (int mt = 0; mt < 6; ++mt) {
          uint32_t u[16];
          tmem_ld16(lane_base + 32 * mt + 16 * half, u);
          tmem_wait_ld();
          float4* dst = reinterpret_cast<float4*>(pbase + static_cast<int64_t>(128 * mt + quad * 32 + lane) * kRB + 16 * half);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dst[q] = make_float4(__uint_as_float(u[4 * q]), __uint_as_float(u[4 * q + 1]), __uint_as_float(u[4 * q + 2]),
                                 __uint_as_float(u[4 * q + 3]));
        }
      }
      tc_fence_before();
      STAMP(12);
      cluster_sync_compute(bars, csn);
      STAMP(13);
      // ---------------- reduce the 16 partials of this CTA's 48 features (fixed order)
      {
        const float* pb = a.part + static_cast<int64_t>(r) * kCS * kH * kRB + static_cast<int64_t>(kXS * c) * kRB;
        // 6 outputs per thread x 16 partials: every load issued before the ordered sums
        constexpr int kPer = kXS * kRB / kCompute;  // 6
        float pv[kPer][kCS];
#pragma unroll
        for (int q = 0; q < kPer; ++q)
#pragma unroll
          for (int cc = 0; cc < kCS; ++cc)
            pv[q][cc] = __ldcg(pb + static_cast<int64_t>(cc) * kH * kRB + threadIdx.x + q * kCompute);
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
          const int e = threadIdx.x + q * kCompute, m = e / kRB, t = e % kRB;
          float sum = 0.0f;
#pragma unroll
          for (int cc = 0; cc < kCS; ++cc) sum = __fadd_rn(sum, pv[q][cc]);
          float& xv = xs[t * kXS + m];
          xv = __fadd_rn(xv, r16(__fadd_rn(r16(sum), w.b2[kXS * c + m])));
        }
      }
      compute_sync();
      STAMP(14);
      publish_x(a, r, nrows, c, xs);
      cluster_sync_compute(bars, csn);
      if (dbs) dbs[15] = wait_cyc;
    }
#undef STAMP
    // ---------------- final LayerNorm -> round16 rows for the tied head
    if (!a.embed_only) block_layernorm(a, r, nrows, a.lnfg, a.lnfb, bop, a.xn16, c);
    compute_sync();
  }
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

// The per-CTA weight streams of one layer (stream_base): 16-byte chunk q of the layer's
// 888 units, gathered from the K-major fp16 weights and written at its SW128 position (the
// 16-byte chunk j of image row t sits at chunk j ^ (t & 7)), so one plain bulk copy into a
// 1024-aligned slot yields the swizzled MMA operand.
__global__ void build_cluster_stream_kernel(const __half* __restrict__ wqkv, const __half* __restrict__ wo,
                                            const __half* __restrict__ w1, const __half* __restrict__ w2,
                                            uint8_t* __restrict__ dst) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= static_cast<int64_t>(kUnitsLayer) * 1024) return;
  const int u = static_cast<int>(q >> 10), cq = static_cast<int>(q & 1023), t = cq >> 3, pch = cq & 7,
            j = pch ^ (t & 7);
  int c, i;
  if (u < kHeads * kUnitsHead) {
    c = u / kUnitsHead;
    i = u % kUnitsHead;
  } else {
    c = kHeads + (u - kHeads * kUnitsHead) / kUnitsOther;
    i = (u - kHeads * kUnitsHead) % kUnitsOther + (kUnitsHead - kUnitsOther);  // no QKV units
  }
  const __half* src;
  int64_t row = 0;
  int kb, K = kH;
  bool zero = false;
  if (i < 18) {  // QKV: [Wq_c; Wk_c] k-block 2kp+sub, or Wv_c k-blocks 2kp, 2kp+1
    const int kp = i / 3, sb = i % 3;
    src = wqkv;
    if (sb < 2) {
      kb = 2 * kp + sb;
      row = t < 64 ? 64 * c + t : kH + 64 * c + (t - 64);
    } else {
      kb = 2 * kp + t / 64;
      row = 2 * kH + 64 * c + (t & 63);
    }
  } else if (i < 24) {  // Wo rows 48c .. 48c+47 (+16 zero rows), k-blocks 2kp, 2kp+1
    const int kp = i - 18, tt = t & 63;
    src = wo;
    kb = 2 * kp + t / 64;
    zero = tt >= kXS;
    row = kXS * c + tt;
  } else if (i < 42) {  // W1 rows 192c .. +127 (one k-block) or +128 .. +191 (two k-blocks)
    const int jj = i - 24, kp = jj / 3, sb = jj % 3;
    src = w1;
    if (sb < 2) {
      kb = 2 * kp + sb;
      row = kFS * c + t;
    } else {
      kb = 2 * kp + t / 64;
      row = kFS * c + 128 + (t & 63);
    }
  } else {  // W2 rows 128mt .. +127, k-block 3c + kbx (the CTA's slice of the hidden dim)
    const int jj = i - 42;
    src = w2;
    row = 128 * (jj / 3) + t;
    kb = 3 * c + jj % 3;
    K = kF;
  }
  const uint4 v = zero ? make_uint4(0, 0, 0, 0)
                       : *reinterpret_cast<const uint4*>(src + row * K + kb * 64 + j * 8);
  *reinterpret_cast<uint4*>(dst + static_cast<int64_t>(u) * kUnit + t * 128 + pch * 16) = v;
}

}  // namespace

size_t cluster_stream_bytes_per_layer() { return static_cast<size_t>(kUnitsLayer) * kUnit; }

void build_cluster_stream(const __half* wqkv, const __half* wo, const __half* w1, const __half* w2, void* dst,
                          cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(kUnitsLayer) * 1024;
  build_cluster_stream_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(wqkv, wo, w1, w2,
                                                                                   static_cast<uint8_t*>(dst));
  PRLAB_CUDA(cudaGetLastError());
}

long long*& cluster_debug_stamps() {
  static long long* p = nullptr;
  return p;
}

// Opt-in (PRLAB_FWD_CLUSTER=1): parity-green on every batch-1 shape, but measured slower than
// fwd_small at C2 (0.72 vs 0.36 ms per trunk): the per-CTA weight stream reaches only
// ~66 B/clk per SM in 16-CTA clusters (scripts/ubench/ubench_cluster_stream.cu), i.e. a
// 7.7 us/layer floor, and every other phase shares that ingress.
bool fwd_cluster_supported(int64_t M, int64_t S, int64_t h, int64_t f, int64_t H, int64_t L) {
  const char* on = std::getenv("PRLAB_FWD_CLUSTER");
  if (on == nullptr || std::atoi(on) == 0) return false;
  return h == kH && f == kF && H == kHeads && L >= 1 && L <= kMaxL && M >= 1 && M <= 128 && S <= 128;
}

size_t fwd_cluster_workspace_bytes(int64_t L) {
  return (128 * kH * 4) + (128 * kH * 2) + static_cast<size_t>(L) * 128 * 2 * kH * 2 +
         static_cast<size_t>(4) * kCS * kH * kRB * 4 + static_cast<size_t>(L) * 4 * 16 * 4 + 4096;
}

void launch_fwd_cluster(const FwdClusterPlan& p, cudaStream_t st) {
  static std::mutex mu;
  static uint64_t done = 0;
  once_per_device(mu, done, [] {
    PRLAB_CUDA(cudaFuncSetAttribute(fwd_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmem)));
    PRLAB_CUDA(cudaFuncSetAttribute(fwd_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  });
  static thread_local ClArgs a;  // ~10 KB of kernel parameters, one per host thread
  a = ClArgs{};
  if (p.L > kMaxL) throw std::invalid_argument("fwd_cluster: too many layers");
  a.ctx_map = p.ctx_map;
  a.wstream = p.wstream;
  std::memcpy(a.lw, p.host_lw, sizeof(ClLayer) * p.L);
  a.M = p.M;
  a.S = p.S;
  a.L = p.L;
  a.V = p.V;
  a.causal = p.causal;
  a.embed_only = p.embed_only;
  a.tok = p.tok;
  a.pos = p.pos;
  a.lnfg = p.lnfg;
  a.lnfb = p.lnfb;
  a.ids = p.ids;
  a.err = p.err;
  a.xg = p.xg;
  a.ctxg = p.ctxg;
  a.kvg = p.kvg;
  a.part = p.part;
  a.flags = p.flags;
  a.xn16 = p.xn16;
  a.dbg = cluster_debug_stamps();
  PRLAB_CUDA(cudaMemsetAsync(p.flags, 0, static_cast<size_t>(p.L) * 4 * 16 * 4, st));
  const int nclus = (p.M + kRB - 1) / kRB;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCS * nclus);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cfg.numAttrs = 0;
  PRLAB_CUDA(cudaLaunchKernelEx(&cfg, fwd_cluster_kernel, a));
}

}  // namespace prlab_gpu
