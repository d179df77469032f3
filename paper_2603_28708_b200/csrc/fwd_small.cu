// Batch-1 forward as ONE persistent kernel (hybrid policy, M = B*S <= 128 rows,
// S <= 128 keys): the 73 dependent steps of a GPT-2/BERT forward_hidden
// (src/model.cpp:350-452) run as stages of a cooperative grid (one CTA per SM)
// separated by grid-wide barriers, instead of ~85 kernel launches whose fixed
// launch/drain cost (~2.9 us each) dominates batch-1 latency.
//
// Per layer (tasks are spread over the CTAs; every stage reads only what the previous
// stages wrote, so one barrier between stages is the whole synchronisation):
//   QKV     xn16 . Wqkv^T   tcgen05 M=128 N=16 tiles, full K, epilogue round16(round16(acc) + b)
//                           -> fp16 q|k|v
//   ATTN+WO per (batch, head, 16 queries), warp-level tensor-core tiles (mma.sync): scores
//           round16(q.k * 0.125), causal -inf, exact two-pass softmax, p = round16(e / sum),
//           ctx = round16(p . v), then the head's share of the output projection
//           ctx_h . Wo[:, head cols]^T -> fp32 partial per head (model.cpp:372-392)
//   RLN2    per row: x += round16(round16(sum of the head partials) + bo); xn16 = round16(LN2(x))
//   FFN1    xn16 . W1^T     N=32 tiles, full K, epilogue round16(gelu(round16(acc+b1)))
//   FFN2    ff16 . W2^T     N=32 tiles x F/512 splits -> fp32 partials
//   RLN1    per row: x += round16(round16(sum) + b2); xn16 = round16(LN(x)) with the next
//           layer's LN1 (or the final LN) -- embed + LN1 of layer 0 is stage 0
// The tied head stays a separate (PDL-chained) GEMM launch on xn16.
// Rounding points are those of the multi-kernel path; the only
// difference is the fp32 summation order (split-K / per-head partials, mma.sync tiles).
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

constexpr int kThreads = 256;            // GEMM tasks: warp 4 TMA, warp 5 MMA, all 8 warps epilogue
constexpr int kTileN = 32;               // GEMM output columns per task
// Operand loads are 3D tensor maps over a K-major matrix viewed as [K/64][rows][64]: one
// TMA request moves several 64-wide k-blocks.  Measured (scripts/ubench/ubench_tma2d.cu,
// profiles/r01/ubench_tma2d.jsonl): a 2D 128-row SW128 box (16 KB) streams at 26.6 B/clk
// per SM, a 3D box of 2 k-blocks (32 KB) at 91.5 B/clk -- the per-request cost dominates.
constexpr int kKPR = 4;                  // max k-blocks per A request (one ring slot)
constexpr int kStages = 2;               // A ring of 2 x 64 KB (the attention scratch aliases it)
constexpr uint32_t kABytes = 128 * 64 * 2;         // 16 KB per k-block
constexpr uint32_t kBBox = kTileN * 64 * 2;        // 4 KB per 64-wide k-block
constexpr int kMaxKB = 16;                         // B for one task: <= 16 k-blocks (1024 of K)
constexpr int kQB = 16;                            // queries per attention task (one m16 MMA row block)

struct SmemL {
  static constexpr uint32_t A = 0;
  static constexpr uint32_t B = A + kStages * kKPR * kABytes;      // 128 KB
  static constexpr uint32_t BAR = B + kMaxKB * kBBox;              // 192 KB
};
// Attention + Wo stage scratch (the A ring and the B region are idle then): the head's
// Wo column slice [h rows][64] (TMA, 128B-swizzled), then K, V, Q, scores, P, ctx with
// padded rows (conflict-free ldmatrix).
constexpr int kRowH = 72;    // fp16 row stride (halves) of K / V / Q / ctx
constexpr int kRowP = 136;   // fp16 row stride of P
constexpr int kRowS = 132;   // fp32 row stride of the scores
__host__ __device__ constexpr uint32_t att_bytes(int h, int qb) {
  return static_cast<uint32_t>(h) * 128 + (2 * 128 + 2 * qb) * kRowH * 2 + qb * kRowS * 4 + qb * kRowP * 2;
}
static_assert(att_bytes(1024, 16) <= SmemL::BAR && att_bytes(768, 32) <= SmemL::BAR, "attention scratch");

struct LayerW {
  const float *ln1g, *ln1b, *ln2g, *ln2b;  // fp32 [h]
  const float *bqkv, *bo, *b1, *b2;        // pre-rounded fp32
  const __half *wqkv, *wo, *w1, *w2;       // fp16 K-major weights (L2 prefetch of the next layer)
};

constexpr int kMaxLayers = 48;
// Everything the stages dereference lives in the (32 KB) kernel parameter space: the
// tensor maps (TMA descriptors are fetched from param space) and the per-layer
// parameter pointers, so no stage starts with a dependent global load.
struct SmallArgs {
  CUtensorMap maps[2 + 4 * kMaxLayers];  // xn16, ff16, then per layer Wqkv, Wo (2D, 256-row box), W1, W2
  LayerW lw[kMaxLayers];
  int M, B, S, h, f, H, L, V, causal;
  int split_ffn2;
  int embed_only;                // debug: stop after stage 0 (x = the embedding gather)
  int q32;                       // attention tasks of 32 queries (else 16)
  const float *tok, *pos, *lnfg, *lnfb;
  const int32_t* ids;
  int* err;
  float* x;
  __half *xn16, *ff16;
  float* part;                   // fp32 partial sums [split][M][h] (split = head for Wo, K split for FFN2)
  unsigned* gbar;                // grid barrier counter (zeroed before each launch)
  // Stage hand-offs without grid barriers (null: barriers): per-task completion counters,
  // zeroed before each launch, released by the producing CTA(s) after their stores.
  unsigned* qkv_flags;           // per QKV task (q|k|v columns of all rows)
  unsigned* qkv_done;            // all QKV tasks (the row stage may overwrite xn16 after it)
  unsigned* rows1_done;          // embed+LN1 / RLN1 rows done (the QKV GEMMs' A operand)
  unsigned* rows2_done;          // RLN2 rows done (the FFN1 GEMMs' A operand)
  unsigned* ffn2_done;           // FFN2 tasks done (every K split partial of every row)
  unsigned* attn_flags;          // per attention task (b, head, query block): its Wo partial rows
  unsigned* ffn1_flags;          // per FFN1 task: its GELU output columns
  long long* dbg;                // optional [stage][grid][2] globaltimer (arrive, release)
};

// Generic-proxy global writes of one stage (epilogue / row-stage stores) are read by
// TMA (async proxy) in a later stage on other CTAs: after the barrier's release/acquire,
// the TMA-issuing thread fences its generic view against the async proxy before its
// loads.  (The unqualified fence.proxy.async by every thread costs a MEMBAR.ALL.GPU each
// -- ~10% of all warp stall samples in ncu, profiles/r01.)
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin (acquire) until *ctr >= want -- one stage hand-off counter; a protocol bug traps after
// ~2 s instead of hanging the GPU (what: 0 QKV task, 1 row, 2 FFN1 task, 3 stage counter).
__device__ __forceinline__ void spin_acquire(const unsigned* ctr, unsigned want, int what, int idx) {
  const long long t0 = clock64();
  while (ld_acquire(ctr) < want) {
    if (clock64() - t0 > (1ll << 32)) {
      printf("prlab_gpu watchdog: hand-off timeout (kind %d, index %d) block %d want %u seen %u\n", what, idx,
             blockIdx.x, want, ld_acquire(ctr));
      __trap();
    }
  }
}

// all CTAs are co-resident (cooperative launch, one CTA per SM).  Arrive = one
// red.release.gpu (cumulative over the CTA's writes ordered by the bar.sync before it),
// wait = ld.acquire.gpu polling by one thread.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& target, long long* dbg = nullptr) {
  __syncthreads();
  const unsigned stage = target / gridDim.x;
  target += gridDim.x;
  if (threadIdx.x == 0) {
    if (dbg) dbg[(static_cast<int64_t>(stage) * gridDim.x + blockIdx.x) * 2] = globaltimer();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    const long long t0 = clock64();
    while (ld_acquire(bar) < target) {
      if (clock64() - t0 > (1ll << 32)) {  // watchdog (~2 s): a protocol bug must trap, not hang
        printf("prlab_gpu watchdog: grid barrier timeout block %d target %u seen %u\n", blockIdx.x, target,
               ld_acquire(bar));
        __trap();
      }
    }
    if (dbg) dbg[(static_cast<int64_t>(stage) * gridDim.x + blockIdx.x) * 2 + 1] = globaltimer();
  }
  __syncthreads();
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// Pull this layer's small fp32 vectors (LN gamma/beta, biases) into L2 -- spread over
// the CTAs, one 128-byte line per thread -- so the row stages do not start with DRAM
// misses on parameters the previous forward evicted.
__device__ void prefetch_layer_params(const SmallArgs& a, const LayerW& w) {
  const int h = a.h, f = a.f;
  const float* vec[8] = {w.ln1g, w.ln1b, w.ln2g, w.ln2b, w.bqkv, w.bo, w.b1, w.b2};
  const int len[8] = {h, h, h, h, 3 * h, h, f, h};
  int idx = static_cast<int>(blockIdx.x * blockDim.x + threadIdx.x);
  for (int v = 0; v < 8; ++v) {
    const int lines = (len[v] + 31) / 32;
    if (idx < lines) prefetch_l2(vec[v] + idx * 32);
    idx -= lines;
  }
}
// ... and the layer's fp16 weights (3h*h + h*h + 2*h*f halves, 14 MB for GPT-2), one
// 128-byte line per prefetch, spread over the whole grid: the next layer streams from
// HBM while this one computes, so its TMA weight loads hit L2
__device__ void prefetch_layer_weights(const SmallArgs& a, const LayerW& w) {
  const int64_t h = a.h, f = a.f;
  const __half* mat[4] = {w.wqkv, w.wo, w.w1, w.w2};
  const int64_t n[4] = {3 * h * h, h * h, f * h, h * f};
  const int64_t nthr = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int m = 0; m < 4; ++m)
    for (int64_t line = tid; line < n[m] / 64; line += nthr) prefetch_l2(mat[m] + line * 64);
}

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float s = 0.0f;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) s += red[w];  // fixed order
  return s;
}

// x (fp32 row, already final) -> round16(LN(x)) into xn16.  Two-pass fp32 statistics
// like layernorm_lastdim (src/kernels.cpp:170-219): mean, population variance,
// inv = 1/sqrt(var + eps), y = gamma*((x - mean)*inv) + beta.  Row stages map thread t
// to columns [4t, 4t + 4) (h <= 1024): one 16-byte access per operand and split.
__device__ void ln_row(const float (&xv)[4], bool act, int h, const float* __restrict__ g,
                       const float* __restrict__ b, __half* __restrict__ out, float* red) {
  const int c = 4 * threadIdx.x;
  float4 gv = make_float4(0.f, 0.f, 0.f, 0.f), bv = gv;
  if (act) {  // parameter loads first: their latency overlaps the reductions
    gv = *reinterpret_cast<const float4*>(g + c);
    bv = *reinterpret_cast<const float4*>(b + c);
  }
  const float s = act ? __fadd_rn(__fadd_rn(__fadd_rn(xv[0], xv[1]), xv[2]), xv[3]) : 0.0f;
  const float mean = __fdiv_rn(block_sum(s, red), static_cast<float>(h));
  float q = 0.0f;
  if (act)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float d = __fsub_rn(xv[i], mean);
      q = __fmaf_rn(d, d, q);
    }
  const float var = __fdiv_rn(block_sum(q, red), static_cast<float>(h));
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
  if (act) {
    const float ga[4] = {gv.x, gv.y, gv.z, gv.w}, ba[4] = {bv.x, bv.y, bv.z, bv.w};
    uint32_t pk[2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
      pk[i] = h2_pack_rn(__fadd_rn(__fmul_rn(ga[2 * i], __fmul_rn(__fsub_rn(xv[2 * i], mean), inv)), ba[2 * i]),
                         __fadd_rn(__fmul_rn(ga[2 * i + 1], __fmul_rn(__fsub_rn(xv[2 * i + 1], mean), inv)),
                                   ba[2 * i + 1]));
    *reinterpret_cast<uint2*>(out + c) = make_uint2(pk[0], pk[1]);
  }
}

struct Ctl {
  uint64_t *full, *empty, *bfull, *accfull, *accempty;
  uint32_t tmem;
  uint32_t kc, tc;   // running k-block and task counters (barrier phases)
  int bpref;         // the next task's weights were already requested (prefetch)
};

// Weights (B) of one task into smem: issued by the producer thread as soon as the
// previous task's MMAs have consumed sB -- at the end of the previous stage, so the
// DRAM latency of the weights hides under the grid barrier.
// PAIR (M in (128, 256], CTA pairs of a 2-CTA cluster, cta_group::2 MMAs issued by the leader):
// each CTA loads half of the task's NT weight rows (rows n0 + rank * NT/2) into the same
// offset; the transaction bytes complete on the leader's barrier, the peer arrives remotely.
template <int NT, bool PAIR>
__device__ void load_b(Ctl& c, uint8_t* smem, const CUtensorMap* mB, int n0, int k0, int nkb) {
  if (threadIdx.x == 4 * 32) {
    if (!PAIR) {
      mbar_wait(c.accempty, (c.tc & 1) ^ 1);  // previous task's MMAs done reading sB
      mbar_expect_tx(c.bfull, static_cast<uint32_t>(nkb) * NT * 128);
      tma_load_3d(smem + SmemL::B, mB, c.bfull, 0, n0, k0 / 64);  // the task's whole B: one request
    } else {
      const uint32_t rank = cluster_ctarank() & 1;
      if (c.tc > 0) mbar_wait(c.accfull, (c.tc - 1) & 1);  // the pair's previous MMAs read this sB
      if (rank == 0) mbar_expect_tx(c.bfull, static_cast<uint32_t>(nkb) * NT * 128);  // both halves
      tma_load_3d_pair(smem + SmemL::B, mB, c.bfull, 0, n0 + static_cast<int>(rank) * (NT / 2), k0 / 64);
      if (rank != 0) mbar_arrive_cluster(to_leader(smem_u32(c.bfull)));
    }
  }
  c.bpref = 1;
}

// One GEMM task: D[128 x NT] = A[:, k0:k0+64*nkb] . B[n0:n0+NT, same]^T, then `EPI`.
// EPI 0: fp32 partial -> out32 (row pitch ld32); 1: round16(gelu(round16(round16(acc) + b)))
// -> out16; 2: round16(round16(acc) + b) -> out16.
template <int NT, int EPI, int KP, bool PAIR = false>
__device__ void gemm_task(const SmallArgs& a, uint8_t* smem, Ctl& c, const CUtensorMap* mA, const CUtensorMap* mB,
                          int n0, int k0, int nkb, float* out32, int64_t ld32, const float* bias, __half* out16,
                          int64_t ld16) {
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = PAIR ? (cluster_ctarank() & 1) : 0;  // PAIR: this CTA's 128 token rows
  uint8_t* sA = smem + SmemL::A;
  uint8_t* sB = smem + SmemL::B;
  if (!c.bpref) load_b<NT, PAIR>(c, smem, mB, n0, k0, nkb);
  c.bpref = 0;
  if (warp == 4) {
    if (lane == 0) {
      fence_proxy_async_global();  // A was written by generic stores of the previous stage
      for (int kb = 0; kb < nkb; kb += KP) {  // one request of KP k-blocks per ring slot
        const uint32_t u = c.kc + kb / KP, st = u % kStages;
        mbar_wait(&c.empty[st], ((u / kStages) & 1) ^ 1);
        if (!PAIR) {
          mbar_expect_tx(&c.full[st], KP * kABytes);
          tma_load_3d(sA + st * kKPR * kABytes, mA, &c.full[st], 0, 0, k0 / 64 + kb);
        } else {
          if (rank == 0) mbar_expect_tx(&c.full[st], 2 * KP * kABytes);  // both CTAs' rows
          tma_load_3d_pair(sA + st * kKPR * kABytes, mA, &c.full[st], 0, static_cast<int>(rank) * 128, k0 / 64 + kb);
          if (rank != 0) mbar_arrive_cluster(to_leader(smem_u32(&c.full[st])));
        }
      }
    }
    __syncwarp();
  } else if (warp == 5 && rank == 0) {
    if (lane == 0) {
      long long* gs = (a.dbg && blockIdx.x == 0 && c.tc < 64) ? a.dbg + 220000 + c.tc * 8 : nullptr;
      if (gs) gs[0] = globaltimer();
      constexpr uint32_t idesc = idesc_f16_f32(PAIR ? 256 : 128, NT, 0, 0);
      mbar_wait(c.accempty, (c.tc & 1) ^ 1);  // epilogue of the previous task read TMEM (PAIR: both CTAs')
      mbar_wait(c.bfull, c.tc & 1);
      if (gs) gs[1] = globaltimer();
      tc_fence_after();
      for (int kb = 0; kb < nkb; kb += KP) {
        const uint32_t u = c.kc + kb / KP, st = u % kStages;
        mbar_wait(&c.full[st], (u / kStages) & 1);
        if (gs && kb == 0) gs[2] = globaltimer();
        tc_fence_after();
#pragma unroll
        for (int j = 0; j < KP; ++j) {
          // the 3D box packs k-blocks at NT rows (PAIR: NT / 2 rows per CTA)
          const uint32_t a0 = smem_u32(sA + (st * kKPR + j) * kABytes),
                         b0 = smem_u32(sB + (kb + j) * ((PAIR ? NT / 2 : NT) * 128));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (PAIR)
              umma_f16_ss_pair(c.tmem, sw128_desc(a0 + kk * 32, 0, 1024), sw128_desc(b0 + kk * 32, 0, 1024), idesc,
                               (kb | j | kk) != 0);
            else
              umma_f16_ss(c.tmem, sw128_desc(a0 + kk * 32, 0, 1024), sw128_desc(b0 + kk * 32, 0, 1024), idesc,
                          (kb | j | kk) != 0);
          }
        }
        if (PAIR)
          umma_commit_pair(&c.empty[st]);  // both CTAs' A slots are free
        else
          umma_commit(&c.empty[st]);
      }
      if (PAIR)
        umma_commit_pair(c.accfull);
      else
        umma_commit(c.accfull);
      if (gs) gs[3] = globaltimer();
    }
    __syncwarp();
  }
  // epilogue on all 8 warps (the TMA and MMA warps join once their loops are issued):
  // warp w reads TMEM lane quadrant w % 4 (rows 32(w%4) ..), column half w / 4
  {
    constexpr int NH = NT / 2;
    const uint32_t quad = warp & 3, half = warp >> 2;
    const int c0 = n0 + static_cast<int>(half) * NH;
    float bv[NH];
    if (EPI != 0) {  // this half's biases before the accumulator wait (latency hidden under the MMAs)
#pragma unroll
      for (int i = 0; i < NH / 4; ++i) {
        const float4 b4 = reinterpret_cast<const float4*>(bias + c0)[i];
        bv[4 * i] = b4.x;
        bv[4 * i + 1] = b4.y;
        bv[4 * i + 2] = b4.z;
        bv[4 * i + 3] = b4.w;
      }
    }
    mbar_wait(c.accfull, c.tc & 1);
    if (a.dbg && blockIdx.x == 0 && c.tc < 64 && threadIdx.x == 0) a.dbg[220000 + c.tc * 8 + 4] = globaltimer();
    tc_fence_after();
    uint32_t u[NH];
    const uint32_t taddr = c.tmem + ((quad * 32) << 16) + half * NH;
    if constexpr (NH == 8) {
      tmem_ld8(taddr, u);
    } else if constexpr (NH == 24) {
      tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(u));
      tmem_ld8(taddr + 16, *reinterpret_cast<uint32_t(*)[8]>(u + 16));
    } else if constexpr (NH == 16) {
      tmem_ld16(taddr, u);
    } else {
      tmem_ld32(taddr, u);
    }
    tmem_wait_ld();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if (PAIR)
        mbar_arrive_cluster(to_leader(smem_u32(c.accempty)));  // the leader's MMAs reuse both TMEMs
      else
        mbar_arrive(c.accempty);
    }
    const int row = static_cast<int>(rank * 128 + quad * 32 + lane);
    if (row < a.M) {
      if (EPI == 0) {
        float4* o = reinterpret_cast<float4*>(out32 + static_cast<int64_t>(row) * ld32 + c0);
#pragma unroll
        for (int i = 0; i < NH / 4; ++i)
          o[i] = make_float4(__uint_as_float(u[4 * i]), __uint_as_float(u[4 * i + 1]), __uint_as_float(u[4 * i + 2]),
                             __uint_as_float(u[4 * i + 3]));
      } else {
        uint32_t pk[NH / 2];
#pragma unroll
        for (int i = 0; i < NH / 2; ++i) {
          uint32_t hh = h2_add_rn(h2_pack_rn(__uint_as_float(u[2 * i]), __uint_as_float(u[2 * i + 1])),
                                  h2_pack_rn(bv[2 * i], bv[2 * i + 1]));
          if (EPI == 1) {
            float x0, x1;
            h2_unpack(hh, x0, x1);
            gelu2_fast(x0, x1);
            hh = h2_pack_rn(x0, x1);
          }
          pk[i] = hh;
        }
        uint4* o = reinterpret_cast<uint4*>(out16 + static_cast<int64_t>(row) * ld16 + c0);
#pragma unroll
        for (int i = 0; i < NH / 8; ++i) o[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
    }
  }
  if (a.dbg && blockIdx.x == 0 && c.tc < 64 && threadIdx.x == 0) a.dbg[220000 + c.tc * 8 + 5] = globaltimer();
  c.kc += nkb / KP;  // ring slots used
  c.tc += 1;
}

// ---- warp-level tensor-core fragments (mma.sync m16n8k16, fp16 x fp16 -> fp32) for the
// attention tiles: 16 queries x <= 128 keys x 64 dims is far below one tcgen05 tile.
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_trans(uint32_t addr, uint32_t (&r)[2]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One (batch, head, 16-query block) of attention fused with its slice of the output
// projection (model.cpp:372-392 + the Wo Linear): scores round16(q.k * 0.125) (causal
// -inf), exact two-pass softmax p = round16(e / sum), ctx = round16(p . v), then the
// head's Wo partial ctx_h . Wo[:, head cols]^T -> part[head][rows] in fp32; the RLN2
// stage sums the heads' partials in head order.  q/k/v come from the QKV stage's fp16
// output (pitch 3h).
template <int QB>  // queries per task: 16 (one m16 row block) or 32 (two; CTA-pair mode, M > 128)
__device__ void attn_wo_task(const SmallArgs& a, uint8_t* smem, const CUtensorMap* mWo, uint64_t* wo_bar,
                             uint32_t wo_phase, int b, int hh, int q0, long long* ts) {
  constexpr int MB = QB / 16;
  // ts (debug, thread 0 only): [0] start [1] q/k/v staged [2] scores [3] softmax [4] ctx [5] Wo landed [6] done [7] row maxima
  if (ts) ts[0] = globaltimer();
  const int h = a.h, S = a.S;
  const uint32_t warp = warp_id(), lane = lane_id();
  uint8_t* sWo = smem;
  __half* sK = reinterpret_cast<__half*>(smem + h * 128);
  __half* sV = sK + 128 * kRowH;
  __half* sQ = sV + 128 * kRowH;
  __half* sC = sQ + QB * kRowH;
  float* sS = reinterpret_cast<float*>(sC + QB * kRowH);
  __half* sP = reinterpret_cast<__half*>(sS + QB * kRowS);
  const int kv = a.causal ? min(S, q0 + QB) : S;  // keys this block can see
  const int kvp = (kv + 15) & ~15;
  __syncthreads();  // the previous task's readers are done with the scratch
  if (threadIdx.x == 0) {  // the head's Wo column slice: h rows x 64 (128 B), 256-row boxes
    mbar_expect_tx(wo_bar, static_cast<uint32_t>(h) * 128);
    for (int r = 0; r < h; r += 256) tma_load_2d(sWo + r * 128, mWo, wo_bar, hh * 64, r);
  }
  {
    const __half* base = a.ff16 + static_cast<int64_t>(b) * S * 3 * h + hh * 64;
    const uint4 z = make_uint4(0, 0, 0, 0);
    // every load in flight before the first smem store: one L2 round trip, not four
    constexpr int PER = 128 * 8 / kThreads;  // 16-byte chunks per thread per tensor (<= 128 keys)
    uint4 kk[PER], vv[PER], qq = z;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + u * kThreads, j = e >> 3, c8 = (e & 7) * 8;
      kk[u] = z;
      vv[u] = z;
      if (j < kv) {
        kk[u] = *reinterpret_cast<const uint4*>(base + static_cast<int64_t>(j) * 3 * h + h + c8);
        vv[u] = *reinterpret_cast<const uint4*>(base + static_cast<int64_t>(j) * 3 * h + 2 * h + c8);
      }
    }
    const int qi = threadIdx.x >> 3, qc8 = (threadIdx.x & 7) * 8;
    if (threadIdx.x < QB * 8 && q0 + qi < S)
      qq = *reinterpret_cast<const uint4*>(base + static_cast<int64_t>(q0 + qi) * 3 * h + qc8);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = threadIdx.x + u * kThreads, j = e >> 3, c8 = (e & 7) * 8;
      if (j < kvp) {
        *reinterpret_cast<uint4*>(sK + j * kRowH + c8) = kk[u];
        *reinterpret_cast<uint4*>(sV + j * kRowH + c8) = vv[u];
      }
    }
    if (threadIdx.x < QB * 8) *reinterpret_cast<uint4*>(sQ + qi * kRowH + qc8) = qq;
  }
  __syncthreads();
  if (ts) ts[1] = globaltimer();
  // per-warp clock64 stamps of the same task (debug): lane 0 of each warp
  long long* wt = (a.dbg && q0 + QB >= S && hh == 0 && b == 0 && lane == 0)
                      ? a.dbg + 240000 + warp * 8 : nullptr;
  if (wt) wt[0] = clock64();
  const int g = lane >> 2, t4 = lane & 3;
  // scores: warp w -> keys [16w, 16w + 16), every 16-query row block; the columns past the
  // visible keys are written as -inf too, so the softmax below reads and writes all 128
  // columns without guards (guarded smem accesses under the trunk's register pressure
  // compile to one branch + address rematerialisation per access: 3-5x slower)
  {
    const bool live = static_cast<int>(warp) * 16 < kvp;
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
      float acc[2][4] = {};
      if (live) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          uint32_t af[4], bf[4];
          ldsm_x4(smem_u32(sQ + (mb * 16 + (lane & 15)) * kRowH + ks * 16 + (lane >> 4) * 8), af);
          ldsm_x4(smem_u32(sK + (warp * 16 + (lane & 7) + (lane >> 4) * 8) * kRowH + ks * 16 + ((lane >> 3) & 1) * 8), bf);
          mma16816(acc[0], af, bf[0], bf[1]);
          mma16816(acc[1], af, bf[2], bf[3]);
        }
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = mb * 16 + g + (e >> 1) * 8, j = warp * 16 + nt * 8 + 2 * t4 + (e & 1);
          const bool valid = j < kv && (!a.causal || j <= q0 + r);
          sS[r * kRowS + j] = valid ? r16(__fmul_rn(acc[nt][e], 0.125f)) : __int_as_float(0xff800000);
        }
    }
  }
  if (wt) wt[1] = clock64();
  __syncthreads();
  if (ts) ts[2] = globaltimer();
  if (wt) wt[2] = clock64();
  // softmax: warp w -> rows w * QB/8 .. (interleaved); lane -> keys lane + 32c
  {
    constexpr int RW = QB / 8;  // rows per warp
    float sc[RW][4], mx[RW], sum[RW], e[RW][4];
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
      mx[rr] = __int_as_float(0xff800000);
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int j = c4 * 32 + lane;
        sc[rr][c4] = sS[(warp * RW + rr) * kRowS + j];
        mx[rr] = fmaxf(mx[rr], sc[rr][c4]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int rr = 0; rr < RW; ++rr) mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], o));
    if (ts) ts[7] = globaltimer();
    if (wt) wt[3] = clock64();
    constexpr float LOG2E = 1.4426950408889634f;
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
      const float mxl = __fmul_rn(mx[rr], LOG2E);
      sum[rr] = 0.0f;
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        e[rr][c4] = ex2_approx(__fmaf_rn(sc[rr][c4], LOG2E, -mxl));  // exp(-inf) = 0 for masked keys
        sum[rr] = __fadd_rn(sum[rr], e[rr][c4]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int rr = 0; rr < RW; ++rr) sum[rr] = __fadd_rn(sum[rr], __shfl_xor_sync(0xffffffffu, sum[rr], o));
    if (wt) wt[4] = clock64();
#pragma unroll
    for (int rr = 0; rr < RW; ++rr) {
      const float inv = __frcp_rn(sum[rr]);
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int j = c4 * 32 + lane;
        sP[(warp * RW + rr) * kRowP + j] = __float2half_rn(__fmul_rn(e[rr][c4], inv));
      }
    }
  }
  if (wt) wt[5] = clock64();
  __syncthreads();
  if (ts) ts[3] = globaltimer();
  if (wt) wt[6] = clock64();
  // ctx = round16(P . V): warp w -> dims [8w, 8w + 8), every row block
#pragma unroll
  for (int mb = 0; mb < MB; ++mb) {
    float o[4] = {};
    for (int ks = 0; ks < kvp / 16; ++ks) {
      uint32_t af[4], bf[2];
      ldsm_x4(smem_u32(sP + (mb * 16 + (lane & 15)) * kRowP + ks * 16 + (lane >> 4) * 8), af);
      ldsm_x2_trans(smem_u32(sV + (ks * 16 + (lane & 15)) * kRowH + warp * 8), bf);
      mma16816(o, af, bf[0], bf[1]);
    }
    *reinterpret_cast<__half2*>(sC + (mb * 16 + g) * kRowH + warp * 8 + 2 * t4) = __floats2half2_rn(o[0], o[1]);
    *reinterpret_cast<__half2*>(sC + (mb * 16 + g + 8) * kRowH + warp * 8 + 2 * t4) = __floats2half2_rn(o[2], o[3]);
  }
  __syncthreads();
  if (ts) ts[4] = globaltimer();
  // Wo partial: out[QB][h] = ctx . WoSlice^T; warp w -> n-tiles [w * h/64, (w+1) * h/64) (pairs)
  mbar_wait(wo_bar, wo_phase);
  if (ts) ts[5] = globaltimer();
  // every row block's ctx fragments stay in registers, so each Wo fragment is loaded once for
  // all of them (QB = 32: half the ldmatrix traffic of a row-block-outer loop)
  uint32_t af[MB][4][4];
#pragma unroll
  for (int mb = 0; mb < MB; ++mb)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
      ldsm_x4(smem_u32(sC + (mb * 16 + (lane & 15)) * kRowH + ks * 16 + (lane >> 4) * 8), af[mb][ks]);
  {
    const int per_warp = h / 64;  // n-tiles of 8 columns per warp (h / 8 tiles over 8 warps)
    float* outp = a.part + static_cast<int64_t>(hh) * a.M * h;
    constexpr int kUnroll = MB == 1 ? 2 : 1;  // two independent column pairs in flight for one row block
#pragma unroll kUnroll
    for (int p2 = 0; p2 < per_warp; p2 += 2) {
      const int n0 = (warp * per_warp + p2) * 8;
      float d[MB][2][4] = {};
      const int n = n0 + (lane & 7) + (lane >> 4) * 8;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t bf[4];
        const int chunk = ks * 2 + ((lane >> 3) & 1);
        ldsm_x4(smem_u32(sWo + n * 128 + ((chunk ^ (n & 7)) << 4)), bf);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
          mma16816(d[mb][0], af[mb][ks], bf[0], bf[1]);
          mma16816(d[mb][1], af[mb][ks], bf[2], bf[3]);
        }
      }
#pragma unroll
      for (int mb = 0; mb < MB; ++mb) {
        const int row0 = b * S + q0 + mb * 16, qr = q0 + mb * 16;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int col = n0 + nt * 8 + 2 * t4;
          if (qr + g < S)
            *reinterpret_cast<float2*>(outp + static_cast<int64_t>(row0 + g) * h + col) =
                make_float2(d[mb][nt][0], d[mb][nt][1]);
          if (qr + g + 8 < S)
            *reinterpret_cast<float2*>(outp + static_cast<int64_t>(row0 + g + 8) * h + col) =
                make_float2(d[mb][nt][2], d[mb][nt][3]);
        }
      }
    }
  }
  if (ts) ts[6] = globaltimer();  // thread 0's warp (lane 0 issues the stamp after its own stores)
}

__device__ __forceinline__ float h2f_lo(uint32_t v) { return __half2float(__ushort_as_half(static_cast<unsigned short>(v & 0xFFFFu))); }
__device__ __forceinline__ float h2f_hi(uint32_t v) { return __half2float(__ushort_as_half(static_cast<unsigned short>(v >> 16))); }

// x[r] += round16(round16(sum_s part[s][r]) + bias); xn16[r] = round16(LN(x[r]))
template <int MAXSP>
__device__ void residual_ln_row(const SmallArgs& a, int r, int nsplit, const float* bias, const float* g,
                                const float* b, float* red, long long* ts = nullptr) {
  const int h = a.h, c = 4 * threadIdx.x;
  const bool act = c < h;
  if (ts && threadIdx.x == 0) ts[0] = globaltimer();
  float xv[4];
  if (act) {
    float4 pv[MAXSP];
#pragma unroll
    for (int sp = 0; sp < MAXSP; ++sp)  // every load of the row in flight before the ordered sums
      if (sp < nsplit) pv[sp] = *reinterpret_cast<const float4*>(a.part + (static_cast<int64_t>(sp) * a.M + r) * h + c);
    float4* xp = reinterpret_cast<float4*>(a.x + static_cast<int64_t>(r) * h + c);
    const float4 xo = *xp, bs = *reinterpret_cast<const float4*>(bias + c);
    float sum[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int sp = 0; sp < MAXSP; ++sp)
      if (sp < nsplit) {
        sum[0] = __fadd_rn(sum[0], pv[sp].x);
        sum[1] = __fadd_rn(sum[1], pv[sp].y);
        sum[2] = __fadd_rn(sum[2], pv[sp].z);
        sum[3] = __fadd_rn(sum[3], pv[sp].w);
      }
    xv[0] = __fadd_rn(xo.x, r16(__fadd_rn(r16(sum[0]), bs.x)));
    xv[1] = __fadd_rn(xo.y, r16(__fadd_rn(r16(sum[1]), bs.y)));
    xv[2] = __fadd_rn(xo.z, r16(__fadd_rn(r16(sum[2]), bs.z)));
    xv[3] = __fadd_rn(xo.w, r16(__fadd_rn(r16(sum[3]), bs.w)));
    *xp = make_float4(xv[0], xv[1], xv[2], xv[3]);
  }
  if (ts && threadIdx.x == 0) ts[1] = globaltimer();
  ln_row(xv, act, h, g, b, a.xn16 + static_cast<int64_t>(r) * h, red);
  if (ts && threadIdx.x == 0) ts[2] = globaltimer();
}

// PAIR = false: M <= 128, one CTA per GEMM task.  PAIR = true: 128 < M <= 256 on 2-CTA clusters,
// GEMM tasks per CTA pair (cta_group::2, M = 256: each CTA its 128 token rows, half the weight
// tile), so a task's MMA chain and per-CTA activation bytes stay those of M = 128; attention
// and row stages are per CTA as before.
// Two rows at once (M > grid): threads [0, 128) row r0, [128, 256) row r1 (if r1 >= 0), VPT
// consecutive columns per thread (h = 128 VPT); the same operations as residual_ln_row /
// ln_row, with each half's block sums over its 4 warps (named barrier per half).
template <int MAXSP, int VPT>
__device__ void residual_ln_rows2(const SmallArgs& a, int r0, int r1, int nsplit, const float* bias, const float* g,
                                  const float* b, float* red, bool final_out) {
  const int h = a.h, half = threadIdx.x >> 7, t = threadIdx.x & 127, c = VPT * t;
  const int r = half ? r1 : r0;
  const bool act = r >= 0;
  const uint32_t wid = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31;
  float* rh = red + 8 + 8 * half;  // [2][4] partials per half (red[0..7] is ln_row's)
  float xv[VPT];
  float gv[VPT], bv[VPT];
  if (act) {
    // partial sums in split order, streamed (the compiler keeps as many loads in flight as
    // registers allow; holding all MAXSP x VPT values spills)
    float psum[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) psum[i] = 0.0f;
#pragma unroll 4
    for (int sp = 0; sp < nsplit; ++sp)
#pragma unroll
      for (int i = 0; i < VPT; i += 2) {
        const float2 v2 = __ldcg(reinterpret_cast<const float2*>(a.part + (static_cast<int64_t>(sp) * a.M + r) * h + c + i));
        psum[i] = __fadd_rn(psum[i], v2.x);
        psum[i + 1] = __fadd_rn(psum[i + 1], v2.y);
      }
    float xo[VPT], bs[VPT];
#pragma unroll
    for (int i = 0; i < VPT; i += 2) {
      const float2 x2 = *reinterpret_cast<const float2*>(a.x + static_cast<int64_t>(r) * h + c + i);
      const float2 b2 = *reinterpret_cast<const float2*>(bias + c + i);
      const float2 g2 = *reinterpret_cast<const float2*>(g + c + i);
      const float2 e2 = *reinterpret_cast<const float2*>(b + c + i);
      xo[i] = x2.x;
      xo[i + 1] = x2.y;
      bs[i] = b2.x;
      bs[i + 1] = b2.y;
      gv[i] = g2.x;
      gv[i + 1] = g2.y;
      bv[i] = e2.x;
      bv[i + 1] = e2.y;
    }
#pragma unroll
    for (int i = 0; i < VPT; ++i) xv[i] = __fadd_rn(xo[i], r16(__fadd_rn(r16(psum[i]), bs[i])));
#pragma unroll
    for (int i = 0; i < VPT; i += 2)
      *reinterpret_cast<float2*>(a.x + static_cast<int64_t>(r) * h + c + i) = make_float2(xv[i], xv[i + 1]);
  }
  auto half_sum = [&](float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    named_bar_sync(2 + half, 128);
    if (lane == 0) rh[wid] = v;
    named_bar_sync(2 + half, 128);
    return (rh[0] + rh[1]) + (rh[2] + rh[3]);  // fixed order
  };
  float s = 0.0f;
  if (act)
#pragma unroll
    for (int i = 0; i < VPT; ++i) s = __fadd_rn(s, xv[i]);
  const float mean = __fdiv_rn(half_sum(s), static_cast<float>(h));
  float q = 0.0f;
  if (act)
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const float d = __fsub_rn(xv[i], mean);
      q = __fmaf_rn(d, d, q);
    }
  const float var = __fdiv_rn(half_sum(q), static_cast<float>(h));
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
  if (act) {
    __half* out = a.xn16 + static_cast<int64_t>(r) * h + c;
#pragma unroll
    for (int i = 0; i < VPT; i += 2)
      *reinterpret_cast<uint32_t*>(out + i) =
          h2_pack_rn(__fadd_rn(__fmul_rn(gv[i], __fmul_rn(__fsub_rn(xv[i], mean), inv)), bv[i]),
                     __fadd_rn(__fmul_rn(gv[i + 1], __fmul_rn(__fsub_rn(xv[i + 1], mean), inv)), bv[i + 1]));
  }
  (void)final_out;
}

// N1P: the CTA-pair kernel's FFN1 task width (64, or 48 when it divides ffn: 64 tasks on the
// 74 pairs instead of 48, a quarter less GELU epilogue per CTA)
template <bool PAIR, int N1P = 64>
__global__ void __launch_bounds__(kThreads, 1) fwd_small_kernel(const __grid_constant__ SmallArgs a) {
  // no static shared memory in this kernel: the dynamic window starts 1024-aligned, and
  // indexing it directly keeps every access in the shared state space (LDS/STS)
  extern __shared__ __align__(1024) uint8_t smem[];
  const int h = a.h, f = a.f, M = a.M, S = a.S, H = a.H;
  const uint32_t warp = warp_id(), lane = lane_id();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SmemL::BAR);
  float* red = reinterpret_cast<float*>(bars + 16);  // [8] ln_row, [8..24) residual_ln_rows2
  uint32_t* tslot = reinterpret_cast<uint32_t*>(red + 24);
  Ctl c;
  c.full = bars;
  c.empty = bars + kStages;
  c.bfull = bars + 2 * kStages;
  c.accfull = bars + 2 * kStages + 1;
  c.accempty = bars + 2 * kStages + 2;
  uint64_t* wo_bar = bars + 2 * kStages + 3;  // the attention task's Wo slice (TMA)
  uint32_t n_att = 0;                         // attention tasks run by this CTA (wo_bar phase)
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&c.full[i], PAIR ? 2 : 1);  // PAIR: both CTAs' producers arrive on the leader's
      mbar_init(&c.empty[i], 1);
    }
    mbar_init(c.bfull, PAIR ? 2 : 1);
    mbar_init(c.accfull, 1);
    mbar_init(c.accempty, PAIR ? 16 : 8);  // every warp (PAIR: of both CTAs) reads its TMEM slice
    mbar_init(wo_bar, 1);
    fence_barrier_init();
  }
  if (PAIR) cluster_sync_all();  // barrier inits visible to the peer before any remote arrival
  if (warp == 5) {
    if (PAIR) {
      tmem_alloc_pair(tslot, 64);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(tslot, 32);
      tmem_relinquish();
    }
  }
  if (warp == 6)
    for (int i = lane; i < 2 + 4 * a.L; i += 32) tma_prefetch_desc(&a.maps[i]);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  c.tmem = *tslot;
  c.kc = 0;
  c.tc = 0;
  c.bpref = 0;
  unsigned target = 0;
  const bool flags = a.qkv_flags != nullptr;  // stage hand-offs through counters, not grid barriers
  auto release_add = [&](unsigned* ctr, unsigned n) {  // this CTA's stores, then +n (all threads call)
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(ctr), "r"(n) : "memory");
  };
  auto wait_ge = [&](const unsigned* ctr, unsigned want) {  // all threads call
    if (threadIdx.x == 0) spin_acquire(ctr, want, 3, static_cast<int>(ctr - a.gbar));
    __syncthreads();
  };
  const unsigned pairx = PAIR ? 2u : 1u;  // CTAs counting each pair task
  // debug (flag mode): per-CTA end time of each stage, [layer][6][grid] (scripts/flag_timeline.py)
  auto stamp = [&](int l, int stage) {
    if (a.dbg && flags && threadIdx.x == 0)
      a.dbg[250000 + (static_cast<int64_t>(l) * 6 + stage) * gridDim.x + blockIdx.x] = globaltimer();
  };
  const CUtensorMap* mXn = a.maps + 0;
  const CUtensorMap* mFf = a.maps + 1;
  // task geometry (same on every CTA; PAIR: per CTA pair, N per pair task)
  constexpr int NQ = PAIR ? 32 : 16, N1 = PAIR ? N1P : kTileN, N2 = PAIR ? 64 : kTileN;
  const int gid = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int gn = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  const int t_qkv = 3 * h / NQ;                 // full K -> fp16 q/k/v
  const int t_ffn1 = f / N1;                    // full K, GELU
  const int t_ffn2 = (h / N2) * a.split_ffn2;   // tiles x K splits -> partials
  const int kb_ffn2 = f / 64 / a.split_ffn2;
  auto pre_qkv = [&](int l) {
    if (gid < t_qkv) load_b<NQ, PAIR>(c, smem, a.maps + 2 + 4 * l + 0, gid * NQ, 0, h / 64);
  };
  auto pre_ffn1 = [&](int l) {
    if (gid < t_ffn1) load_b<N1, PAIR>(c, smem, a.maps + 2 + 4 * l + 2, gid * N1, 0, h / 64);
  };
  auto pre_ffn2 = [&](int l) {
    const int t = gid;
    if (t < t_ffn2)
      load_b<N2, PAIR>(c, smem, a.maps + 2 + 4 * l + 3, (t / a.split_ffn2) * N2, (t % a.split_ffn2) * kb_ffn2 * 64,
                       kb_ffn2);
  };

  // ---- stage 0: embedding gather (bit-exact fp32 tok + pos) + LN1 of layer 0
  if (!a.embed_only) pre_qkv(0);  // (no TMA may be in flight when an embed-only launch exits)
  prefetch_layer_params(a, a.lw[0]);
  prefetch_layer_weights(a, a.lw[0]);
  for (int r = blockIdx.x; r < M; r += gridDim.x) {
    const int id = a.ids[r];
    const bool ok = id >= 0 && id < a.V;
    if (!ok && threadIdx.x == 0) atomicExch(a.err, 1);
    const int t = r % S, cc = 4 * threadIdx.x;
    const bool act = cc < h;
    float xv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (act) {
      const float4 pe = *reinterpret_cast<const float4*>(a.pos + static_cast<int64_t>(t) * h + cc);
      const float4 te = ok ? *reinterpret_cast<const float4*>(a.tok + static_cast<int64_t>(id) * h + cc)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      xv[0] = __fadd_rn(te.x, pe.x);
      xv[1] = __fadd_rn(te.y, pe.y);
      xv[2] = __fadd_rn(te.z, pe.z);
      xv[3] = __fadd_rn(te.w, pe.w);
      *reinterpret_cast<float4*>(a.x + static_cast<int64_t>(r) * h + cc) = make_float4(xv[0], xv[1], xv[2], xv[3]);
    }
    ln_row(xv, act, h, a.lw[0].ln1g, a.lw[0].ln1b, a.xn16 + static_cast<int64_t>(r) * h, red);
  }
  if (!flags) {
    grid_sync(a.gbar, target, a.dbg);
  } else if (static_cast<int>(blockIdx.x) < M) {
    release_add(a.rows1_done, static_cast<unsigned>((M - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1));
  }

  for (int l = 0; l < (a.embed_only ? 0 : a.L); ++l) {
    const LayerW& w = a.lw[l];
    const CUtensorMap* mW = a.maps + 2 + 4 * l;
    if (l + 1 < a.L) {
      prefetch_layer_params(a, a.lw[l + 1]);
      prefetch_layer_weights(a, a.lw[l + 1]);
    }
    // ---- QKV: N=16 tiles, full K, round16(round16(acc) + b) -> fp16 q|k|v (ff16 buffer)
    // QKV -> attention without a grid barrier (a.qkv_flags): each task releases a counter once
    // its q/k/v columns are stored (both CTAs of a pair count), and an attention task acquires
    // only the 12 (pair: 6) tasks holding its head's q, k and v -- one L2 hop instead of the
    // barrier's two, and no wait for unrelated heads
    if (flags && gid < t_qkv) wait_ge(a.rows1_done, static_cast<unsigned>(M * (l + 1)));  // every xn16 row
    if (a.dbg && flags && threadIdx.x == 0) a.dbg[262000 + l * gridDim.x + blockIdx.x] = globaltimer();  // (debug)
    for (int t = gid; t < t_qkv; t += gn) {
      gemm_task<NQ, 2, 4, PAIR>(a, smem, c, mXn, mW + 0, t * NQ, 0, h / 64, nullptr, 0, w.bqkv, a.ff16, 3 * h);
      if (a.qkv_flags) {
        __syncthreads();  // every thread's q/k/v stores precede the release
        if (threadIdx.x == 0) {
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.qkv_flags + t) : "memory");
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.qkv_done) : "memory");
        }
      }
    }
    stamp(l, 0);
    if (!a.qkv_flags) grid_sync(a.gbar, target, a.dbg);
    // ---- attention + Wo: (batch, head, 16-query block) tasks, head partials -> part[head]
    {
      // PAIR (M > 128): 32-query tasks -- at most 96 for S <= 128, one round on 148 CTAs
      const bool q32 = a.q32 != 0;  // (host: CTA-pair mode and h <= 768, where the 32-query scratch fits)
      const int QB = q32 ? 32 : kQB;
      const int nqb = (S + QB - 1) / QB;
      long long* ats = (a.dbg && blockIdx.x == 0 && threadIdx.x == 0) ? a.dbg + 210000 + l * 8 : nullptr;
      if (ats) ats[0] = globaltimer();
      for (int t = blockIdx.x; t < a.B * H * nqb; t += gridDim.x) {
        const int qb = t % nqb, hh = (t / nqb) % H, b = t / (nqb * H);
        // generic reads of the previous task's Wo slice before this task's TMA rewrites it
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        // debug stamps: the heaviest causal task of head 0 (last query block)
        long long* ts = (a.dbg && qb == nqb - 1 && hh == 0 && b == 0 && threadIdx.x == 0) ? a.dbg + 230000 + l * 8 : nullptr;
        if (a.qkv_flags) {  // this head's q | k | v column tasks are stored (acquire; attn_wo_task's
                            // opening __syncthreads orders the whole CTA's loads after it)
          constexpr int PER = 64 / NQ;
          if (static_cast<int>(threadIdx.x) < 3 * PER) {
            const int sec = static_cast<int>(threadIdx.x) / PER, j = static_cast<int>(threadIdx.x) % PER;
            const int task = (sec * h + hh * 64) / NQ + j;
            spin_acquire(a.qkv_flags + task, static_cast<unsigned>(l + 1) * (PAIR ? 2u : 1u), 0, task);
          }
        }
        if (q32)
          attn_wo_task<32>(a, smem, mW + 1, wo_bar, n_att & 1, b, hh, qb * QB, ts);
        else
          attn_wo_task<kQB>(a, smem, mW + 1, wo_bar, n_att & 1, b, hh, qb * QB, ts);
        ++n_att;
        if (a.qkv_flags) {  // this task's Wo partial rows are stored
          __syncthreads();
          if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.attn_flags + t) : "memory");
        }
      }
      if (ats) ats[1] = globaltimer();
      stamp(l, 1);
      // the scratch (generic writes) overlaps the B region the FFN1 weights are fetched into
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      pre_ffn1(l);
    }
    if (!a.qkv_flags) grid_sync(a.gbar, target, a.dbg);
    // rows of a query block wait for its H attention tasks (and for every QKV task: the row
    // stage rewrites xn16, the QKV GEMMs' A operand)
    auto wait_row = [&](int r, int tid0) {
      const int QB = a.q32 ? 32 : kQB, nqb = (S + QB - 1) / QB;
      const int i = static_cast<int>(threadIdx.x) - tid0;
      if (r < 0 || i < 0 || i > H) return;
      const unsigned* f = i < H ? a.attn_flags + ((r / S) * H + i) * nqb + (r % S) / QB : a.qkv_done;
      const unsigned want = i < H ? static_cast<unsigned>(l + 1)
                                  : static_cast<unsigned>((l + 1) * t_qkv) * (PAIR ? 2u : 1u);
      spin_acquire(f, want, 1, r);
    };
    // ---- residual + LN2: x += round16(round16(sum over heads of the Wo partials) + bo)
    if (PAIR && M > static_cast<int>(gridDim.x) && h == 768 && H <= 12) {  // two rows per CTA at once
      for (int r = blockIdx.x; r < M; r += 2 * gridDim.x) {
        const int r2 = r + static_cast<int>(gridDim.x) < M ? r + static_cast<int>(gridDim.x) : -1;
        if (a.qkv_flags) {
          wait_row(r, 0);
          wait_row(r2, 32);
          __syncthreads();
        }
        residual_ln_rows2<12, 6>(a, r, r2, H, w.bo, w.ln2g, w.ln2b, red, false);
      }
    } else {
      for (int r = blockIdx.x; r < M; r += gridDim.x) {
        if (a.qkv_flags) {
          wait_row(r, 0);
          __syncthreads();
        }
        residual_ln_row<16>(a, r, H, w.bo, w.ln2g, w.ln2b, red,
                            (a.dbg && blockIdx.x == 0) ? a.dbg + 200000 + l * 8 : nullptr);
      }
    }
    stamp(l, 2);
    const unsigned my_rows = static_cast<int>(blockIdx.x) < M
                                 ? static_cast<unsigned>((M - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1)
                                 : 0u;
    if (!flags)
      grid_sync(a.gbar, target, a.dbg);
    else if (my_rows)
      release_add(a.rows2_done, my_rows);
    if (flags && gid < t_ffn1) wait_ge(a.rows2_done, static_cast<unsigned>(M * (l + 1)));  // every LN2 row
    if (a.dbg && flags && threadIdx.x == 0) a.dbg[264000 + l * gridDim.x + blockIdx.x] = globaltimer();  // (debug)
    // ---- FFN1 + GELU, full K
    for (int t = gid; t < t_ffn1; t += gn) {
      gemm_task<N1, 1, 4, PAIR>(a, smem, c, mXn, mW + 2, t * N1, 0, h / 64, nullptr, 0, w.b1, a.ff16, f);
      if (a.qkv_flags) {  // this task's GELU columns are stored
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.ffn1_flags + t) : "memory");
      }
    }
    pre_ffn2(l);
    stamp(l, 3);
    if (!a.qkv_flags) grid_sync(a.gbar, target, a.dbg);
    // ---- FFN2: partials over K splits (a split waits only for the FFN1 tasks of its K range;
    // gemm_task's TMA warp fences the generic->async proxy before loading them)
    for (int t = gid; t < t_ffn2; t += gn) {
      if (a.qkv_flags) {
        // the FFN1 tasks whose columns overlap this split's K range
        const int c0 = (t % a.split_ffn2) * kb_ffn2 * 64, t_lo = c0 / N1, t_hi = (c0 + kb_ffn2 * 64 - 1) / N1;
        const int i = static_cast<int>(threadIdx.x);
        if (i <= t_hi - t_lo) {
          const int task = t_lo + i;
          spin_acquire(a.ffn1_flags + task, static_cast<unsigned>(l + 1) * (PAIR ? 2u : 1u), 2, task);
        }
        __syncthreads();
      }
      gemm_task<N2, 0, 4, PAIR>(a, smem, c, mFf, mW + 3, (t / a.split_ffn2) * N2, (t % a.split_ffn2) * kb_ffn2 * 64,
                                kb_ffn2, a.part + static_cast<int64_t>(t % a.split_ffn2) * M * h, h, nullptr, nullptr,
                                0);
      if (flags) release_add(a.ffn2_done, 1u);
    }
    if (l + 1 < a.L) pre_qkv(l + 1);
    stamp(l, 4);
    if (!flags)
      grid_sync(a.gbar, target, a.dbg);
    else if (my_rows)
      wait_ge(a.ffn2_done, static_cast<unsigned>(t_ffn2 * (l + 1)) * pairx);  // every K-split partial
    // ---- residual + LN1 of the next layer (or the final LN)
    {
      const float* g = l + 1 < a.L ? a.lw[l + 1].ln1g : a.lnfg;
      const float* bb = l + 1 < a.L ? a.lw[l + 1].ln1b : a.lnfb;
      if (PAIR && M > static_cast<int>(gridDim.x) && h == 768) {
        for (int r = blockIdx.x; r < M; r += 2 * gridDim.x)
          residual_ln_rows2<8, 6>(a, r, r + static_cast<int>(gridDim.x) < M ? r + static_cast<int>(gridDim.x) : -1,
                                  a.split_ffn2, w.b2, g, bb, red, false);
      } else {
        for (int r = blockIdx.x; r < M; r += gridDim.x) residual_ln_row<8>(a, r, a.split_ffn2, w.b2, g, bb, red);
      }
    }
    if (!flags) {
      if (l + 1 < a.L) grid_sync(a.gbar, target, a.dbg);
    } else if (my_rows && l + 1 < a.L) {
      release_add(a.rows1_done, my_rows);
    }
    stamp(l, 5);
  }
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();  // the peer's remote arrivals / MMAs on this CTA are done
  if (warp == 5) {
    tc_fence_after();
    if (PAIR)
      tmem_dealloc_pair(c.tmem, 64);
    else
      tmem_dealloc(c.tmem, 32);
  }
}

constexpr size_t kSmem = SmemL::BAR + 16 * 8 + 24 * 4 + 16;
static_assert(kFlagFfn1 - kFlagQkv >= 3 * 1024 / 16 && kFlagAttn - kFlagFfn1 >= 4096 / 32 &&
                  kFlagAttn + 256 * 16 <= kBarRegionBytes / 4,
              "per-task flags fit the barrier region (max tasks: QKV 3h/16, FFN1 f/32, attention B*H*ceil(S/16))");
static_assert(kSmem <= 227 * 1024, "fwd_small smem");


}  // namespace

long long*& small_debug_stamps() {
  static long long* p = nullptr;
  return p;
}

bool fwd_small_supported(int64_t M, int64_t S, int64_t h, int64_t f, int64_t hd, int64_t L) {
  if (std::getenv("PRLAB_NO_FWD_SMALL")) return false;
  const int64_t max_m = std::getenv("PRLAB_NO_SMALL_PAIR") ? 128 : 256;  // 128 < M <= 256: CTA-pair kernel
  return L <= kMaxLayers && M >= 1 && M <= max_m && S <= 128 && hd == 64 && L >= 1 && h % 256 == 0 && h <= 1024 && f % 512 == 0 &&
         h / 64 <= kMaxKB && (f / 512) <= 8 && (f / 512) * 64 <= kMaxKB * 64;
}

int fwd_small_pair_n1(int64_t f) {  // the CTA-pair kernel's FFN1 task width
  return (f % 48 == 0 && !std::getenv("PRLAB_SMALL_N1_64")) ? 48 : 64;
}

size_t fwd_small_workspace_floats(int64_t M, int64_t h, int64_t f) {
  const int64_t heads = h / 64, sp_ffn2 = f / 512;  // Wo partials per head, FFN2 K splits
  return static_cast<size_t>(std::max(heads, sp_ffn2) * M * h + 64);
}

void launch_fwd_small(const FwdSmallPlan& p, cudaStream_t st) {
  static std::mutex mu;
  static uint64_t done = 0;
  once_per_device(mu, done, [] {
    PRLAB_CUDA(cudaFuncSetAttribute(fwd_small_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmem)));
    PRLAB_CUDA(cudaFuncSetAttribute(fwd_small_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmem)));
    PRLAB_CUDA(cudaFuncSetAttribute(fwd_small_kernel<true, 48>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmem)));
  });
  // 28 KB of kernel parameters, copied at launch: one per host thread (models driven from
  // several threads each launch with their own maps and weights), not on the stack
  static thread_local SmallArgs a;
  a = SmallArgs{};
  a.M = p.M;
  a.B = p.B;
  a.S = p.S;
  a.h = p.h;
  a.f = p.f;
  a.H = p.H;
  a.L = p.L;
  a.V = p.V;
  a.causal = p.causal;
  a.split_ffn2 = p.f / 512;
  a.embed_only = p.embed_only;
  {
    const char* e = std::getenv("PRLAB_SMALL_Q32");  // A/B switch: 0 / 1 forces 16 / 32-query tasks
    a.q32 = (e && *e) ? (std::atoi(e) != 0 && p.h <= 768) : (p.M > 128 && p.h <= 768);
  }
  if (p.L > kMaxLayers) throw std::invalid_argument("fwd_small: too many layers");
  std::memcpy(a.maps, p.host_maps, sizeof(CUtensorMap) * (2 + 4 * p.L));
  std::memcpy(a.lw, p.host_lw, sizeof(LayerW) * p.L);
  a.tok = p.tok;
  a.pos = p.pos;
  a.lnfg = p.lnfg;
  a.lnfb = p.lnfb;
  a.ids = p.ids;
  a.err = p.err;
  a.x = p.x;
  a.xn16 = p.xn16;
  a.ff16 = p.ff16;
  a.part = p.scratch;
  a.gbar = p.gbar;
  {  // the bar region: [0] grid barrier, [1] QKV-done counter, then the per-task flags
    const bool barriers = std::getenv("PRLAB_SMALL_BARRIERS") || std::getenv("PRLAB_SMALL_QKV_BARRIER");
    a.qkv_flags = barriers ? nullptr : p.gbar + kFlagQkv;
    a.qkv_done = p.gbar + 1;
    a.rows1_done = p.gbar + 2;
    a.rows2_done = p.gbar + 3;
    a.ffn2_done = p.gbar + 4;
    a.ffn1_flags = p.gbar + kFlagFfn1;
    a.attn_flags = p.gbar + kFlagAttn;
  }
  a.dbg = small_debug_stamps();
  PRLAB_CUDA(cudaMemsetAsync(p.gbar, 0, kBarRegionBytes, st));  // the barrier counter and the QKV flags
  const bool pair = p.M > 128;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pair ? num_sms() & ~1 : num_sms());
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pair ? 2 : 1;
  if (pair)
    if (fwd_small_pair_n1(p.f) == 48)
      PRLAB_CUDA(cudaLaunchKernelEx(&cfg, fwd_small_kernel<true, 48>, a));
    else
      PRLAB_CUDA(cudaLaunchKernelEx(&cfg, fwd_small_kernel<true>, a));
  else
    PRLAB_CUDA(cudaLaunchKernelEx(&cfg, fwd_small_kernel<false>, a));
}

}  // namespace prlab_gpu
