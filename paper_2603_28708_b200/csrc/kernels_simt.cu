// SIMT CUDA kernels: the generic (any shape, any per-class policy) path and the
// HBM-bound LayerNorm / embedding kernels of the fast path.
//
// The generic kernels keep fp32 storage and honour the reference KernelConfig
// of each op class exactly: inputs conformed onto the compute lattice,
// F16E accumulation rounded after every product and partial sum in ascending
// order (src/kernels.cpp:55-66), outputs conformed.  Products of fp16-lattice
// values are exact in fp32, so fmaf() is bit-identical to the reference's
// separate multiply+add under the hybrid config.
#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline int blocks_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < (1 << 30) ? b : (1 << 30));
}

// ---------------------------------------------------------------------------
// generic GEMM: out[m, n] = epi( sum_k A[m, k] * Bt[n, k] )  (reference matmul +
// linear_bias + fused GELU / residual).  64x64 tile, BK 16, 256 threads, 4x4
// outputs per thread, ascending-k accumulation per output.
// MODE 0: F32/F32 (fmaf)   1: F16E/F32 (inputs rounded; fmaf exact)   2: F16E/F16E
// ---------------------------------------------------------------------------
struct GemmEpiDev {
  const float* bias;
  int op;
  int lin_c, act_c, res_c;
  const float* resid;
};

template <int MODE>
__global__ void __launch_bounds__(256) simt_gemm_kernel(const float* __restrict__ A, int64_t lda,
                                                        const float* __restrict__ Bt, int64_t ldb,
                                                        float* out, int64_t ldo, int M, int N,
                                                        int K, GemmEpiDev e) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;

  for (int k0 = 0; k0 < K; k0 += 16) {
    // 64 rows x 16 k for A and Bt: 1024 values each, 4 per thread
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = threadIdx.x + i * 256;
      const int r = idx >> 4, kk = idx & 15;
      float av = 0.0f, bv = 0.0f;
      if (m0 + r < M && k0 + kk < K) av = A[static_cast<int64_t>(m0 + r) * lda + k0 + kk];
      if (n0 + r < N && k0 + kk < K) bv = Bt[static_cast<int64_t>(n0 + r) * ldb + k0 + kk];
      if (MODE != 0) {
        av = r16(av);
        bv = r16(bv);
      }
      As[kk][r] = av;
      Bs[kk][r] = bv;
    }
    __syncthreads();
    const int kmax = min(16, K - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (MODE == 2)
            acc[i][j] = r16(__fadd_rn(acc[i][j], r16(__fmul_rn(a[i], b[j]))));
          else
            acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = conform(acc[i][j], e.lin_c);
      if (e.bias) v = conform(__fadd_rn(v, conform(e.bias[n], e.lin_c)), e.lin_c);
      if (e.op == 1) {
        const float x = conform(v, e.act_c);
        v = conform(gelu_erf(x), e.act_c);
      } else if (e.op == 2) {
        const float x = conform(e.resid[static_cast<int64_t>(m) * ldo + n], e.res_c);
        v = conform(__fadd_rn(x, conform(v, e.res_c)), e.res_c);
      }
      out[static_cast<int64_t>(m) * ldo + n] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// embedding gather + add, reference src/kernels.cpp:256-294
// ---------------------------------------------------------------------------
__global__ void simt_embed_kernel(const float* __restrict__ tok, int64_t vocab,
                                  const float* __restrict__ pos, int h,
                                  const int32_t* __restrict__ ids, int B, int S, int c16,
                                  float* __restrict__ out, int* err) {
  const int64_t total = static_cast<int64_t>(B) * S * h;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / h;
    const int c = static_cast<int>(i % h);
    const int32_t id = ids[r];
    if (id < 0 || id >= vocab) {
      if (err) atomicExch(err, 1);
      out[i] = 0.0f;
      continue;
    }
    const float t = conform(tok[static_cast<int64_t>(id) * h + c], c16);
    const float p = conform(pos[static_cast<int64_t>(r % S) * h + c], c16);
    out[i] = conform(__fadd_rn(t, p), c16);
  }
}

// fast path: fp32 gather + add with float4 (h % 4 == 0); bit-exact with the reference.
__global__ void embed_f32_kernel(const float4* __restrict__ tok, int64_t vocab,
                                 const float4* __restrict__ pos, int h4,
                                 const int32_t* __restrict__ ids, int S, int64_t rows,
                                 float4* __restrict__ out, int* err) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = rows * h4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / h4;
    const int c = static_cast<int>(i % h4);
    const int32_t id = __ldg(ids + r);
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if (id < 0 || id >= vocab) {
      if (err) atomicExch(err, 1);
    } else {
      const float4 t = __ldg(tok + static_cast<int64_t>(id) * h4 + c);
      const float4 p = __ldg(pos + static_cast<int64_t>(r % S) * h4 + c);
      o = make_float4(__fadd_rn(t.x, p.x), __fadd_rn(t.y, p.y), __fadd_rn(t.z, p.z),
                      __fadd_rn(t.w, p.w));
    }
    out[i] = o;
  }
}

// ---------------------------------------------------------------------------
// LayerNorm, reference src/kernels.cpp:170-219.  One warp per row.  F32
// accumulation uses warp-shuffle reductions (fp32 reassociation only); F16E
// accumulation runs the reference's sequential rounded recurrence on lane 0.
// ---------------------------------------------------------------------------
__global__ void simt_layernorm_kernel(const float* __restrict__ x, int rows, int n,
                                      const float* __restrict__ gamma,
                                      const float* __restrict__ beta, float eps, int c16, int a16,
                                      float* __restrict__ out32, __half* __restrict__ out16,
                                      int round_out16) {
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* in = x + static_cast<int64_t>(row) * n;
  float mean, inv;
  if (!a16) {
    float s = 0.0f;
    for (int i = lane; i < n; i += 32) s += conform(in[i], c16);
    s = warp_sum(s);
    mean = __fdiv_rn(s, static_cast<float>(n));
    float vs = 0.0f;
    for (int i = lane; i < n; i += 32) {
      const float d = __fsub_rn(conform(in[i], c16), mean);
      vs = __fadd_rn(vs, __fmul_rn(d, d));
    }
    vs = warp_sum(vs);
    const float var = __fdiv_rn(vs, static_cast<float>(n));
    inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, eps)));
  } else {
    float m = 0.0f, iv = 0.0f;
    if (lane == 0) {
      float s = 0.0f;
      for (int i = 0; i < n; ++i) s = r16(__fadd_rn(s, conform(in[i], c16)));
      m = r16(__fdiv_rn(s, static_cast<float>(n)));
      float vs = 0.0f;
      for (int i = 0; i < n; ++i) {
        const float d = r16(__fsub_rn(conform(in[i], c16), m));
        vs = r16(__fadd_rn(vs, r16(__fmul_rn(d, d))));
      }
      const float var = r16(__fdiv_rn(vs, static_cast<float>(n)));
      iv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, eps)));
    }
    mean = __shfl_sync(0xffffffffu, m, 0);
    inv = __shfl_sync(0xffffffffu, iv, 0);
  }
  for (int i = lane; i < n; i += 32) {
    const float g = conform(gamma[i], c16), b = conform(beta[i], c16);
    float y = conform(
        __fadd_rn(__fmul_rn(g, __fmul_rn(__fsub_rn(conform(in[i], c16), mean), inv)), b), c16);
    if (out16) {
      out16[static_cast<int64_t>(row) * n + i] = __float2half_rn(y);
    } else {
      if (round_out16) y = r16(y);
      out32[static_cast<int64_t>(row) * n + i] = y;
    }
  }
}

// Fast-path LayerNorm (hybrid: F32 LN, output consumed by an F16E Linear, so the
// round16 of the next op is applied here).  One warp per row, n = 128*VPT,
// row held in registers (two-pass mean / variance like the reference).
template <int VPT>
__global__ void __launch_bounds__(256) ln_f16_kernel(const float* x, int rows,
                                                     const float* __restrict__ gamma,
                                                     const float* __restrict__ beta, float eps,
                                                     __half* __restrict__ out, float* x_round) {
  // Persistent warps over rows (grid-stride, as many blocks as are co-resident), the next
  // row's loads issued before the current row's reductions, so DRAM stays busy through the
  // reduction and store phases (C4: 15.2 -> 14.2 us per call; a TMA bulk-copy ring of 4
  // rows per warp measured slower, 19.2 us -- 3 KB requests).
  constexpr int n = 128 * VPT;
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * 8;
  int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  pdl_trigger();
  pdl_wait();  // x is produced by the upstream residual GEMM
  if (row >= rows) return;
  float4 nxt[VPT];
  {
    const float4* in = reinterpret_cast<const float4*>(x + static_cast<int64_t>(row) * n);
#pragma unroll
    for (int i = 0; i < VPT; ++i) nxt[i] = __ldg(in + lane + 32 * i);
  }
  for (; row < rows; row += stride) {
    float4 v[VPT];
#pragma unroll
    for (int i = 0; i < VPT; ++i) v[i] = nxt[i];
    if (x_round) {
      // full_fp16 fast path: the residual stream lives on the binary16 lattice (Residual
      // class F16E, kernels.cpp:237-254): the fp32 sum the residual GEMM added in L2 is
      // rounded here, once, before anything reads it -- round16(x + y) exactly
      float4* w = reinterpret_cast<float4*>(x_round + static_cast<int64_t>(row) * n);
#pragma unroll
      for (int i = 0; i < VPT; ++i) {
        v[i] = make_float4(r16(v[i].x), r16(v[i].y), r16(v[i].z), r16(v[i].w));
        w[lane + 32 * i] = v[i];
      }
    }
    if (row + stride < rows) {
      const float4* in = reinterpret_cast<const float4*>(x + static_cast<int64_t>(row + stride) * n);
#pragma unroll
      for (int i = 0; i < VPT; ++i) nxt[i] = __ldg(in + lane + 32 * i);
    }
    ln_row_f16<VPT>(v, lane, gamma, beta, eps, out + static_cast<int64_t>(row) * n);
  }
}

// ---------------------------------------------------------------------------
// generic attention (any S, any head_dim): one warp per query row.
// scores (kernels.cpp:85-125) -> causal mask (model.cpp:405-413) -> softmax
// (kernels.cpp:127-168, sequential sum like the reference) -> P.V (matmul).
// ---------------------------------------------------------------------------
__global__ void simt_attention_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                      const float* __restrict__ v, int64_t ld_in,
                                      float* __restrict__ ctx, int64_t ld_ctx, int B, int S, int H,
                                      int hd, float scale, int causal, Kcfg att, Kcfg sm,
                                      float* __restrict__ tap) {
  extern __shared__ float sh[];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* srow = sh + w * (S + hd);
  float* qrow = srow + S;
  const int64_t gq = static_cast<int64_t>(blockIdx.x) * warps + w;  // (b, h, i) flattened
  if (gq >= static_cast<int64_t>(B) * H * S) return;
  const int i = static_cast<int>(gq % S);
  const int head = static_cast<int>((gq / S) % H);
  const int b = static_cast<int>(gq / (static_cast<int64_t>(S) * H));
  const int ac = att.compute, aa = att.accum;
  for (int t = lane; t < hd; t += 32)
    qrow[t] = conform(q[(static_cast<int64_t>(b) * S + i) * ld_in + head * hd + t], ac);
  __syncwarp();
  for (int j = lane; j < S; j += 32) {
    const float* kr = k + (static_cast<int64_t>(b) * S + j) * ld_in + head * hd;
    float value, ref = 0.0f;
    if (aa) {
      float acc = 0.0f;
      for (int t = 0; t < hd; ++t) acc = r16(__fadd_rn(acc, r16(__fmul_rn(qrow[t], conform(kr[t], ac)))));
      value = r16(__fmul_rn(acc, scale));
      if (tap)
        for (int t = 0; t < hd; ++t) ref = __fadd_rn(ref, __fmul_rn(qrow[t], conform(kr[t], ac)));
      ref = __fmul_rn(ref, scale);
    } else {
      float acc = 0.0f;
      for (int t = 0; t < hd; ++t) acc = __fadd_rn(acc, __fmul_rn(qrow[t], conform(kr[t], ac)));
      ref = __fmul_rn(acc, scale);
      value = conform(ref, ac);
    }
    if (tap) tap[((static_cast<int64_t>(b) * H + head) * S + i) * S + j] = ref;
    if (causal && j > i) value = __int_as_float(0xff800000);
    srow[j] = conform(value, sm.compute);
  }
  __syncwarp();
  float shift = 0.0f;
  if (sm.stabilized) {
    float mx = __int_as_float(0xff800000);
    for (int j = lane; j < S; j += 32) mx = fmaxf(mx, srow[j]);
    shift = warp_max(mx);
  }
  for (int j = lane; j < S; j += 32) {
    const float e = sm.stabilized ? expf(__fsub_rn(srow[j], shift)) : expf(srow[j]);
    srow[j] = conform(e, sm.compute);
  }
  __syncwarp();
  float sum = 0.0f;
  if (lane == 0) {
    if (sm.accum)
      for (int j = 0; j < S; ++j) sum = r16(__fadd_rn(sum, srow[j]));
    else
      for (int j = 0; j < S; ++j) sum = __fadd_rn(sum, srow[j]);
    sum = conform(sum, sm.compute);
  }
  sum = __shfl_sync(0xffffffffu, sum, 0);
  for (int j = lane; j < S; j += 32)
    srow[j] = conform(conform(__fdiv_rn(srow[j], sum), sm.compute), ac);  // probs onto att lattice
  __syncwarp();
  for (int t = lane; t < hd; t += 32) {
    float acc = 0.0f;
    const float* vc = v + static_cast<int64_t>(b) * S * ld_in + head * hd + t;
    if (aa) {
      for (int j = 0; j < S; ++j) acc = r16(__fadd_rn(acc, r16(__fmul_rn(srow[j], conform(vc[j * ld_in], ac)))));
    } else {
      for (int j = 0; j < S; ++j) acc = __fadd_rn(acc, __fmul_rn(srow[j], conform(vc[j * ld_in], ac)));
      acc = conform(acc, ac);
    }
    ctx[(static_cast<int64_t>(b) * S + i) * ld_ctx + head * hd + t] = acc;
  }
}

// ---------------------------------------------------------------------------
// fp32-policy attention (att = F32/F32, softmax F32 stabilised; hd 64, S <= 512, no tap):
// register-tiled two-pass form.  One CTA per (b, head, 64-query block): scores
// s = (q . k) * scale (causal -inf after scaling, model.cpp:405-413) for the whole key range
// into shared memory, exact softmax p = e / sum with e = expf(s - max) (kernels.cpp:127-168),
// then ctx = P . V.  The same operations as simt_attention_kernel in fp32; only the summation
// orders differ (4x4 register tiles, fmaf, warp-tree row sums) -- the fp32 parity budget
// (1e-3 relative) is the reference's own fp32-vs-fp32 contract.  One warp per query row
// with sequential sums (simt_attention_kernel) measured 859 us per layer at BERT s512.
// ---------------------------------------------------------------------------
constexpr int kAtQ = 64, kAtD = 64, kAtPad = 68;
__global__ void __launch_bounds__(256) attn_f32_tiled_kernel(const float* __restrict__ q, const float* __restrict__ k,
                                                             const float* __restrict__ v, int64_t ld_in,
                                                             float* __restrict__ ctx, int64_t ld_ctx, int S, int H,
                                                             float scale, int causal) {
  extern __shared__ __align__(16) float sh[];
  float* sQt = sh;                      // [d][q]  (transposed, padded)
  float* sKV = sQt + kAtD * kAtPad;     // K tile transposed [d][key], then V tile [key][d]
  float* sS = sKV + kAtD * kAtPad;      // [q][S + 4] scores / probabilities
  const int ldS = S + 4;
  const int qb = blockIdx.x, head = blockIdx.y, b = blockIdx.z;
  const int q0 = qb * kAtQ, nq = min(kAtQ, S - q0);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int kend = causal ? min(S, q0 + nq) : S;  // keys any query of the block sees
  const float* qbase = q + (static_cast<int64_t>(b) * S) * ld_in + head * kAtD;
  const float* kbase = k + (static_cast<int64_t>(b) * S) * ld_in + head * kAtD;
  const float* vbase = v + (static_cast<int64_t>(b) * S) * ld_in + head * kAtD;
  for (int e = tid; e < kAtQ * kAtD; e += 256) {
    const int r = e >> 6, d = e & 63;
    sQt[d * kAtPad + r] = r < nq ? qbase[static_cast<int64_t>(q0 + r) * ld_in + d] : 0.0f;
  }
  // ---- scores, 64 keys at a time
  for (int j0 = 0; j0 < kend; j0 += 64) {
    __syncthreads();  // sKV free (previous tile's readers done); sQt visible
    for (int e = tid; e < 64 * kAtD; e += 256) {
      const int r = e >> 6, d = e & 63;
      sKV[d * kAtPad + r] = j0 + r < S ? kbase[static_cast<int64_t>(j0 + r) * ld_in + d] : 0.0f;
    }
    __syncthreads();
    float acc[4][4] = {};
#pragma unroll 8
    for (int d = 0; d < kAtD; ++d) {
      const float4 a4 = *reinterpret_cast<const float4*>(sQt + d * kAtPad + 4 * ty);
      const float4 b4 = *reinterpret_cast<const float4*>(sKV + d * kAtPad + 4 * tx);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w}, bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = fmaf(a[i], bb[jj], acc[i][jj]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int qi = 4 * ty + i;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = j0 + 4 * tx + jj;
        if (j < kend) {
          const float sv = __fmul_rn(acc[i][jj], scale);
          sS[qi * ldS + j] = (causal && j > q0 + qi) ? __int_as_float(0xff800000) : sv;
        }
      }
    }
  }
  __syncthreads();
  // ---- softmax per row: warp w -> rows w, w + 8, ...
  {
    const int w = tid >> 5, lane = tid & 31;
    for (int r = w; r < nq; r += 8) {
      float* row = sS + r * ldS;
      float mx = __int_as_float(0xff800000);
      for (int j = lane; j < kend; j += 32) mx = fmaxf(mx, row[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      float sum = 0.0f;
      for (int j = lane; j < kend; j += 32) {
        const float e = expf(__fsub_rn(row[j], mx));
        row[j] = e;
        sum = __fadd_rn(sum, e);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum = __fadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
      for (int j = lane; j < kend; j += 32) row[j] = __fdiv_rn(row[j], sum);
    }
  }
  // ---- ctx = P . V, 64 keys at a time; thread: queries 4ty.., dims 4tx..
  float o[4][4] = {};
  for (int j0 = 0; j0 < kend; j0 += 64) {
    __syncthreads();  // probabilities written / previous V tile consumed
    for (int e = tid; e < 64 * kAtD; e += 256) {
      const int r = e >> 6, d = e & 63;
      sKV[r * kAtPad + d] = j0 + r < S ? vbase[static_cast<int64_t>(j0 + r) * ld_in + d] : 0.0f;
    }
    __syncthreads();
    const int jn = min(64, kend - j0);
    for (int jj = 0; jj < jn; ++jj) {
      const float4 v4 = *reinterpret_cast<const float4*>(sKV + jj * kAtPad + 4 * tx);
      const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float pv = sS[(4 * ty + i) * ldS + j0 + jj];
#pragma unroll
        for (int dd = 0; dd < 4; ++dd) o[i][dd] = fmaf(pv, vv[dd], o[i][dd]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int qi = 4 * ty + i;
    if (qi < nq)
      *reinterpret_cast<float4*>(ctx + (static_cast<int64_t>(b) * S + q0 + qi) * ld_ctx + head * kAtD + 4 * tx) =
          make_float4(o[i][0], o[i][1], o[i][2], o[i][3]);
  }
}

// per-op softmax (kernels.cpp:127-168): one warp per row, sequential sum.
__global__ void simt_softmax_kernel(const float* __restrict__ x, int64_t rows, int64_t n, Kcfg cfg,
                                    float* __restrict__ out) {
  const int warps = blockDim.x >> 5;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* in = x + row * n;
  float* o = out + row * n;
  float shift = 0.0f;
  if (cfg.stabilized) {
    float mx = __int_as_float(0xff800000);
    for (int64_t j = lane; j < n; j += 32) mx = fmaxf(mx, conform(in[j], cfg.compute));
    shift = warp_max(mx);
  }
  for (int64_t j = lane; j < n; j += 32) {
    const float xv = conform(in[j], cfg.compute);
    o[j] = conform(cfg.stabilized ? expf(__fsub_rn(xv, shift)) : expf(xv), cfg.compute);
  }
  __syncwarp();
  float sum = 0.0f;
  if (lane == 0) {
    for (int64_t j = 0; j < n; ++j) sum = cfg.accum ? r16(__fadd_rn(sum, o[j])) : __fadd_rn(sum, o[j]);
    sum = conform(sum, cfg.compute);
  }
  sum = __shfl_sync(0xffffffffu, sum, 0);
  for (int64_t j = lane; j < n; j += 32) o[j] = conform(__fdiv_rn(o[j], sum), cfg.compute);
}

__global__ void simt_gelu_kernel(const float* x, int64_t n, int c16, float* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = conform(gelu_erf(conform(x[i], c16)), c16);
}
__global__ void simt_add_kernel(const float* a, const float* b, int64_t n, int c16, float* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = conform(__fadd_rn(conform(a[i], c16), conform(b[i], c16)), c16);
}
__global__ void simt_tanh_kernel(const float* x, int64_t n, int c16, float* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = conform(tanhf(conform(x[i], c16)), c16);
}
__global__ void round_copy_kernel(const float* x, int64_t n, int c16, float* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = conform(x[i], c16);
}
__global__ void f32_to_f16_kernel(const float* x, __half* out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = __float2half_rn(x[i]);
}
__global__ void convert_f16_f32_kernel(const __half* __restrict__ in, int64_t ld_in,
                                       float* __restrict__ out, int64_t ld_out, int M, int N) {
  pdl_trigger();
  pdl_wait();
  const int64_t total = static_cast<int64_t>(M) * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / N, c = i % N;
    out[r * ld_out + c] = __half2float(in[r * ld_in + c]);
  }
}
// out[c, r] = in[r, c] (rows x cols -> cols x rows), 32x32 smem tiles
template <typename OutT>
__global__ void transpose_kernel(const float* __restrict__ in, int rows, int cols,
                                 OutT* __restrict__ out, int64_t ld_out, int rnd) {
  __shared__ float tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (r < rows && c < cols) ? in[static_cast<int64_t>(r) * cols + c] : 0.0f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) {
      const float v = tile[threadIdx.x][i];
      if constexpr (sizeof(OutT) == 2)
        out[static_cast<int64_t>(c) * ld_out + r] = __float2half_rn(v);
      else
        out[static_cast<int64_t>(c) * ld_out + r] = rnd ? r16(v) : v;
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
void simt_gemm(const float* A, int64_t lda, const float* Bt, int64_t ldb, float* out, int64_t ldo,
               int M, int N, int K, Kcfg lin, const SimtGemmEpi& epi, cudaStream_t st) {
  GemmEpiDev e{epi.bias, epi.op, lin.compute, epi.act.compute, epi.res.compute, epi.resid};
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  if (lin.compute == 0)
    simt_gemm_kernel<0><<<grid, 256, 0, st>>>(A, lda, Bt, ldb, out, ldo, M, N, K, e);
  else if (lin.accum == 0)
    simt_gemm_kernel<1><<<grid, 256, 0, st>>>(A, lda, Bt, ldb, out, ldo, M, N, K, e);
  else
    simt_gemm_kernel<2><<<grid, 256, 0, st>>>(A, lda, Bt, ldb, out, ldo, M, N, K, e);
  PRLAB_CUDA(cudaGetLastError());
}

void simt_embed(const float* tok, int64_t vocab, const float* pos, int h, const int32_t* ids,
                int B, int S, Kcfg cfg, float* out, int* err, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(B) * S * h;
  simt_embed_kernel<<<blocks_for(n, 256), 256, 0, st>>>(tok, vocab, pos, h, ids, B, S, cfg.compute,
                                                         out, err);
  PRLAB_CUDA(cudaGetLastError());
}

void embed_f32(const float* tok, int64_t vocab, const float* pos, int h, const int32_t* ids, int B,
               int S, float* out, int* err, cudaStream_t st) {
  const int64_t rows = static_cast<int64_t>(B) * S;
  const int h4 = h / 4;
  const int64_t n = rows * h4;
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, num_sms() * 8));
  launch_pdl(embed_f32_kernel, dim3(blocks), dim3(256), 0, st, reinterpret_cast<const float4*>(tok), vocab,
             reinterpret_cast<const float4*>(pos), h4, ids, S, rows, reinterpret_cast<float4*>(out), err);
}

void simt_layernorm(const float* x, int rows, int n, const float* gamma, const float* beta,
                    float eps, Kcfg cfg, float* out32, __half* out16, int round_out16,
                    cudaStream_t st) {
  simt_layernorm_kernel<<<(rows + 7) / 8, 256, 0, st>>>(x, rows, n, gamma, beta, eps, cfg.compute,
                                                        cfg.accum, out32, out16, round_out16);
  PRLAB_CUDA(cudaGetLastError());
}

// persistent warps: as many 256-thread blocks as are co-resident (register-bound)
template <int VPT>
void launch_ln(const float* x, int rows, const float* gamma, const float* beta, float eps, __half* out,
               cudaStream_t st, float* x_round) {
  static int per_sm_dev[64] = {};
  int& per_sm = per_sm_dev[current_device() & 63];
  if (per_sm == 0) {
    int v = 0;
    PRLAB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, ln_f16_kernel<VPT>, 256, 0));
    per_sm = std::max(1, v);
  }
  const int grid = std::min((rows + 7) / 8, num_sms() * per_sm);
  launch_pdl(ln_f16_kernel<VPT>, dim3(grid), dim3(256), 0, st, x, rows, gamma, beta, eps, out, x_round);
}

void ln_f32_to_f16(const float* x, int rows, int n, const float* gamma, const float* beta,
                   float eps, __half* out, cudaStream_t st, float* x_round) {
  switch (n) {
    case 128: launch_ln<1>(x, rows, gamma, beta, eps, out, st, x_round); break;
    case 256: launch_ln<2>(x, rows, gamma, beta, eps, out, st, x_round); break;
    case 384: launch_ln<3>(x, rows, gamma, beta, eps, out, st, x_round); break;
    case 512: launch_ln<4>(x, rows, gamma, beta, eps, out, st, x_round); break;
    case 768: launch_ln<6>(x, rows, gamma, beta, eps, out, st, x_round); break;
    case 1024: launch_ln<8>(x, rows, gamma, beta, eps, out, st, x_round); break;
    default:
      if (x_round) throw std::invalid_argument("fp16-lattice LayerNorm needs h in {128..1024, step 128}");
      simt_layernorm(x, rows, n, gamma, beta, eps, Kcfg{0, 0, 1}, nullptr, out, 0, st);
      return;
  }
}

void simt_attention(const float* q, const float* k, const float* v, int64_t ld_in, float* ctx,
                    int64_t ld_ctx, int B, int S, int H, int hd, float scale, int causal, Kcfg att,
                    Kcfg sm, float* tap, cudaStream_t st) {
  // plain fp32 configs: the register-tiled kernel (same operations, other summation order)
  if (tap == nullptr && hd == kAtD && S <= 512 && att.compute == 0 && att.accum == 0 && sm.compute == 0 &&
      sm.accum == 0 && sm.stabilized && ld_in % 4 == 0 && ld_ctx % 4 == 0 && !std::getenv("PRLAB_NO_ATTN_F32_TILED")) {
    const size_t shm = static_cast<size_t>(2 * kAtD * kAtPad + kAtQ * (S + 4)) * sizeof(float);
    static std::mutex mu;
    static uint64_t done = 0;
    once_per_device(mu, done, [] {
      PRLAB_CUDA(cudaFuncSetAttribute(attn_f32_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>((2 * kAtD * kAtPad + kAtQ * (512 + 4)) * sizeof(float))));
    });
    attn_f32_tiled_kernel<<<dim3((S + kAtQ - 1) / kAtQ, H, B), 256, shm, st>>>(q, k, v, ld_in, ctx, ld_ctx, S, H, scale,
                                                                                causal);
    PRLAB_CUDA(cudaGetLastError());
    return;
  }
  const int warps = 4;
  const size_t shmem = static_cast<size_t>(warps) * (S + hd) * sizeof(float);
  {
    static std::mutex mu;
    static int configured_bytes[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    int& cb = configured_bytes[current_device() & 63];
    if (cb == 0) cb = 48 * 1024;
    if (shmem > static_cast<size_t>(cb)) {
      PRLAB_CUDA(cudaFuncSetAttribute(simt_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(shmem)));
      cb = static_cast<int>(shmem);
    }
  }
  const int64_t rows = static_cast<int64_t>(B) * H * S;
  simt_attention_kernel<<<static_cast<int>((rows + warps - 1) / warps), warps * 32, shmem, st>>>(
      q, k, v, ld_in, ctx, ld_ctx, B, S, H, hd, scale, causal, att, sm, tap);
  PRLAB_CUDA(cudaGetLastError());
}

void simt_scores(const float* q, const float* k, int sq, int sk, int d, float scale, Kcfg cfg,
                 float* out, float* tap, cudaStream_t st);

void simt_softmax(const float* x, int64_t rows, int64_t n, Kcfg cfg, float* out, cudaStream_t st) {
  simt_softmax_kernel<<<static_cast<int>((rows + 7) / 8), 256, 0, st>>>(x, rows, n, cfg, out);
  PRLAB_CUDA(cudaGetLastError());
}
void simt_gelu(const float* x, int64_t n, Kcfg cfg, float* out, cudaStream_t st) {
  simt_gelu_kernel<<<blocks_for(n, 256), 256, 0, st>>>(x, n, cfg.compute, out);
  PRLAB_CUDA(cudaGetLastError());
}
void simt_add(const float* a, const float* b, int64_t n, Kcfg cfg, float* out, cudaStream_t st) {
  simt_add_kernel<<<blocks_for(n, 256), 256, 0, st>>>(a, b, n, cfg.compute, out);
  PRLAB_CUDA(cudaGetLastError());
}
// classifier_probs mean pool (src/model.cpp:496-511): one thread per (batch row, column),
// tokens summed in order under the Linear accumulation contract, then conform(acc / S).
__global__ void pool_mean_kernel(const float* x32, const __half* x16, int B, int S, int h, int c16, int a16,
                                 float* out) {
  const int b = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || c >= h) return;
  float acc = 0.0f;
  for (int t = 0; t < S; ++t) {
    const int64_t i = (static_cast<int64_t>(b) * S + t) * h + c;
    const float xv = conform(x16 ? __half2float(x16[i]) : x32[i], c16);
    acc = a16 ? r16(__fadd_rn(acc, xv)) : __fadd_rn(acc, xv);
  }
  out[static_cast<int64_t>(b) * h + c] = conform(__fdiv_rn(acc, static_cast<float>(S)), c16);
}
void simt_pool_mean(const float* x32, const __half* x16, int B, int S, int h, Kcfg lin, float* out,
                    cudaStream_t st) {
  pool_mean_kernel<<<dim3((h + 127) / 128, B), 128, 0, st>>>(x32, x16, B, S, h, lin.compute, lin.accum, out);
  PRLAB_CUDA(cudaGetLastError());
}
void simt_tanh(const float* x, int64_t n, Kcfg cfg, float* out, cudaStream_t st) {
  simt_tanh_kernel<<<blocks_for(n, 256), 256, 0, st>>>(x, n, cfg.compute, out);
  PRLAB_CUDA(cudaGetLastError());
}
void simt_round_copy(const float* x, int64_t n, int f16, float* out, cudaStream_t st) {
  round_copy_kernel<<<blocks_for(n, 256), 256, 0, st>>>(x, n, f16, out);
  PRLAB_CUDA(cudaGetLastError());
}
void round16_inplace(float* x, int64_t n, cudaStream_t st) { simt_round_copy(x, n, 1, x, st); }
void f32_to_f16(const float* in, __half* out, int64_t n, cudaStream_t st) {
  f32_to_f16_kernel<<<blocks_for(n, 256), 256, 0, st>>>(in, out, n);
  PRLAB_CUDA(cudaGetLastError());
}
void convert_f16_to_f32(const __half* in, int64_t ld_in, float* out, int64_t ld_out, int M, int N,
                        cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(M) * N;
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, num_sms() * 16));
  launch_pdl(convert_f16_f32_kernel, dim3(blocks), dim3(256), 0, st, in, ld_in, out, ld_out, M, N);
}
void transpose_f32(const float* in, int rows, int cols, float* out, int rnd, cudaStream_t st) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
  transpose_kernel<float><<<grid, block, 0, st>>>(in, rows, cols, out, rows, rnd);
  PRLAB_CUDA(cudaGetLastError());
}
void transpose_to_f16(const float* in, int rows, int cols, __half* out, int64_t ld_out,
                      cudaStream_t st) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
  transpose_kernel<__half><<<grid, block, 0, st>>>(in, rows, cols, out, ld_out, 0);
  PRLAB_CUDA(cudaGetLastError());
}

// per-op attention_scores (kernels.cpp:85-125) via the generic attention
// machinery would compute more than asked; a dedicated tiny kernel instead.
namespace {
__global__ void simt_scores_kernel(const float* __restrict__ q, const float* __restrict__ k, int sq,
                                   int sk, int d, float scale, Kcfg cfg, float* out, float* tap) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<int64_t>(sq) * sk) return;
  const int i = static_cast<int>(idx / sk), j = static_cast<int>(idx % sk);
  const float* qr = q + static_cast<int64_t>(i) * d;
  const float* kr = k + static_cast<int64_t>(j) * d;
  const int c = cfg.compute;
  float value;
  if (cfg.accum) {
    float acc = 0.0f;
    for (int t = 0; t < d; ++t) acc = r16(__fadd_rn(acc, r16(__fmul_rn(conform(qr[t], c), conform(kr[t], c)))));
    value = r16(__fmul_rn(acc, scale));
    if (tap) {
      float ref = 0.0f;
      for (int t = 0; t < d; ++t) ref = __fadd_rn(ref, __fmul_rn(conform(qr[t], c), conform(kr[t], c)));
      tap[idx] = __fmul_rn(ref, scale);
    }
  } else {
    float acc = 0.0f;
    for (int t = 0; t < d; ++t) acc = __fadd_rn(acc, __fmul_rn(conform(qr[t], c), conform(kr[t], c)));
    const float scaled = __fmul_rn(acc, scale);
    if (tap) tap[idx] = scaled;
    value = conform(scaled, c);
  }
  out[idx] = value;
}
}  // namespace

void simt_scores(const float* q, const float* k, int sq, int sk, int d, float scale, Kcfg cfg,
                 float* out, float* tap, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(sq) * sk;
  simt_scores_kernel<<<blocks_for(n, 128), 128, 0, st>>>(q, k, sq, sk, d, scale, cfg, out, tap);
  PRLAB_CUDA(cudaGetLastError());
}

namespace {
template <typename T>
__global__ void argmax_kernel(const T* __restrict__ x, int64_t n, int64_t ld, int32_t* out) {
  const T* row = x + static_cast<int64_t>(blockIdx.x) * ld;
  float best = __int_as_float(0xff800000);
  int idx = 0x7fffffff;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const float v = static_cast<float>(row[j]);
    if (v > best || (v == best && j < idx)) {
      best = v;
      idx = static_cast<int>(j);
    }
  }
  __shared__ float sb[32];
  __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ob > best || (ob == best && oi < idx)) {
      best = ob;
      idx = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sb[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (sb[w] > best || (sb[w] == best && si[w] < idx)) {
        best = sb[w];
        idx = si[w];
      }
    out[blockIdx.x] = idx == 0x7fffffff ? 0 : idx;
  }
}
}  // namespace

void argmax_rows(const void* logits, int dtype, int64_t rows, int64_t n, int64_t ld, int32_t* out,
                 cudaStream_t st) {
  if (dtype == 1)
    argmax_kernel<__half><<<static_cast<int>(rows), 512, 0, st>>>(static_cast<const __half*>(logits), n, ld, out);
  else
    argmax_kernel<float><<<static_cast<int>(rows), 512, 0, st>>>(static_cast<const float*>(logits), n, ld, out);
  PRLAB_CUDA(cudaGetLastError());
}

}  // namespace prlab_gpu
