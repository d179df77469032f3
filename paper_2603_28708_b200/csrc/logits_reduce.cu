// Device-side reductions over logits: the statistics the
// reference computes on host logits (src/fidelity.cpp) evaluated where the logits
// live, so perplexity / greedy decoding / fidelity checks read the [M, V] logits
// once from HBM instead of copying them to the host (1.65 GB fp16 at C4).
//
//  * row_nll_kernel     one CTA per row: row max, sum_v exp(x_v - max) (fp32 exp,
//                       double accumulation), NLL of the target token
//                       -((x_t - max) - log(denom)) like window_nll_sum
//                       (fidelity.cpp:213-240), argmax (lowest index on ties);
//                       a non-finite row max yields NaN (the reference's poison).
//  * compare_rows_kernel one CTA per row: compare_logits (fidelity.cpp:11-37)
//                       partials in double -- finite pairs, non-finite candidates,
//                       max |b-c|, sum |b-c|, sum b*c, sum b*b, sum c*c; the host
//                       folds the rows in order (deterministic).
// Both read 16-byte vectors where the row pitch allows and size the grid by rows.
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {

template <typename T>
__device__ __forceinline__ float ld_val(const T* p, int64_t j) {
  return static_cast<float>(p[j]);
}
template <>
__device__ __forceinline__ float ld_val<__half>(const __half* p, int64_t j) {
  return __half2float(p[j]);
}

constexpr int kThreads = 256;

template <typename T, typename R>
__device__ R block_reduce(R v, R (*op)(R, R), R* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  R r = sh[0];
  for (int w = 1; w < kThreads / 32; ++w) r = op(r, sh[w]);  // fixed order: deterministic
  return r;
}
__device__ float op_max(float a, float b) { return fmaxf(a, b); }
__device__ double op_addd(double a, double b) { return a + b; }
__device__ double op_maxd(double a, double b) { return fmax(a, b); }
__device__ unsigned long long op_addu(unsigned long long a, unsigned long long b) { return a + b; }

template <typename T>
__global__ void __launch_bounds__(kThreads) row_nll_kernel(const T* __restrict__ x, int64_t n, int64_t ld,
                                                           const int32_t* __restrict__ targets,
                                                           double* __restrict__ nll, int32_t* __restrict__ amax) {
  __shared__ float shf[32];
  __shared__ double shd[32];
  __shared__ int shi[32];
  const T* row = x + static_cast<int64_t>(blockIdx.x) * ld;
  // pass 1: max and argmax (lowest index among equal maxima)
  float best = __int_as_float(0xff800000);
  int idx = 0x7fffffff;
  bool nonfinite = false;
  for (int64_t j = threadIdx.x; j < n; j += kThreads) {
    const float v = ld_val(row, j);
    nonfinite |= !isfinite(v) && !(isinf(v) && v < 0.0f);
    if (v > best || (v == best && j < idx)) {
      best = v;
      idx = static_cast<int>(j);
    }
  }
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
    shf[threadIdx.x >> 5] = best;
    shi[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w)
      if (shf[w] > best || (shf[w] == best && shi[w] < idx)) {
        best = shf[w];
        idx = shi[w];
      }
    shf[0] = best;
    shi[0] = idx;
  }
  __syncthreads();
  const float mx = shf[0];
  if (amax != nullptr && threadIdx.x == 0) amax[blockIdx.x] = shi[0];
  const int any_bad = __syncthreads_or(nonfinite ? 1 : 0);
  if (nll == nullptr) return;
  // pass 2: denominator in double over fp32 exponentials
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += kThreads) s += static_cast<double>(expf(ld_val(row, j) - mx));
  s = block_reduce<T, double>(s, op_addd, shd);
  if (threadIdx.x == 0) {
    const int32_t t = targets != nullptr ? targets[blockIdx.x] : -1;
    if (t < 0 || t >= n) {
      nll[blockIdx.x] = 0.0;  // no target for this row (last position of a window)
    } else if (!isfinite(mx) || any_bad) {
      nll[blockIdx.x] = __longlong_as_double(0x7ff8000000000000ll);  // NaN poison
    } else {
      nll[blockIdx.x] = -((static_cast<double>(ld_val(row, t)) - mx) - log(s));
    }
  }
}

template <typename TB, typename TC>
__global__ void __launch_bounds__(kThreads) compare_rows_kernel(const TB* __restrict__ b, int64_t ldb,
                                                                const TC* __restrict__ c, int64_t ldc,
                                                                int64_t n, double* __restrict__ part) {
  __shared__ double shd[32];
  __shared__ unsigned long long shu[32];
  const TB* rb = b + static_cast<int64_t>(blockIdx.x) * ldb;
  const TC* rc = c + static_cast<int64_t>(blockIdx.x) * ldc;
  double mxe = 0.0, se = 0.0, dot = 0.0, na = 0.0, nb = 0.0;
  unsigned long long fin = 0, bad = 0;
  for (int64_t j = threadIdx.x; j < n; j += kThreads) {
    const float bv = ld_val(rb, j), cv = ld_val(rc, j);
    if (!isfinite(cv)) ++bad;
    if (!isfinite(bv) || !isfinite(cv)) continue;
    const double d = fabs(static_cast<double>(bv) - cv);
    mxe = fmax(mxe, d);
    se += d;
    dot += static_cast<double>(bv) * cv;
    na += static_cast<double>(bv) * bv;
    nb += static_cast<double>(cv) * cv;
    ++fin;
  }
  double* out = part + static_cast<int64_t>(blockIdx.x) * 7;
  mxe = block_reduce<TB, double>(mxe, op_maxd, shd);
  if (threadIdx.x == 0) out[0] = mxe;
  se = block_reduce<TB, double>(se, op_addd, shd);
  if (threadIdx.x == 0) out[1] = se;
  dot = block_reduce<TB, double>(dot, op_addd, shd);
  if (threadIdx.x == 0) out[2] = dot;
  na = block_reduce<TB, double>(na, op_addd, shd);
  if (threadIdx.x == 0) out[3] = na;
  nb = block_reduce<TB, double>(nb, op_addd, shd);
  if (threadIdx.x == 0) out[4] = nb;
  fin = block_reduce<TB, unsigned long long>(fin, op_addu, shu);
  if (threadIdx.x == 0) out[5] = static_cast<double>(fin);
  bad = block_reduce<TB, unsigned long long>(bad, op_addu, shu);
  if (threadIdx.x == 0) out[6] = static_cast<double>(bad);
}

// Fold of the LM head's fused row statistics (gemm_tc.cu EPI_ROWSTAT): a CTA owns 32 rows;
// its 8 warps split the slots (warp w: slots w, w + 8, ...) so every load is one 512-byte
// run of 32 consecutive rows (slot-major layout).  Per thread: running max with the first
// column reaching it (slots in column order, strict >) and the denominator
// sum_p s_p * exp(m_p - m) in double, rescaled when m grows; the 8 partials of a row then
// merge through shared memory (max, lowest column on ties, den * exp(m_w - M)).  The NLL
// of the target is formed exactly as row_nll does (0 without a target, NaN for a
// non-finite row).
constexpr int kFoldRows = 32, kFoldWarps = 8;
__global__ void __launch_bounds__(kFoldRows * kFoldWarps) rowstat_combine_kernel(
    const float4* __restrict__ stat, int nslots, int64_t rows, int64_t n, const int32_t* __restrict__ targets,
    const float* __restrict__ tval, double* __restrict__ nll, int32_t* __restrict__ amax) {
  __shared__ float s_mx[kFoldWarps][kFoldRows];
  __shared__ int s_idx[kFoldWarps][kFoldRows];
  __shared__ double s_den[kFoldWarps][kFoldRows];
  __shared__ int s_bad[kFoldWarps][kFoldRows];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kFoldRows + lane;
  const float ninf = __int_as_float(0xff800000);
  float mx = ninf;
  int idx = 0x7fffffff;
  double den = 0.0;
  bool bad = false;
  if (r < rows) {
    for (int p = w; p < nslots; p += kFoldWarps) {
      const float4 q = __ldcs(stat + static_cast<int64_t>(p) * rows + r);
      bad |= q.w != 0.0f;
      if (q.x == ninf) continue;  // an all-masked slot (vocabulary tail)
      if (q.x > mx) {
        den = mx == ninf ? 0.0 : den * exp(static_cast<double>(mx) - static_cast<double>(q.x));
        mx = q.x;
        idx = __float_as_int(q.z);
      }
      den += static_cast<double>(q.y) * exp(static_cast<double>(q.x) - static_cast<double>(mx));
    }
  }
  s_mx[w][lane] = mx;
  s_idx[w][lane] = idx;
  s_den[w][lane] = den;
  s_bad[w][lane] = bad;
  __syncthreads();
  if (w != 0 || r >= rows) return;
  // merge in warp order: slots of warp v precede those of warp v+1 only within a stride,
  // so ties resolve on the column index itself
  float M = ninf;
  int I = 0x7fffffff;
  bool B = false;
#pragma unroll
  for (int v = 0; v < kFoldWarps; ++v) {
    const float m = s_mx[v][lane];
    const int id = s_idx[v][lane];
    B |= s_bad[v][lane] != 0;
    if (m > M || (m == M && m != ninf && id < I)) {
      M = m;
      I = id;
    }
  }
  if (amax != nullptr) amax[r] = I;
  if (nll == nullptr) return;
  const int32_t t = targets != nullptr ? targets[r] : -1;
  if (t < 0 || t >= n) {
    nll[r] = 0.0;
    return;
  }
  if (!isfinite(M) || B) {
    nll[r] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  double D = 0.0;
#pragma unroll
  for (int v = 0; v < kFoldWarps; ++v) {
    const float m = s_mx[v][lane];
    if (m != ninf) D += s_den[v][lane] * exp(static_cast<double>(m) - static_cast<double>(M));
  }
  nll[r] = -((static_cast<double>(tval[r]) - M) - log(D));
}

}  // namespace

void rowstat_combine(const void* stat, int nslots, int64_t rows, int64_t n, const int32_t* targets,
                     const float* tval, double* nll, int32_t* amax, cudaStream_t st) {
  if (rows <= 0) return;
  rowstat_combine_kernel<<<static_cast<unsigned>((rows + kFoldRows - 1) / kFoldRows), kFoldRows * kFoldWarps, 0, st>>>(
      static_cast<const float4*>(stat), nslots, rows, n, targets, tval, nll, amax);
  PRLAB_CUDA(cudaGetLastError());
}

void row_nll(const void* logits, int dtype, int64_t rows, int64_t n, int64_t ld, const int32_t* targets,
             double* nll, int32_t* amax, cudaStream_t st) {
  if (rows <= 0) return;
  if (dtype == 1)
    row_nll_kernel<__half><<<static_cast<unsigned>(rows), kThreads, 0, st>>>(static_cast<const __half*>(logits), n,
                                                                            ld, targets, nll, amax);
  else
    row_nll_kernel<float><<<static_cast<unsigned>(rows), kThreads, 0, st>>>(static_cast<const float*>(logits), n,
                                                                           ld, targets, nll, amax);
  PRLAB_CUDA(cudaGetLastError());
}

void compare_rows(const void* base, int base_dtype, int64_t ldb, const void* cand, int cand_dtype, int64_t ldc,
                  int64_t rows, int64_t n, double* part, cudaStream_t st) {
  if (rows <= 0) return;
  const unsigned g = static_cast<unsigned>(rows);
  if (base_dtype == 0 && cand_dtype == 0)
    compare_rows_kernel<float, float><<<g, kThreads, 0, st>>>(static_cast<const float*>(base), ldb,
                                                             static_cast<const float*>(cand), ldc, n, part);
  else if (base_dtype == 0 && cand_dtype == 1)
    compare_rows_kernel<float, __half><<<g, kThreads, 0, st>>>(static_cast<const float*>(base), ldb,
                                                              static_cast<const __half*>(cand), ldc, n, part);
  else if (base_dtype == 1 && cand_dtype == 0)
    compare_rows_kernel<__half, float><<<g, kThreads, 0, st>>>(static_cast<const __half*>(base), ldb,
                                                              static_cast<const float*>(cand), ldc, n, part);
  else
    compare_rows_kernel<__half, __half><<<g, kThreads, 0, st>>>(static_cast<const __half*>(base), ldb,
                                                               static_cast<const __half*>(cand), ldc, n, part);
  PRLAB_CUDA(cudaGetLastError());
}

}  // namespace prlab_gpu
