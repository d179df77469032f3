// Device-side helpers shared by the sm_100a kernels: binary16 lattice,
// mbarrier / TMA / tcgen05 PTX wrappers.  Written directly against the PTX
// ISA (no CUTLASS/CuTe); descriptor bit layouts follow the tcgen05 "matrix
// descriptor" and "instruction descriptor" formats for kind::f16.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

namespace prlab_gpu {

// ---------------------------------------------------------------------------
// binary16 lattice (reference include/prlab/float16.hpp:33-50).  cvt.rn.f16.f32
// is RNE with overflow (>= 65520) to +/-inf, identical in value to round16 for
// every fp32 input (NaN payloads differ; compare NaNs with isnan).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float r16(float x) { return __half2float(__float2half_rn(x)); }
__device__ __forceinline__ float conform(float x, int f16) { return f16 ? r16(x) : x; }

// 2^x on the SFU (ex2.approx, rel. error ~2^-22): the softmax exponent feeds an fp16
// rounding of p, so the last fp32 bits are immaterial for the hybrid lattice.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// exact-erf GELU, reference src/kernels.cpp:221-235 (same expression order)
__device__ __forceinline__ float gelu_erf(float v) {
  return __fmul_rn(__fmul_rn(0.5f, v), __fadd_rn(1.0f, erff(__fmul_rn(v, 0.70710678118654752440f))));
}

// ---------------------------------------------------------------------------
// Packed pair arithmetic (sm_100: FFMA2 / FMUL2 / FADD2 on .f32x2, HADD2 on f16x2).
// A pair is two fp32 lanes in one 64-bit register; every op rounds each lane RN,
// exactly as the scalar op would.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// (round16(lo), round16(hi)) packed as f16x2 (lo in the low half)
__device__ __forceinline__ uint32_t h2_pack_rn(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// binary16 RNE add of two f16x2 words: equals round16(fp32(a) + fp32(b)) lane-wise for
// every pair of binary16 inputs (24 >= 2*11+2, so the fp32 sum rounded again to
// binary16 is the correctly rounded binary16 sum -- SURVEY App. C.2).
__device__ __forceinline__ uint32_t h2_add_rn(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ void h2_unpack(uint32_t v, float& lo, float& hi) {
  const __half2 h = *reinterpret_cast<const __half2*>(&v);
  lo = __low2float(h);
  hi = __high2float(h);
}

// 2^x for a pair on the FMA pipe (offloads the SFU in the softmax): x clamped to
// [-125, 0] (the callers' exponents are <= 0; below -125 the result is < 2^-125,
// which is 0 after any fp16 rounding and negligible in an fp32 row sum),
// n = rint(x) by the 1.5*2^23 trick, 2^f on [-0.5, 0.5] by a degree-5 minimax
// polynomial (rel. error 3.5e-7, ex2.approx is ~2^-22), exponent added as an integer.
__device__ __forceinline__ uint64_t exp2_pair_poly(float x0, float x1) {
  const uint64_t x = f2_pack(fmaxf(x0, -125.0f), fmaxf(x1, -125.0f));
  const uint64_t M = f2_pack(12582912.0f, 12582912.0f);
  const uint64_t j = f2_add(x, M);
  const uint64_t nM = f2_pack(-12582912.0f, -12582912.0f);
  const uint64_t n = f2_add(j, nM);
  float n0, n1;
  f2_unpack(n, n0, n1);
  const uint64_t f = f2_add(x, f2_pack(-n0, -n1));
  auto C = [](float c) { return f2_pack(c, c); };
  uint64_t p = C(1.339528011e-03f);
  p = f2_fma(p, f, C(9.670763277e-03f));
  p = f2_fma(p, f, C(5.550340563e-02f));
  p = f2_fma(p, f, C(2.402221113e-01f));
  p = f2_fma(p, f, C(6.931471825e-01f));
  p = f2_fma(p, f, C(1.0f));
  float p0, p1, j0, j1;
  f2_unpack(p, p0, p1);
  f2_unpack(j, j0, j1);
  return f2_pack(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(j0) << 23)),
                 __uint_as_float(__float_as_uint(p1) + (__float_as_uint(j1) << 23)));
}

// GELU of two binary16-lattice values in the reference's expression order
// 0.5f * v * (1.0f + erf(v * 0.70710678f)) (src/kernels.cpp:221-235), with erf
// evaluated branch-free on the FMA pipe as sign(u) * (1 - erfc|u|),
// erfc(t) = 2^(-t^2 log2 e + P(t)) for t = min(|u|, 4.5) and P a degree-12 fit of
// log2(erfc(t) e^(t^2)) (abs. error 4e-7 in the exponent).  The 1 + erf sum and the
// products are the reference's fp32 operations, so the result differs from the
// correctly rounded reference formula only where erf's last fp32 bit flips the fp16
// rounding of the output (5 of the 63 488 finite binary16 inputs in a double-precision
// emulation; scripts/gelu_fit.py).  ~14 issue slots per element instead of ~30.
__device__ __forceinline__ void gelu2_fast(float& x0, float& x1) {
  const uint64_t x = f2_pack(x0, x1);
  const uint64_t u = f2_mul(x, f2_pack(0.70710678118654752440f, 0.70710678118654752440f));
  float u0, u1;
  f2_unpack(u, u0, u1);
  const uint64_t t = f2_pack(fminf(fabsf(u0), 4.5f), fminf(fabsf(u1), 4.5f));
  const uint64_t xc = f2_fma(t, f2_pack(2.0f / 4.5f, 2.0f / 4.5f), f2_pack(-1.0f, -1.0f));
  auto C = [](float c) { return f2_pack(c, c); };
  uint64_t p = C(-2.227836521e-04f);
  p = f2_fma(p, xc, C(5.317298928e-04f));
  p = f2_fma(p, xc, C(-2.733187575e-04f));
  p = f2_fma(p, xc, C(-4.225545854e-04f));
  p = f2_fma(p, xc, C(1.940271002e-03f));
  p = f2_fma(p, xc, C(-6.848694291e-03f));
  p = f2_fma(p, xc, C(1.920940541e-02f));
  p = f2_fma(p, xc, C(-4.619692266e-02f));
  p = f2_fma(p, xc, C(1.024701148e-01f));
  p = f2_fma(p, xc, C(-2.187634408e-01f));
  p = f2_fma(p, xc, C(4.757040143e-01f));
  p = f2_fma(p, xc, C(-1.242962837e+00f));
  p = f2_fma(p, xc, C(-2.113490343e+00f));
  const uint64_t e = f2_fma(f2_mul(t, t), C(-1.4426950408889634f), p);
  float e0, e1;
  f2_unpack(e, e0, e1);
  const uint64_t q = f2_pack(ex2_approx(e0), ex2_approx(e1));  // erfc(|u|)
  float a0, a1;
  f2_unpack(f2_fma(q, C(-1.0f), C(1.0f)), a0, a1);  // erf|u| = 1 - erfc|u|
  const uint64_t erf2 = f2_pack(copysignf(a0, u0), copysignf(a1, u1));
  const uint64_t g = f2_mul(f2_mul(C(0.5f), x), f2_add(C(1.0f), erf2));
  f2_unpack(g, x0, x1);
}

// ---------------------------------------------------------------------------
// shared-memory / mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}

// Watchdog: a protocol bug must trap (kernel error) instead of hanging the
// GPU.  ~2^31 cycles (>1 s) of waiting on one phase is never legitimate.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  uint32_t spins = 0;
  while (!mbar_try_wait(addr, parity)) {
    if ((++spins & 1023u) == 0 && clock64() - t0 > (1ll << 31)) {
      printf("prlab_gpu watchdog: mbarrier wait timeout block %d thread %d parity %u\n",
             blockIdx.x, threadIdx.x, parity);
      __trap();
    }
  }
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk.tensor) -- completion counted on an mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// TMA stores (smem -> global, bulk async-group completion, per issuing thread)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
// global[c] += smem (element type from the tensor map; f32 add performed at L2)
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// Hybrid LayerNorm of one row held by a warp (lane owns float4 columns lane + 32 i, n =
// 128 VPT): two-pass fp32 mean / population variance like layernorm_lastdim
// (src/kernels.cpp:170-219), y = gamma ((x - mean) inv) + beta, round16 -> fp16 row.
// Shared by the standalone LN kernel and the GEMM epilogues that fuse it (one summation
// order, so both paths give the same bits).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float ln_warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int VPT>
__device__ __forceinline__ void ln_row_f16(const float4 (&v)[VPT], int lane, const float* __restrict__ gamma,
                                           const float* __restrict__ beta, float eps, __half* __restrict__ out_row) {
  constexpr int n = 128 * VPT;
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  s = ln_warp_sum(s);
  const float mean = __fdiv_rn(s, static_cast<float>(n));
  float vs = 0.0f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const float a = __fsub_rn(v[i].x, mean), b = __fsub_rn(v[i].y, mean);
    const float c = __fsub_rn(v[i].z, mean), d = __fsub_rn(v[i].w, mean);
    vs += (__fmul_rn(a, a) + __fmul_rn(b, b)) + (__fmul_rn(c, c) + __fmul_rn(d, d));
  }
  vs = ln_warp_sum(vs);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(vs, static_cast<float>(n)), eps)));
  const float4* g4 = reinterpret_cast<const float4*>(gamma);
  const float4* b4 = reinterpret_cast<const float4*>(beta);
  uint2* o = reinterpret_cast<uint2*>(out_row);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const float4 g = __ldg(g4 + lane + 32 * i), b = __ldg(b4 + lane + 32 * i);
    const float y0 = __fadd_rn(__fmul_rn(g.x, __fmul_rn(__fsub_rn(v[i].x, mean), inv)), b.x);
    const float y1 = __fadd_rn(__fmul_rn(g.y, __fmul_rn(__fsub_rn(v[i].y, mean), inv)), b.y);
    const float y2 = __fadd_rn(__fmul_rn(g.z, __fmul_rn(__fsub_rn(v[i].z, mean), inv)), b.z);
    const float y3 = __fadd_rn(__fmul_rn(g.w, __fmul_rn(__fsub_rn(v[i].w, mean), inv)), b.w);
    __half2 h01 = __floats2half2_rn(y0, y1), h23 = __floats2half2_rn(y2, y3);
    o[lane + 32 * i] = make_uint2(*reinterpret_cast<uint32_t*>(&h01), *reinterpret_cast<uint32_t*>(&h23));
  }
}

// ---------------------------------------------------------------------------
// tcgen05 (5th-gen tensor cores, TMEM)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16, issued by one thread.
__device__ __forceinline__ void umma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread i gets lane (base+i), columns col..col+31.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"), SWIZZLE_128B:
//   [0,14) start>>4 | [16,30) LBO>>4 | [32,46) SBO>>4 | [46,48) version=1 |
//   [49,52) base offset=0 | [52] lbo mode=0 | [61,64) layout=2 (128B swizzle).
// K-major operand: rows of 128 B (64 fp16 of K), 8-row core groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor, kind::f16: fp16 A/B, fp32 D, M x N, A/B major (0 = K-major, 1 = MN-major).
__host__ __device__ constexpr uint32_t idesc_f16_f32(uint32_t M, uint32_t N, uint32_t a_mn,
                                                     uint32_t b_mn) {
  return (1u << 4) | (0u << 7) | (0u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}

// Programmatic dependent launch: wait for the upstream grid's memory, and let the
// downstream grid start its prologue (barrier init, TMEM alloc, weight prefetch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- CTA-pair (cta_group::2) variants -------------------------------------
// Address of the same shared-memory object in the pair's leader CTA (rank 0):
// cluster shared addresses carry the CTA rank above bit 24.
__device__ __forceinline__ uint32_t to_leader(uint32_t smem_addr) { return smem_addr & 0xFEFFFFFFu; }
// TMA load whose transaction bytes complete on the LEADER's mbarrier.
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(to_leader(smem_u32(bar))), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(to_leader(smem_u32(bar))), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// Pair TMA load multicast to the CTAs in `mask` (cluster-relative ranks): each
// destination receives the box at the same shared offset and the transaction bytes
// complete on the mbarrier of its pair's leader (same offset).
__device__ __forceinline__ void tma_load_2d_pair_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                                    uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(to_leader(smem_u32(bar))), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// Plain (cta_group::1) TMA load multicast to the CTAs in `mask`: each destination CTA
// receives the box at the same shared offset and the bytes complete on ITS mbarrier
// at the same offset.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                                               int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}
// cta_group::1 commit arriving on the same-offset mbarrier of every CTA in `mask`
__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)), "h"(mask)
      : "memory");
}
// arrive on a barrier of another CTA of the cluster (shared::cluster address).
// Default (CTA-scope release) semantics: the data these arrivals announce is either
// tracked by TMA transaction bytes or ordered by tcgen05 fences, so no cluster-scope
// fence (MEMBAR + ERRBAR per arrival) is needed.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish_pair() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// D[tmem of both CTAs] (+)= A[smem of both] * B[smem of both]^T, M = 256, issued by the leader.
__device__ __forceinline__ void umma_f16_ss_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit to the same-offset mbarrier in the CTAs of `mask` (cluster-relative ranks;
// default: both CTAs of a pair in a 2-CTA cluster)
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar, uint16_t mask = 3) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)), "h"(mask)
      : "memory");
}

// Thread-block clusters / distributed shared memory
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
// every thread of every CTA in the cluster must call this
__device__ __forceinline__ void st_dsmem_f4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

}  // namespace prlab_gpu
