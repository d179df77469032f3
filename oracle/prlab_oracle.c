/*
 * prlab CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle.h header).
 *
 * Plain-C restatement of the reference hot path.  Every function cites the
 * reference file:line it restates.  Built with -ffp-contract=off (the
 * reference's own contract, CMakeLists.txt:13) so that every fp32 operation
 * is a separately rounded IEEE op in the same order as the reference: the
 * outputs are bit-identical to the reference's (pinned by
 * tests/test_oracle_vs_ref.py against oracle/_ref/libprlab_ref.so).
 *
 * OpenMP only splits independent output rows / (batch, head) pairs; every
 * individual reduction keeps the reference's sequential ascending order, so
 * the result does not depend on the thread count.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ */
/* binary16 lattice                                                    */
/* ------------------------------------------------------------------ */

static inline uint32_t f2u(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }
static inline float u2f(uint32_t u) { float x; memcpy(&x, &u, 4); return x; }

/* include/prlab/float16.hpp:33-50 -- RNE onto the binary16 lattice on fp32 bits. */
float or_round16(float x) {
  uint32_t u = f2u(x);
  const uint32_t abs_ = u & 0x7FFFFFFFu;
  if (abs_ >= 0x38800000u) {
    if (abs_ >= 0x477FF000u) {
      if (abs_ > 0x7F800000u) return u2f(0x7FC00000u);
      return u2f((u & 0x80000000u) | 0x7F800000u);
    }
    u += 0xFFFu + ((u >> 13) & 1u);
    return u2f(u & 0xFFFFE000u);
  }
  /* subnormal lattice, spacing 2^-24: scale, let fp32 addition round. */
  const float a = u2f(abs_) * 16777216.0f;            /* 2^24 */
  const float r = ((a + 8388608.0f) - 8388608.0f) * 5.9604644775390625e-08f; /* 2^23, 2^-24 */
  return u2f(f2u(r) | (u & 0x80000000u));
}

/* src/float16.cpp:7-37 */
uint16_t or_f16_encode(float x) {
  const uint32_t bits = f2u(x);
  const uint32_t abs_ = bits & 0x7FFFFFFFu;
  const uint16_t sign = (uint16_t)((bits >> 16) & 0x8000u);
  if (abs_ > 0x7F800000u) return 0x7E00u;
  if (abs_ >= 0x477FF000u) return sign | 0x7C00u;
  if (abs_ <= 0x33000000u) return sign;
  uint32_t e = abs_ >> 23, man = abs_ & 0x7FFFFFu, shift;
  if (e > 0x70u) { e -= 0x70u; shift = 13; }
  else { man |= 0x800000u; shift = 0x7Eu - e; e = 0; }
  const uint32_t half = 1u << (shift - 1);
  const uint32_t rem = man & ((1u << shift) - 1u);
  man >>= shift;
  if (rem > half || (rem == half && (man & 1u))) ++man;
  return sign | (uint16_t)((e << 10) + man);
}

/* src/float16.cpp:39-58 */
float or_f16_decode(uint16_t h) {
  const uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1Fu, man = h & 0x3FFu;
  if (e == 0x1Fu) return man ? u2f(0x7FC00000u) : u2f(sign | 0x7F800000u);
  if (e == 0) {
    if (man == 0) return u2f(sign);
    e = 113;
    while (!(man & 0x400u)) { man <<= 1; --e; }
    man &= 0x3FFu;
  } else {
    e += 112;
  }
  return u2f(sign | (e << 23) | (man << 13));
}

/* include/prlab/tensor.hpp:25-27 */
static inline float conform(float v, int d) { return d == OR_F16E ? or_round16(v) : v; }

void or_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------ */
/* policies -- src/policy.cpp:15-17, 49-67                             */
/* ------------------------------------------------------------------ */

int or_resolve_policy(const char* name, or_policy* p) {
  const or_kcfg f32 = {OR_F32, OR_F32, 1}, full = {OR_F16E, OR_F16E, 0},
                wide = {OR_F16E, OR_F32, 1};
  int i;
  if (strcmp(name, "fp32") == 0) {
    for (i = 0; i < OR_NUM_CLASSES; ++i) p->cls[i] = f32;
  } else if (strcmp(name, "full_fp16") == 0) {
    for (i = 0; i < OR_NUM_CLASSES; ++i) p->cls[i] = full;
  } else if (strcmp(name, "hybrid") == 0) {
    for (i = 0; i < OR_NUM_CLASSES; ++i) p->cls[i] = f32;
    p->cls[OR_LINEAR] = wide;
    p->cls[OR_ATTN] = wide;
    p->cls[OR_ACTIVATION] = wide;
  } else {
    return -1;
  }
  return 0;
}

/* KernelConfig::validate, src/kernels.cpp:33-38 */
static int cfg_ok(or_kcfg c) { return !(c.compute == OR_F32 && c.accum == OR_F16E); }

/* on_lattice, src/kernels.cpp:16-22: a rounded copy when narrowing. */
static float* lattice_copy(const float* x, int64_t n, int d) {
  float* y = (float*)malloc((size_t)(n > 0 ? n : 1) * sizeof(float));
  int64_t i;
  if (d == OR_F16E) {
    for (i = 0; i < n; ++i) y[i] = or_round16(x[i]);
  } else {
    memcpy(y, x, (size_t)n * sizeof(float));
  }
  return y;
}

/* ------------------------------------------------------------------ */
/* operators                                                           */
/* ------------------------------------------------------------------ */

/* matmul with B given transposed (bt[n][k]); reduction order identical to
 * src/kernels.cpp:55-81 (ascending k per output). a and bt must already be
 * on the compute lattice. */
static void matmul_bt(const float* a, const float* bt, int64_t m, int64_t k, int64_t n,
                      or_kcfg cfg, float* out) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < m; ++i) {
    const float* arow = a + i * k;
    int64_t j, kk;
    for (j = 0; j < n; ++j) {
      const float* brow = bt + j * k;
      float acc = 0.0f;
      if (cfg.accum == OR_F16E) {
        for (kk = 0; kk < k; ++kk) acc = or_round16(acc + or_round16(arow[kk] * brow[kk]));
        out[i * n + j] = acc;  /* already on the lattice (compute is F16E) */
      } else {
        for (kk = 0; kk < k; ++kk) acc += arow[kk] * brow[kk];
        out[i * n + j] = conform(acc, cfg.compute);
      }
    }
  }
}

static float* transpose(const float* b, int64_t k, int64_t n) {
  float* bt = (float*)malloc((size_t)(k * n > 0 ? k * n : 1) * sizeof(float));
  int64_t r, c;
  for (r = 0; r < k; ++r)
    for (c = 0; c < n; ++c) bt[c * k + r] = b[r * n + c];
  return bt;
}

/* src/kernels.cpp:40-83 */
int or_matmul(const float* a_in, const float* b_in, int64_t m, int64_t k, int64_t n,
              or_kcfg cfg, float* out) {
  if (!cfg_ok(cfg)) return -1;
  float* a = lattice_copy(a_in, m * k, cfg.compute);
  float* b = lattice_copy(b_in, k * n, cfg.compute);
  float* bt = transpose(b, k, n);
  matmul_bt(a, bt, m, k, n, cfg, out);
  free(a); free(b); free(bt);
  return 0;
}

/* src/kernels.cpp:85-125 (q, k already on the compute lattice). */
static void scores_core(const float* q, const float* k, int64_t sq, int64_t sk, int64_t d,
                        int64_t qstride, int64_t kstride, float scale, or_kcfg cfg,
                        float* out, float* capture) {
  int64_t i, j, t;
  for (i = 0; i < sq; ++i) {
    const float* qrow = q + i * qstride;
    for (j = 0; j < sk; ++j) {
      const float* krow = k + j * kstride;
      float value;
      if (cfg.accum == OR_F16E) {
        float acc = 0.0f;
        for (t = 0; t < d; ++t) acc = or_round16(acc + or_round16(qrow[t] * krow[t]));
        value = or_round16(acc * scale);
        if (capture) {
          float ref = 0.0f;
          for (t = 0; t < d; ++t) ref += qrow[t] * krow[t];
          capture[i * sk + j] = ref * scale;
        }
      } else {
        float acc = 0.0f;
        for (t = 0; t < d; ++t) acc += qrow[t] * krow[t];
        const float scaled = acc * scale;
        if (capture) capture[i * sk + j] = scaled;
        value = conform(scaled, cfg.compute);
      }
      out[i * sk + j] = value;
    }
  }
}

int or_attention_scores(const float* q_in, const float* k_in, int64_t sq, int64_t sk,
                        int64_t d, float scale, or_kcfg cfg, float* out, float* capture) {
  if (!cfg_ok(cfg)) return -1;
  float* q = lattice_copy(q_in, sq * d, cfg.compute);
  float* k = lattice_copy(k_in, sk * d, cfg.compute);
  scores_core(q, k, sq, sk, d, d, d, scale, cfg, out, capture);
  free(q); free(k);
  return 0;
}

/* src/kernels.cpp:127-168 -- one row, input already on the compute lattice. */
static void softmax_row(const float* in, float* o, int64_t n, or_kcfg cfg) {
  int64_t i;
  float shift = 0.0f, sum = 0.0f;
  if (cfg.stabilized) {
    shift = -INFINITY;
    for (i = 0; i < n; ++i) shift = in[i] > shift ? in[i] : shift;
  }
  for (i = 0; i < n; ++i) {
    const float e = cfg.stabilized ? expf(in[i] - shift) : expf(in[i]);
    o[i] = conform(e, cfg.compute);
  }
  if (cfg.accum == OR_F16E) {
    for (i = 0; i < n; ++i) sum = or_round16(sum + o[i]);
  } else {
    for (i = 0; i < n; ++i) sum += o[i];
  }
  sum = conform(sum, cfg.compute);
  for (i = 0; i < n; ++i) o[i] = conform(o[i] / sum, cfg.compute);
}

int or_softmax(const float* x_in, int64_t rows, int64_t n, or_kcfg cfg, float* out) {
  int64_t r;
  if (!cfg_ok(cfg) || n <= 0) return -1;
  float* x = lattice_copy(x_in, rows * n, cfg.compute);
  for (r = 0; r < rows; ++r) softmax_row(x + r * n, out + r * n, n, cfg);
  free(x);
  return 0;
}

/* src/kernels.cpp:170-219 -- one row; x, gamma, beta on the compute lattice. */
static void layernorm_row(const float* in, float* o, int64_t n, const float* gamma,
                          const float* beta, float eps, or_kcfg cfg) {
  const int narrow = cfg.accum == OR_F16E;
  int64_t i;
  float sum = 0.0f, var_sum = 0.0f;
  for (i = 0; i < n; ++i) sum = narrow ? or_round16(sum + in[i]) : sum + in[i];
  const float mean = conform(sum / (float)n, cfg.accum);
  for (i = 0; i < n; ++i) {
    const float d = conform(in[i] - mean, cfg.accum);
    const float sq = conform(d * d, cfg.accum);
    var_sum = narrow ? or_round16(var_sum + sq) : var_sum + sq;
  }
  const float var = conform(var_sum / (float)n, cfg.accum);
  const float inv = 1.0f / sqrtf(var + eps);
  for (i = 0; i < n; ++i) o[i] = conform(gamma[i] * ((in[i] - mean) * inv) + beta[i], cfg.compute);
}

int or_layernorm(const float* x_in, int64_t rows, int64_t n, const float* g_in,
                 const float* b_in, float eps, or_kcfg cfg, float* out) {
  int64_t r;
  if (!cfg_ok(cfg) || n <= 0) return -1;
  float* x = lattice_copy(x_in, rows * n, cfg.compute);
  float* g = lattice_copy(g_in, n, cfg.compute);
  float* b = lattice_copy(b_in, n, cfg.compute);
#pragma omp parallel for schedule(static)
  for (r = 0; r < rows; ++r) layernorm_row(x + r * n, out + r * n, n, g, b, eps, cfg);
  free(x); free(g); free(b);
  return 0;
}

/* src/kernels.cpp:221-235 */
int or_gelu(const float* x, int64_t n, or_kcfg cfg, float* out) {
  int64_t i;
  if (!cfg_ok(cfg)) return -1;
  const float kInvSqrt2 = 0.70710678118654752440f;
  for (i = 0; i < n; ++i) {
    const float v = conform(x[i], cfg.compute);
    out[i] = conform(0.5f * v * (1.0f + erff(v * kInvSqrt2)), cfg.compute);
  }
  return 0;
}

/* src/kernels.cpp:237-254 */
int or_add(const float* a, const float* b, int64_t n, or_kcfg cfg, float* out) {
  int64_t i;
  if (!cfg_ok(cfg)) return -1;
  for (i = 0; i < n; ++i)
    out[i] = conform(conform(a[i], cfg.compute) + conform(b[i], cfg.compute), cfg.compute);
  return 0;
}

/* src/kernels.cpp:296-308 */
int or_tanh(const float* x, int64_t n, or_kcfg cfg, float* out) {
  int64_t i;
  if (!cfg_ok(cfg)) return -1;
  for (i = 0; i < n; ++i) out[i] = conform(tanhf(conform(x[i], cfg.compute)), cfg.compute);
  return 0;
}

/* src/kernels.cpp:256-294 */
int or_embed(const float* tok, int64_t vocab, const float* pos, int64_t npos, int64_t h,
             const int32_t* ids, int64_t batch, int64_t seq, or_kcfg cfg, float* out) {
  int64_t r, c;
  if (!cfg_ok(cfg)) return -1;
  if (seq > npos) return -2;
  for (r = 0; r < batch * seq; ++r)
    if (ids[r] < 0 || ids[r] >= vocab) return -2;
  for (r = 0; r < batch * seq; ++r) {
    const float* t = tok + (int64_t)ids[r] * h;
    const float* p = pos + (r % seq) * h;
    for (c = 0; c < h; ++c)
      out[r * h + c] = conform(conform(t[c], cfg.compute) + conform(p[c], cfg.compute), cfg.compute);
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* model                                                               */
/* ------------------------------------------------------------------ */

/* ModelConfig::validate, src/model.cpp:101-117 */
int or_validate_config(const or_model_cfg* c) {
  if (c->num_layers < 0 || c->hidden < 1 || c->heads < 1 || c->ffn < 1 || c->vocab < 1 ||
      c->max_positions < 1)
    return -1;
  if (c->hidden % c->heads != 0) return -1;
  if (c->ffn < c->hidden) return -1;
  return 0;
}

/* src/model.cpp:267-281 */
uint64_t or_param_count(const or_model_cfg* c) {
  const uint64_t h = (uint64_t)c->hidden, f = (uint64_t)c->ffn;
  const uint64_t emb = (uint64_t)c->vocab * h + (uint64_t)c->max_positions * h;
  const uint64_t per_layer = 4 * h + 4 * (h * h + h) + (h * f + f) + (f * h + h);
  uint64_t total = emb + (uint64_t)c->num_layers * per_layer + 2 * h;
  if (c->archetype == 0) total += (h * h + h) + (2 * h + 2);
  return total;
}

int64_t or_num_param_tensors(const or_model_cfg* c) {
  return 2 + 16 * c->num_layers + 2 + (c->archetype == 0 ? 4 : 0);
}

/* mt19937_64 (the std::mt19937_64 engine used at src/model.cpp:23,292). */
typedef struct { uint64_t mt[312]; int mti; } mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  int i;
  s->mt[0] = seed;
  for (i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  uint64_t x;
  int i;
  if (s->mti >= 312) {
    for (i = 0; i < 312 - 156; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    for (; i < 311; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    }
    x = (s->mt[311] & UM) | (s->mt[0] & LM);
    s->mt[311] = s->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
    s->mti = 0;
  }
  x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* NormalSampler, src/model.cpp:22-44 (fixed Box-Muller). */
typedef struct { mt64 rng; double spare; int have_spare; } normal_sampler;

static float ns_next(normal_sampler* s, float stddev) {
  if (s->have_spare) {
    s->have_spare = 0;
    return (float)(s->spare * (double)stddev);
  }
  const double u1 = ((double)(mt64_next(&s->rng) >> 11) + 0.5) * 0x1.0p-53;
  const double u2 = (double)(mt64_next(&s->rng) >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double a = 2.0 * 3.14159265358979323846 * u2;
  s->spare = r * sin(a);
  s->have_spare = 1;
  return (float)(r * cos(a) * (double)stddev);
}

/* Canonical parameter walk (Model::for_each_param, src/model.cpp:178-209)
 * yields (numel, kind) where kind: 0 matrix (N(0,0.02)), 1 gamma (ones), 2 zero. */
typedef struct { int64_t numel; int kind; } ptensor;

static int64_t param_walk(const or_model_cfg* c, ptensor* out) {
  const int64_t h = c->hidden, f = c->ffn;
  int64_t n = 0, l;
#define P(num, kind_) do { if (out) { out[n].numel = (num); out[n].kind = (kind_); } ++n; } while (0)
  P(c->vocab * h, 0);
  P(c->max_positions * h, 0);
  for (l = 0; l < c->num_layers; ++l) {
    P(h, 1); P(h, 2);            /* ln1 gamma, beta */
    P(h * h, 0); P(h, 2);        /* wq bq */
    P(h * h, 0); P(h, 2);        /* wk bk */
    P(h * h, 0); P(h, 2);        /* wv bv */
    P(h * h, 0); P(h, 2);        /* wo bo */
    P(h, 1); P(h, 2);            /* ln2 */
    P(h * f, 0); P(f, 2);        /* w1 b1 */
    P(f * h, 0); P(h, 2);        /* w2 b2 */
  }
  P(h, 1); P(h, 2);              /* final ln */
  if (c->archetype == 0) {
    P(h * h, 0); P(h, 2);        /* pooler */
    P(h * 2, 0); P(2, 2);        /* classifier */
  }
#undef P
  return n;
}

/* build_model, src/model.cpp:217-265 */
int or_build_model(const or_model_cfg* c, float* params) {
  if (or_validate_config(c)) return -1;
  const int64_t nt = param_walk(c, NULL);
  ptensor* ts = (ptensor*)malloc((size_t)nt * sizeof(ptensor));
  param_walk(c, ts);
  normal_sampler s;
  int64_t t, i;
  mt64_seed(&s.rng, c->seed);
  s.have_spare = 0;
  s.spare = 0.0;
  float* p = params;
  for (t = 0; t < nt; ++t) {
    for (i = 0; i < ts[t].numel; ++i)
      p[i] = ts[t].kind == 0 ? ns_next(&s, 0.02f) : (ts[t].kind == 1 ? 1.0f : 0.0f);
    p += ts[t].numel;
  }
  free(ts);
  return 0;
}

/* random_tokens, src/model.cpp:283-296 */
void or_random_tokens(int64_t vocab, int64_t batch, int64_t seq, uint64_t seed, int32_t* ids) {
  mt64 r;
  int64_t i;
  mt64_seed(&r, seed);
  for (i = 0; i < batch * seq; ++i) ids[i] = (int32_t)(mt64_next(&r) % (uint64_t)vocab);
}

/* linear_bias, src/model.cpp:66-78: x already on the compute lattice,
 * wt = W^T ([out,in]) on the compute lattice. */
static void linear_bias(const float* x, const float* wt, const float* b, int64_t m, int64_t k,
                        int64_t n, or_kcfg cfg, float* out) {
  int64_t r, c;
  matmul_bt(x, wt, m, k, n, cfg, out);
  for (r = 0; r < m; ++r)
    for (c = 0; c < n; ++c)
      out[r * n + c] = conform(out[r * n + c] + conform(b[c], cfg.compute), cfg.compute);
}

static void lattice_inplace(float* x, int64_t n, int d) {
  int64_t i;
  if (d == OR_F16E)
    for (i = 0; i < n; ++i) x[i] = or_round16(x[i]);
}

/* forward_hidden + forward, src/model.cpp:350-482.  hidden_out (optional): the final
 * LayerNorm output [B*S, h] (forward_hidden's result) -- then no head is computed. */
static int forward_impl(const or_model_cfg* c, const float* params, const int32_t* ids, int64_t B,
                        int64_t S, const or_policy* pol, float* logits, uint64_t* calls,
                        float* scores_tap, float* hidden_out) {
  int i;
  if (or_validate_config(c)) return -1;
  for (i = 0; i < OR_NUM_CLASSES; ++i)
    if (!cfg_ok(pol->cls[i])) return -1;
  if (B < 1 || S < 1) return -1;
  if (S > c->max_positions) return -1;
  const int64_t h = c->hidden, f = c->ffn, H = c->heads, hd = h / H, V = c->vocab;
  const int64_t M = B * S;
  const float scale = 1.0f / sqrtf((float)hd);
  const int causal = c->archetype == 1;
  const or_kcfg lin = pol->cls[OR_LINEAR], att = pol->cls[OR_ATTN], sm = pol->cls[OR_SOFTMAX],
                ln = pol->cls[OR_LAYERNORM], act = pol->cls[OR_ACTIVATION],
                emb = pol->cls[OR_EMBEDDING], res = pol->cls[OR_RESIDUAL];
  uint64_t local_calls[OR_NUM_CLASSES * 2];
  uint64_t* cc = calls ? calls : local_calls;
  memset(cc, 0, sizeof(local_calls));
#define COUNT(cls_, cfg_) (cc[(cls_) * 2 + (cfg_).compute] += 1)

  /* parameter views in canonical order */
  const float* tok = params;
  const float* pos = tok + V * h;
  const float* lp = pos + c->max_positions * h;
  const int64_t per_layer = 4 * h + 4 * (h * h + h) + (h * f + f) + (f * h + h);
  const float* fin = lp + c->num_layers * per_layer;

  float* x = (float*)malloc((size_t)(M * h) * sizeof(float));
  COUNT(OR_EMBEDDING, emb);
  {
    int rc = or_embed(tok, V, pos, c->max_positions, h, ids, B, S, emb, x);
    if (rc) { free(x); return rc; }
  }

  float* xn = (float*)malloc((size_t)(M * h) * sizeof(float));
  float* q = (float*)malloc((size_t)(M * h) * sizeof(float));
  float* k = (float*)malloc((size_t)(M * h) * sizeof(float));
  float* v = (float*)malloc((size_t)(M * h) * sizeof(float));
  float* ctx = (float*)malloc((size_t)(M * h) * sizeof(float));
  float* br = (float*)malloc((size_t)(M * h) * sizeof(float));
  float* ff = (float*)malloc((size_t)(M * f) * sizeof(float));
  float* wt = (float*)malloc((size_t)(h * f) * sizeof(float));
  int64_t l;

  for (l = 0; l < c->num_layers; ++l) {
    const float* P = lp + l * per_layer;
    const float *ln1g = P, *ln1b = P + h;
    const float *wq = P + 2 * h, *bq = wq + h * h;
    const float *wk = bq + h, *bk = wk + h * h;
    const float *wv = bk + h, *bv = wv + h * h;
    const float *wo = bv + h, *bo = wo + h * h;
    const float *ln2g = bo + h, *ln2b = ln2g + h;
    const float *w1 = ln2b + h, *b1 = w1 + h * f;
    const float *w2 = b1 + f, *b2 = w2 + f * h;
    int64_t r;

    /* LN1 (model.cpp:383-385) */
    COUNT(OR_LAYERNORM, ln);
    or_layernorm(x, M, h, ln1g, ln1b, 1e-5f, ln, xn);
    /* Q, K, V projections (model.cpp:386-391); x rounded onto Linear lattice. */
    lattice_inplace(xn, M * h, lin.compute);
#define LIN(W_, B_, IN_, K_, N_, OUT_)                                 \
    do {                                                               \
      int64_t rr_, cc_;                                                \
      for (rr_ = 0; rr_ < (K_); ++rr_)                                 \
        for (cc_ = 0; cc_ < (N_); ++cc_)                               \
          wt[cc_ * (K_) + rr_] = conform((W_)[rr_ * (N_) + cc_], lin.compute); \
      COUNT(OR_LINEAR, lin);                                           \
      linear_bias((IN_), wt, (B_), M, (K_), (N_), lin, (OUT_));        \
    } while (0)
    LIN(wq, bq, xn, h, h, q);
    LIN(wk, bk, xn, h, h, k);
    LIN(wv, bv, xn, h, h, v);

    /* attention (model.cpp:393-427) */
    {
      float* qa = lattice_copy(q, M * h, att.compute);
      float* ka = lattice_copy(k, M * h, att.compute);
      float* va = lattice_copy(v, M * h, att.compute);
      int64_t bh;
      for (bh = 0; bh < B * H; ++bh) {
        COUNT(OR_ATTN, att);
        COUNT(OR_SOFTMAX, sm);
        COUNT(OR_ATTN, att);
      }
#pragma omp parallel for schedule(dynamic)
      for (bh = 0; bh < B * H; ++bh) {
        const int64_t b = bh / H, head = bh % H;
        float* sc = (float*)malloc((size_t)(S * S) * sizeof(float));
        float* pr = (float*)malloc((size_t)(S * S) * sizeof(float));
        float* tap = scores_tap ? scores_tap + ((l * B + b) * H + head) * S * S : NULL;
        int64_t ii, jj, t;
        scores_core(qa + (b * S) * h + head * hd, ka + (b * S) * h + head * hd, S, S, hd, h, h,
                    scale, att, sc, tap);
        if (causal)
          for (ii = 0; ii < S; ++ii)
            for (jj = ii + 1; jj < S; ++jj) sc[ii * S + jj] = -INFINITY;
        /* softmax (model.cpp:416): input onto the softmax lattice */
        for (ii = 0; ii < S * S; ++ii) sc[ii] = conform(sc[ii], sm.compute);
        for (ii = 0; ii < S; ++ii) softmax_row(sc + ii * S, pr + ii * S, S, sm);
        /* PV (model.cpp:418-420): probs and V on the attention lattice */
        for (ii = 0; ii < S * S; ++ii) pr[ii] = conform(pr[ii], att.compute);
        for (ii = 0; ii < S; ++ii) {
          for (t = 0; t < hd; ++t) {
            float acc = 0.0f;
            if (att.accum == OR_F16E) {
              for (jj = 0; jj < S; ++jj)
                acc = or_round16(acc + or_round16(pr[ii * S + jj] * va[(b * S + jj) * h + head * hd + t]));
            } else {
              for (jj = 0; jj < S; ++jj) acc += pr[ii * S + jj] * va[(b * S + jj) * h + head * hd + t];
              acc = conform(acc, att.compute);
            }
            ctx[(b * S + ii) * h + head * hd + t] = acc;
          }
        }
        free(sc); free(pr);
      }
      free(qa); free(ka); free(va);
    }

    /* Wo + residual (model.cpp:429-431) */
    lattice_inplace(ctx, M * h, lin.compute);
    LIN(wo, bo, ctx, h, h, br);
    COUNT(OR_RESIDUAL, res);
    for (r = 0; r < M * h; ++r)
      x[r] = conform(conform(x[r], res.compute) + conform(br[r], res.compute), res.compute);

    /* LN2, W1, GELU, W2, residual (model.cpp:433-442) */
    COUNT(OR_LAYERNORM, ln);
    or_layernorm(x, M, h, ln2g, ln2b, 1e-5f, ln, xn);
    lattice_inplace(xn, M * h, lin.compute);
    LIN(w1, b1, xn, h, f, ff);
    COUNT(OR_ACTIVATION, act);
    or_gelu(ff, M * f, act, ff);
    lattice_inplace(ff, M * f, lin.compute);
    LIN(w2, b2, ff, f, h, br);
    COUNT(OR_RESIDUAL, res);
    for (r = 0; r < M * h; ++r)
      x[r] = conform(conform(x[r], res.compute) + conform(br[r], res.compute), res.compute);
#undef LIN
  }

  if (hidden_out) {
    /* forward_hidden (model.cpp:445-451): zero layers -> the embeddings, else final LN */
    if (c->num_layers == 0) {
      memcpy(hidden_out, x, (size_t)(M * h) * sizeof(float));
    } else {
      COUNT(OR_LAYERNORM, ln);
      or_layernorm(x, M, h, fin, fin + h, 1e-5f, ln, hidden_out);
    }
  } else if (c->num_layers == 0) {
    memcpy(logits, x, (size_t)(M * h) * sizeof(float));
  } else {
    /* final LN (model.cpp:449-451) and tied head (model.cpp:469-480):
     * logits = matmul(hidden, E^T) -- E rows are exactly the rows of E^T's transpose. */
    COUNT(OR_LAYERNORM, ln);
    or_layernorm(x, M, h, fin, fin + h, 1e-5f, ln, xn);
    lattice_inplace(xn, M * h, lin.compute);
    float* et = lattice_copy(tok, V * h, lin.compute);
    COUNT(OR_LINEAR, lin);
    matmul_bt(xn, et, M, h, V, lin, logits);
    free(et);
  }
#undef COUNT
  free(x); free(xn); free(q); free(k); free(v); free(ctx); free(br); free(ff); free(wt);
  return 0;
}

int or_forward(const or_model_cfg* c, const float* params, const int32_t* ids, int64_t B,
               int64_t S, const or_policy* pol, float* logits, uint64_t* calls,
               float* scores_tap) {
  return forward_impl(c, params, ids, B, S, pol, logits, calls, scores_tap, NULL);
}

/* classifier_probs, src/model.cpp:484-526: mean-pool (Linear accumulation contract),
 * tanh pooler, 2-way head, softmax; out[b] = P(class 1). */
int or_classifier_probs(const or_model_cfg* c, const float* params, const int32_t* ids, int64_t B,
                        int64_t S, const or_policy* pol, float* out) {
  if (c->archetype != 0) return -1; /* encoder_only only (model.cpp:486-488) */
  if (or_validate_config(c)) return -1;
  const int64_t h = c->hidden, f = c->ffn, V = c->vocab;
  const or_kcfg lin = pol->cls[OR_LINEAR], act = pol->cls[OR_ACTIVATION], sm = pol->cls[OR_SOFTMAX];
  float* hidden = (float*)malloc((size_t)(B * S * h) * sizeof(float));
  int rc = forward_impl(c, params, ids, B, S, pol, NULL, NULL, NULL, hidden);
  if (rc) { free(hidden); return rc; }
  const int64_t per_layer = 4 * h + 4 * (h * h + h) + (h * f + f) + (f * h + h);
  const float* fin = params + V * h + c->max_positions * h + c->num_layers * per_layer;
  const float *pw = fin + 2 * h, *pb = pw + h * h, *cw = pb + h, *cb = cw + h * 2;
  float* pooled = (float*)malloc((size_t)(B * h) * sizeof(float));
  float* pre = (float*)malloc((size_t)(B * h) * sizeof(float));
  float* wt = (float*)malloc((size_t)(h * h) * sizeof(float));
  float logits2[2], probs2[2];
  int64_t b, cc, t, r;
  const int narrow = lin.accum == OR_F16E;
  for (b = 0; b < B; ++b)
    for (cc = 0; cc < h; ++cc) {
      float acc = 0.0f;
      for (t = 0; t < S; ++t) {
        const float xv = conform(hidden[(b * S + t) * h + cc], lin.compute);
        acc = narrow ? or_round16(acc + xv) : acc + xv;
      }
      pooled[b * h + cc] = conform(acc / (float)S, lin.compute);
    }
  for (r = 0; r < h; ++r)
    for (cc = 0; cc < h; ++cc) wt[cc * h + r] = conform(pw[r * h + cc], lin.compute);
  linear_bias(pooled, wt, pb, B, h, h, lin, pre);
  or_tanh(pre, B * h, act, pre);
  lattice_inplace(pre, B * h, lin.compute);
  for (r = 0; r < h; ++r)
    for (cc = 0; cc < 2; ++cc) wt[cc * h + r] = conform(cw[r * 2 + cc], lin.compute);
  for (b = 0; b < B; ++b) {
    linear_bias(pre + b * h, wt, cb, 1, h, 2, lin, logits2);
    or_softmax(logits2, 1, 2, sm, probs2);
    out[b] = probs2[1];
  }
  free(hidden); free(pooled); free(pre); free(wt);
  return 0;
}
