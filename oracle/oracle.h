/*
 * prlab CPU oracle -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference hot path (prlab::forward and the
 * operators under it) used as the parity checker for the CUDA product path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it, and only as the checker / the CPU baseline -- never as the thing
 * measured or shipped.  The product (paper_2603_28708_b200) never links it.
 *
 * Parity of this restatement is pinned two ways:
 *   1. the reference's own known-answer tests (test_float16.cpp,
 *      test_kernels.cpp, test_model.cpp, test_policy.cpp) restated in
 *      tests/test_oracle_kats.py;
 *   2. bitwise comparison against the reference itself, compiled from
 *      /root/reference/proj/src into oracle/_ref/libprlab_ref.so by
 *      oracle/Makefile (tests/test_oracle_vs_ref.py, tests/golden/).
 */
#ifndef PRLAB_ORACLE_H
#define PRLAB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Lattice tags: reference Dtype (include/prlab/tensor.hpp:17). */
enum { OR_F32 = 0, OR_F16E = 1 };

/* Reference KernelConfig (include/prlab/kernels.hpp:16-22). */
typedef struct {
  int compute; /* OR_F32 / OR_F16E */
  int accum;   /* OR_F32 / OR_F16E */
  int stabilized;
} or_kcfg;

/* Op classes in reference order (include/prlab/policy.hpp:19-27). */
enum {
  OR_LINEAR = 0, OR_ATTN = 1, OR_SOFTMAX = 2, OR_LAYERNORM = 3,
  OR_ACTIVATION = 4, OR_EMBEDDING = 5, OR_RESIDUAL = 6, OR_NUM_CLASSES = 7
};

typedef struct {
  or_kcfg cls[OR_NUM_CLASSES];
} or_policy;

/* Reference ModelConfig (include/prlab/model.hpp:21-52). archetype: 0 encoder, 1 decoder. */
typedef struct {
  int archetype;
  int64_t num_layers, hidden, heads, ffn, vocab, max_positions;
  uint64_t seed;
} or_model_cfg;

/* --- binary16 lattice (include/prlab/float16.hpp:33-50, src/float16.cpp:7-58) --- */
float or_round16(float x);
uint16_t or_f16_encode(float x);
float or_f16_decode(uint16_t h);

/* --- policies (src/policy.cpp:49-67): name in {"fp32","full_fp16","hybrid"}; 0 ok, -1 unknown --- */
int or_resolve_policy(const char* name, or_policy* out);

/* --- operators (src/kernels.cpp). Return 0, or -1 (invalid_argument) / -2 (out_of_range). --- */
int or_matmul(const float* a, const float* b, int64_t m, int64_t k, int64_t n,
              or_kcfg cfg, float* out);
int or_attention_scores(const float* q, const float* k, int64_t sq, int64_t sk, int64_t d,
                        float scale, or_kcfg cfg, float* out, float* capture_f32);
int or_softmax(const float* x, int64_t rows, int64_t n, or_kcfg cfg, float* out);
int or_layernorm(const float* x, int64_t rows, int64_t n, const float* gamma,
                 const float* beta, float eps, or_kcfg cfg, float* out);
int or_gelu(const float* x, int64_t n, or_kcfg cfg, float* out);
int or_add(const float* a, const float* b, int64_t n, or_kcfg cfg, float* out);
int or_tanh(const float* x, int64_t n, or_kcfg cfg, float* out);
int or_embed(const float* tok, int64_t vocab, const float* pos, int64_t npos, int64_t h,
             const int32_t* ids, int64_t batch, int64_t seq, or_kcfg cfg, float* out);

/* --- model (src/model.cpp) --- */
int or_validate_config(const or_model_cfg* c);
uint64_t or_param_count(const or_model_cfg* c);
/* Number of parameter tensors in canonical (for_each_param) order. */
int64_t or_num_param_tensors(const or_model_cfg* c);
/* Fill `params` (param_count floats, canonical order) exactly as build_model. */
int or_build_model(const or_model_cfg* c, float* params);
void or_random_tokens(int64_t vocab, int64_t batch, int64_t seq, uint64_t seed, int32_t* ids);
/* Full forward. logits: [B,S,V] (or [B,S,h] for a zero-layer model).
 * kernel_calls (optional): [7][2] counts like ForwardTrace::kernel_calls.
 * scores_tap (optional): [L,B,H,S,S] fp32 pre-mask scores (retain_scores). */
int or_forward(const or_model_cfg* c, const float* params, const int32_t* ids, int64_t batch,
               int64_t seq, const or_policy* policy, float* logits, uint64_t* kernel_calls,
               float* scores_tap);

/* classifier_probs (src/model.cpp:484-526): out[b] = positive-class probability.
 * encoder_only models only (-1 otherwise). */
int or_classifier_probs(const or_model_cfg* c, const float* params, const int32_t* ids, int64_t batch,
                        int64_t seq, const or_policy* policy, float* out);

/* OpenMP thread count used by the oracle loops (results are independent of it). */
void or_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
