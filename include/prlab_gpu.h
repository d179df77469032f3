/*
 * prlab_gpu.h -- C-ABI drop-in boundary of the B200-native prlab forward.
 *
 * The reference (`prlab`, C++20) has no FFI layer: its operator API is the set
 * of value-semantic free functions in include/prlab/kernels.hpp:30-70 plus
 * forward()/build_model()/resolve_policy() (include/prlab/model.hpp:88-140,
 * include/prlab/policy.hpp:66).  Each entry point below replaces one of those
 * (cited per function).  Plain pointers and sizes only -- no torch or C++ types.
 * include/prlab_gpu.hpp wraps this ABI back into the reference's C++ signatures
 * (same names, same exception types and messages).
 *
 * Threading / streams: a model may be used from several host threads (calls on one model
 * are serialised by its mutex) and from several CUDA streams: every call orders its work
 * after the previous call's work on the same model (event wait when the stream differs),
 * because all calls share the model's workspace.  Calls on distinct models run
 * concurrently.  A stream that is being captured by the CALLER is not ordered (the
 * caller's graph defines the order).  prlab_gpu_forward (hybrid, logits widened on the
 * host, logits <= 512 MB) holds the model's mutex only while it enqueues its compute into
 * one of two model-owned logits slots; its copy-out then runs on the slot's own stream with
 * the mutex released, so a concurrent caller's compute overlaps it (at most two calls in
 * flight; each call returns exactly its own logits).
 *
 * Errors: every function returns PRLAB_OK (0) or a status; the thread-local
 * message is available from prlab_gpu_last_error().  The status maps onto the
 * reference's exception types: PRLAB_EINVAL -> std::invalid_argument,
 * PRLAB_ERANGE -> std::out_of_range, PRLAB_ERUNTIME / PRLAB_ECUDA ->
 * std::runtime_error.  There is no CPU fallback anywhere behind this ABI: a
 * missing/unsupported device is PRLAB_ECUDA.
 */
#ifndef PRLAB_GPU_H
#define PRLAB_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRLAB_GPU_ABI_VERSION 1

enum prlab_status {
  PRLAB_OK = 0,
  PRLAB_EINVAL = 1,   /* std::invalid_argument */
  PRLAB_ERANGE = 2,   /* std::out_of_range     */
  PRLAB_ERUNTIME = 3, /* std::runtime_error    */
  PRLAB_ECUDA = 4     /* CUDA error -> std::runtime_error */
};

/* Lattices: reference Dtype (include/prlab/tensor.hpp:17). */
enum prlab_dtype { PRLAB_F32 = 0, PRLAB_F16E = 1 };

/* Reference KernelConfig (include/prlab/kernels.hpp:16-22). */
typedef struct {
  int32_t compute;    /* prlab_dtype */
  int32_t accum;      /* prlab_dtype */
  int32_t stabilized; /* softmax only */
} prlab_kcfg;

/* Op classes in the reference order (include/prlab/policy.hpp:19-27). */
enum prlab_op_class {
  PRLAB_LINEAR = 0,
  PRLAB_ATTENTION_SCORE_MATMUL = 1,
  PRLAB_SOFTMAX = 2,
  PRLAB_LAYERNORM = 3,
  PRLAB_ACTIVATION = 4,
  PRLAB_EMBEDDING = 5,
  PRLAB_RESIDUAL = 6,
  PRLAB_NUM_OP_CLASSES = 7
};

/* Reference PrecisionPolicy assignment (include/prlab/policy.hpp:43-56). */
typedef struct {
  prlab_kcfg cls[PRLAB_NUM_OP_CLASSES];
} prlab_policy;

/* Reference ModelConfig (include/prlab/model.hpp:21-52); archetype 0 = encoder_only, 1 = decoder_only. */
typedef struct {
  int32_t archetype;
  int64_t num_layers, hidden, heads, ffn, vocab, max_positions;
  uint64_t seed;
} prlab_model_desc;

/* Reference ForwardTrace instrumentation (include/prlab/model.hpp:113-125):
 * seconds per op class (CUDA-event time, instrumented mode only) and kernel
 * invocation counts per (class, compute dtype). */
typedef struct {
  double seconds[PRLAB_NUM_OP_CLASSES];
  uint64_t kernel_calls[PRLAB_NUM_OP_CLASSES][2];
} prlab_trace;

typedef struct prlab_gpu_model prlab_gpu_model;

/* Output storage of device-resident logits. */
enum prlab_out_dtype { PRLAB_OUT_F32 = 0, PRLAB_OUT_F16 = 1 };

const char* prlab_gpu_last_error(void);
int prlab_gpu_abi_version(void);

/* ---- policy: resolve_policy (src/policy.cpp:49-67) ---- */
int prlab_gpu_resolve_policy(const char* name, prlab_policy* out);
/* PrecisionPolicy::validate / KernelConfig::validate (src/policy.cpp:27-47, src/kernels.cpp:33-38) */
int prlab_gpu_validate_policy(const prlab_policy* p);

/* ---- model: build_model output -> device arena (replaces the per-call
 * on_lattice copies of src/kernels.cpp:16-22 with one preplanned upload).
 * params: host fp32 tensors in the canonical Model::for_each_param order
 * (src/model.cpp:178-209), n_params tensors. */
int prlab_gpu_model_create(const prlab_model_desc* desc, const float* const* params,
                           int64_t n_params, int device, prlab_gpu_model** out);
/* Same, with the canonical tensors concatenated into one flat buffer. */
int prlab_gpu_model_create_flat(const prlab_model_desc* desc, const float* flat, int device,
                                prlab_gpu_model** out);
void prlab_gpu_model_destroy(prlab_gpu_model* m);
/* load_checkpoint (src/checkpoint.cpp:133-162): a PRLABCKP v1 file (config JSON + tensor
 * records in canonical order, f32 or f16 payloads) straight into the device arena; the
 * file's config is returned in *desc (may be NULL).  Same checks and messages as the
 * reference (PRLAB_ERUNTIME for format errors). */
int prlab_gpu_model_load_checkpoint(const char* path, int device, prlab_model_desc* desc,
                                    prlab_gpu_model** out);
/* Bytes held on the device: resident weights (per precision copy) and the
 * activation workspace currently planned. */
int prlab_gpu_model_memory(const prlab_gpu_model* m, uint64_t* weight_bytes,
                           uint64_t* workspace_bytes);

/* Device bytes by purpose (the memory planner's accounting):
 * weights_fast  = the hybrid arena (fp16 K-major linears + tied head, fp32 tables, LN, biases);
 * weights_fp32  = fp32 copies materialised only when a non-hybrid policy ran (+ classifier head);
 * workspace     = the liveness-planned activation arena (max over the planned (B, S) keys);
 * logits        = library-side [B*S, V] logits buffers, allocated only when a call needs the
 *                 logits inside the library (host forward, unfused NLL);
 * scratch       = split-K scratch, persistent-kernel partials, fused-head partials, error word. */
typedef struct {
  uint64_t weights_fast, weights_fp32, workspace, logits, scratch, total;
} prlab_memory_report;
int prlab_gpu_model_memory_ex(prlab_gpu_model* m, prlab_memory_report* out);

/* ---- host fixture generators, same streams as the reference ----
 * build_model (src/model.cpp:217-265): N(0,0.02) fixed Box-Muller over
 * mt19937_64(seed) in canonical order, biases 0, gammas 1.  out: param_count floats. */
int prlab_gpu_build_model(const prlab_model_desc* desc, float* out, int64_t out_len);
uint64_t prlab_gpu_param_count(const prlab_model_desc* desc);   /* src/model.cpp:267-281 */
/* random_tokens (src/model.cpp:283-296): ids[i] = mt19937_64(seed)() % vocab. */
int prlab_gpu_random_tokens(int64_t vocab, int64_t batch, int64_t seq, uint64_t seed, int32_t* ids);
/* Greedy argmax over device logits rows (lowest index wins ties): d_logits [rows, ld]
 * in out_dtype, d_tokens int32 [rows].  Asynchronous on stream. */
int prlab_gpu_argmax_device(const void* d_logits, int32_t dtype, int64_t rows, int64_t n, int64_t ld,
                            int32_t* d_tokens, void* stream);

/* ---- device-side logits reductions (src/fidelity.cpp) ----
 * Per row of device logits [rows, ld] (out_dtype): d_nll (double, may be NULL) =
 * -log_softmax(row)[d_targets[row]] evaluated like window_nll_sum (fidelity.cpp:213-240:
 * max-stabilised, double accumulation; NaN when the row holds NaN/+inf; 0 when the
 * target is < 0), d_argmax (may be NULL) = first index of the row maximum.  Async. */
int prlab_gpu_row_nll_device(const void* d_logits, int32_t dtype, int64_t rows, int64_t n, int64_t ld,
                              const int32_t* d_targets, double* d_nll, int32_t* d_argmax, void* stream);

/* compare_logits (src/fidelity.cpp:11-37) of two device logit tensors; synchronous. */
typedef struct {
  double max_abs_error, mean_abs_error, cosine;
  int32_t has_cosine; /* std::optional<double> cosine engaged */
  uint64_t finite_pairs, candidate_nonfinite;
  int32_t nan_affected;
} prlab_logit_comparison;
int prlab_gpu_compare_logits_device(const void* d_base, int32_t base_dtype, int64_t ld_base, const void* d_cand,
                                    int32_t cand_dtype, int64_t ld_cand, int64_t rows, int64_t n, void* stream,
                                    prlab_logit_comparison* out);

/* perplexity (src/fidelity.cpp:248-279): sliding windows of context_len over a host
 * token stream, forwards batched on the device, next-token NLL reduced on the device
 * (only one double per row crosses PCIe).  Same validation and messages. */
int prlab_gpu_perplexity(prlab_gpu_model* m, const int32_t* tokens, int64_t n_tokens, int64_t context_len,
                         const prlab_policy* policy, double* ppl);

/* ---- forward (src/model.cpp:456-482) ----
 * Drop-in form: host token ids [B*S], host fp32 logits [B,S,V] (or [B,S,h]
 * for a zero-layer model), synchronous.  trace may be NULL. */
int prlab_gpu_forward(prlab_gpu_model* m, const int32_t* ids, int64_t batch, int64_t seq,
                      const prlab_policy* policy, float* logits, prlab_trace* trace);

/* forward with the reference's optional outputs (src/model.cpp:456-482):
 * flags PRLAB_FWD_RETAIN_SCORES -> scores (host fp32 [L][B][H][S][S]) receives every
 *   layer's fp32 pre-mask scaled scores (ForwardTrace::layer_scores, kernels.cpp:108-118);
 * flags PRLAB_FWD_TIMED -> trace->seconds holds CUDA-event time per op class (the
 *   reference's timed() wrappers, model.cpp:55-62; fused kernels count for the class
 *   that produces their output, the fused attention for AttentionScoreMatmul).
 * Without flags this is prlab_gpu_forward. */
enum prlab_fwd_flags { PRLAB_FWD_RETAIN_SCORES = 1, PRLAB_FWD_TIMED = 2 };
int prlab_gpu_forward_ex(prlab_gpu_model* m, const int32_t* ids, int64_t batch, int64_t seq,
                         const prlab_policy* policy, int32_t flags, float* logits, prlab_trace* trace,
                         float* scores);

/* classifier_probs (src/model.cpp:484-526): mean-pooled final hidden states, tanh
 * pooler, 2-way head, softmax; probs[b] = positive-class probability.  encoder_only
 * models only (PRLAB_EINVAL otherwise, with the reference's message). */
int prlab_gpu_classifier_probs(prlab_gpu_model* m, const int32_t* ids, int64_t batch, int64_t seq,
                               const prlab_policy* policy, float* probs);

/* Device-resident form: d_ids [B*S] int32 on the device, logits written to
 * d_out with row pitch `ld` elements (ld >= V) in out_dtype (columns V .. ld-1 are
 * scratch: the head's TMA store may fill them up to the next 16-byte boundary; fp32
 * logits with ld % 4 == 0 come straight from the head's epilogue, other pitches through
 * per-thread stores).  Asynchronous on
 * `stream` (cudaStream_t; NULL = legacy default).  With use_graph != 0 the
 * forward is captured once per (B,S,policy,out) key and replayed as a CUDA
 * graph.  Ids are validated on the device; an out-of-range id is reported by
 * the next call to prlab_gpu_sync_status(). */
int prlab_gpu_forward_device(prlab_gpu_model* m, const int32_t* d_ids, int64_t batch,
                             int64_t seq, const prlab_policy* policy, void* d_out,
                             int32_t out_dtype, int64_t ld, void* stream, int32_t use_graph);
/* The shared trunk alone (embeddings .. final LayerNorm, src/model.cpp:350-452
 * forward_hidden, which forward() and classifier_probs() build on), enqueued on
 * `stream` without a graph; the hidden states stay in the model's workspace.  For
 * timing the trunk's kernels (batch-1 shapes: the single persistent kernel).
 * *kernels (optional) receives the number of kernels launched. */
int prlab_gpu_forward_trunk_device(prlab_gpu_model* m, const int32_t* d_ids, int64_t batch,
                                   int64_t seq, const prlab_policy* policy, void* stream,
                                   int64_t* kernels);
/* Forward with the tied head's log-softmax statistics fused into the head GEMM's
 * epilogue (the reduction window_nll_sum, src/fidelity.cpp:213-240,
 * and greedy argmax apply to the logits of src/model.cpp:469-480): per row b*seq + s,
 * d_nll (double, may be NULL) = -log_softmax(logits row)[d_targets[row]] as
 * prlab_gpu_row_nll_device defines it, d_argmax (may be NULL) = first column of the row
 * maximum.  The [batch*seq, V] logits are never written to HBM.  Device pointers, async
 * on `stream`, no graph.  The fused epilogue runs on the tensor-core path (hybrid policy)
 * when the head is tiled by CTA pairs (batch*seq >= 512 rows); otherwise the logits go
 * through a workspace buffer and prlab_gpu_row_nll_device's kernel -- *fused (may be
 * NULL) tells which.  Bad ids: reported by prlab_gpu_sync_status(). */
int prlab_gpu_forward_nll_device(prlab_gpu_model* m, const int32_t* d_ids, const int32_t* d_targets,
                                 int64_t batch, int64_t seq, const prlab_policy* policy, double* d_nll,
                                 int32_t* d_argmax, void* stream, int32_t* fused);
/* Synchronizes the stream and reports deferred device-side errors (bad ids). */
int prlab_gpu_sync_status(prlab_gpu_model* m, void* stream);
/* Number of kernels one forward_device launch with FP16 logits issues for this key (for
 * bench accounting); _ex counts for either logits dtype (fp32 adds the widening kernel). */
int prlab_gpu_forward_kernel_count(prlab_gpu_model* m, int64_t batch, int64_t seq,
                                   const prlab_policy* policy, int64_t* count);
int prlab_gpu_forward_kernel_count_ex(prlab_gpu_model* m, int64_t batch, int64_t seq,
                                      const prlab_policy* policy, int32_t out_dtype, int64_t* count);

/* How prlab_gpu_forward moves this key's logits to the host (after its first call):
 * 0 = not decided yet, 1 = fp16 rows widened exactly on host threads (hybrid: the
 * logits are round16'd), 2 = fp32 device->host copy.  For bench accounting. */
int prlab_gpu_host_copy_mode(prlab_gpu_model* m, int64_t batch, int64_t seq, const prlab_policy* policy,
                             int32_t* mode);

/* ---- per-operator entry points mirroring include/prlab/kernels.hpp:30-70.
 * Host fp32 buffers in/out (the reference's Tensor storage), synchronous. */
int prlab_gpu_matmul(const float* a, const float* b, int64_t m, int64_t k, int64_t n,
                     prlab_kcfg cfg, float* out);                        /* kernels.cpp:40 */
int prlab_gpu_attention_scores(const float* q, const float* k, int64_t sq, int64_t sk,
                               int64_t d, float scale, prlab_kcfg cfg, float* out,
                               float* capture_f32);                      /* kernels.cpp:85 */
int prlab_gpu_softmax(const float* x, int64_t rows, int64_t n, prlab_kcfg cfg,
                      float* out);                                       /* kernels.cpp:127 */
int prlab_gpu_layernorm(const float* x, int64_t rows, int64_t n, const float* gamma,
                        const float* beta, float eps, prlab_kcfg cfg,
                        float* out);                                     /* kernels.cpp:170 */
int prlab_gpu_gelu(const float* x, int64_t n, prlab_kcfg cfg, float* out);      /* kernels.cpp:221 */
int prlab_gpu_add(const float* a, const float* b, int64_t n, prlab_kcfg cfg,
                  float* out);                                           /* kernels.cpp:237 */
int prlab_gpu_tanh(const float* x, int64_t n, prlab_kcfg cfg, float* out);      /* kernels.cpp:296 */
int prlab_gpu_embed(const float* tok, int64_t vocab, const float* pos, int64_t npos,
                    int64_t h, const int32_t* ids, int64_t batch, int64_t seq, prlab_kcfg cfg,
                    float* out);                                         /* kernels.cpp:256 */

/* ---- device-pointer building blocks (tests / bench of the hot kernels) ----
 * Hybrid Linear on tensor cores (tcgen05): out = epi(round16(A.W^T)), A fp16
 * [M,K] row-major, Wt fp16 [N,K] row-major (K-major), bias fp32 [N] or NULL.
 * epi: 0 = bias -> fp16 out; 1 = bias+GELU -> fp16 out; 2 = bias then fp32
 * residual add in place into out (fp32 [M,N]); 3 = no bias -> fp16 out; 5 = no bias ->
 * fp32 out holding the binary16 value round16(acc) (the tied head with fp32 logits).
 * ldo = row pitch of out in elements; when ldo > N the TMA-store epilogue may write the
 * row padding up to the next 16-byte boundary (never past ldo). */
int prlab_gpu_linear_f16_device(const void* A, const void* Wt, const float* bias, void* out,
                                int64_t M, int64_t N, int64_t K, int64_t ldo, int32_t epi,
                                void* stream);
/* Same with an explicit tile configuration (tuning sweeps): bn in {0 (auto), 64, 128, 256},
 * splits (0 = auto), lean (0 = auto, 1 = half-depth pipeline, -1 = full depth).  epi 4 (the
 * LM head's fused log-softmax statistics, CTA-pair kernel only, M >= 512): out = float4
 * [ceil(N / BN)][M] per-row (max, sum exp(v - max), first argmax column, non-finite flag)
 * partials, no targets -- the head kernel of forward_nll_device, for timing. */
int prlab_gpu_linear_f16_device_ex(const void* A, const void* Wt, const float* bias, void* out,
                                   int64_t M, int64_t N, int64_t K, int64_t ldo, int32_t epi,
                                   int32_t bn, int32_t splits, int32_t lean, void* stream);
/* fp32-policy linear on the tensor cores (3xTF32, gemm_tf32.cu), device pointers:
 * out[M, N] (row pitch N) = epi(A[M, K] . Wt[N, K]^T), epi 0 = + bias (bias may be null),
 * 1 = GELU(+ bias) with exact erf, 2 = resid + (acc + bias) (resid [M, N], may alias out).
 * Replaces the fp32 linear_bias of src/kernels.cpp:40-83 under the fp32 policy; K % 32 == 0. */
int prlab_gpu_linear_f32_device(const float* A, const float* Wt, const float* bias, float* out, int64_t M,
                                int64_t N, int64_t K, int32_t epi, const float* resid, void* stream);
/* Fused hybrid attention on tensor cores: qkv fp16 [B*S, 3h] (q|k|v), ctx fp16 [B*S, h].
 * The streaming kernel's dynamic unit counter is per host thread and device: one host thread
 * must not have two of these calls in flight on different streams at once. */
int prlab_gpu_attention_f16_device(const void* qkv, void* ctx, int64_t batch, int64_t seq,
                                   int64_t heads, int64_t head_dim, int32_t causal,
                                   void* stream);

/* Debug variant: dbg (device, [grid][8] int64) receives clock64() phase stamps per CTA. */
int prlab_gpu_attention_f16_device_dbg(const void* qkv, void* ctx, int64_t batch, int64_t seq,
                                       int64_t heads, int64_t head_dim, int32_t causal,
                                       void* stream, long long* dbg);

/* Debug: GEMM launches after this call write %globaltimer phase stamps ([grid][8] int64,
 * device memory) into dbg (NULL switches the stamps off). */
int prlab_gpu_debug_gemm_stamps(long long* dbg);
/* Debug / parity: the hybrid hot path's embedding gather alone (embed(), src/kernels.cpp:256-294),
 * d_out fp32 [B*S, h] on the device.  path 0 = the multi-kernel path's gather kernel
 * (embed_f32_kernel), path 1 = stage 0 of the batch-1 persistent kernel (fwd_small).  Async. */
int prlab_gpu_debug_embedding_device(prlab_gpu_model* m, const int32_t* d_ids, int64_t batch, int64_t seq,
                                     int32_t path, float* d_out, void* stream);
/* Debug: per-stage %globaltimer stamps of the batch-1 persistent forward, [stage][grid][2]. */
int prlab_gpu_debug_small_stamps(long long* dbg);
/* Debug: phase stamps of the cluster batch-1 kernel, [cluster][CTA 0 / 15][layer][16]
 * (%globaltimer; slot 15 = cycles the MMA issuer waited for weights in that layer). */
int prlab_gpu_debug_cluster_stamps(long long* dbg);

#ifdef __cplusplus
}
#endif
#endif /* PRLAB_GPU_H */
