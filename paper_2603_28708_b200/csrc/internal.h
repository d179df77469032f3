// Host-side declarations shared between the C-ABI layer and the kernel files.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

namespace prlab_gpu {

// Exceptions thrown inside the library and mapped onto prlab_status codes at
// the C-ABI boundary (same classes the reference throws).
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define PRLAB_CUDA(call)                                                                    \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      throw ::prlab_gpu::cuda_error(std::string(#call) + ": " + cudaGetErrorString(e_));    \
  } while (0)

int num_sms();  // of the current device (cached per device)
bool pdl_enabled();
int current_device();

// Per-device one-time initialisation (cudaFuncSetAttribute, occupancy queries are per
// device): runs f() the first time it is reached on the current device, under `mu`, so a
// second model on another GPU -- or two threads racing on one -- never launches before
// its device is configured.
template <typename F>
void once_per_device(std::mutex& mu, uint64_t& done_mask, F&& f) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(mu);
  if ((done_mask >> (dev & 63)) & 1u) return;
  f();
  done_mask |= 1ull << (dev & 63);
}

// Launch with programmatic stream serialization (PDL) so the kernel's prologue
// overlaps the tail of the previous kernel in the stream / graph.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PRLAB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// --- TMA descriptors (driver entry point fetched through the runtime) ---
// 2-D fp16 tensor [rows, cols] with row pitch `pitch_elems`, box {box_cols, box_rows},
// 128-byte swizzle (box_cols * 2 must be 128).
CUtensorMap make_tmap_f16_2d(const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_elems,
                             uint32_t box_rows, uint32_t box_cols);
// 3-D fp16 tensor [d2, d1, d0] (d0 contiguous) with pitches in elements.
// 2-D fp32 tensor [rows, cols], box {box_cols, box_rows}, 128-byte swizzle (box_cols*4 == 128)
CUtensorMap make_tmap_f32_2d(const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_elems,
                             uint32_t box_rows, uint32_t box_cols);
CUtensorMap make_tmap_f16_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                             uint64_t pitch1_elems, uint64_t pitch2_elems, uint32_t box0,
                             uint32_t box1, uint32_t box2);

// --- tcgen05 GEMM: out = epi(A[M,K] . Wt[N,K]^T) ---
enum GemmEpi : int {
  EPI_BIAS_F16 = 0,       // round16(round16(acc) + b)              -> fp16
  EPI_BIAS_GELU_F16 = 1,  // round16(gelu(round16(round16(acc)+b))) -> fp16
  EPI_BIAS_RESID_F32 = 2, // x += round16(round16(acc) + b)          (fp32, in place)
  EPI_F16 = 3,            // round16(acc)                           -> fp16
  // per-row statistics of round16(acc) instead of the values (the LM head's fused
  // log-softmax / argmax): out = float4 [nslots][M] partials
  // (max, sum exp(v - max), first argmax column, non-finite flag), one slot per
  // n-block; tval[row] = v at targets[row].  Pair kernel only.
  EPI_ROWSTAT = 4,
  EPI_F16_F32 = 5,        // round16(acc)                           -> fp32 (the binary16 value, widened)
};
struct GemmPlan {
  CUtensorMap tmA, tmB, tmC;  // tmC: output map for the TMA-store epilogue
  bool tma_store;
  int M, N, K, bn, epi;
  int splits, kb_per_split;
  bool lean;
  bool cluster;  // split-K reduced through DSMEM inside a thread-block cluster
  bool pair;     // CTA-pair (cta_group::2) kernel, 256-row tiles
  bool pair_mc;  // pair kernel in 4-CTA clusters: weight tile multicast to both pairs
  const float* bias;
  void* out;
  int64_t ldo;
  float* ws;
  int* tickets;
  int grid;
  int group_m;  // raster band height (m-blocks)
  const int32_t* targets = nullptr;  // EPI_ROWSTAT
  float* tval = nullptr;
  int nslots = 0;
  bool acc16 = false;  // FP16 accumulator (full_fp16 fast path)
};
// Split-K scratch: fp32 partial tiles + per-tile tickets (zero between launches).
// One per model: kernels of one forward run in stream order, so they share it.
struct SplitScratch {
  float* ws = nullptr;
  size_t ws_floats = 0;
  int* tickets = nullptr;
  int n_tickets = 0;
};
SplitScratch& global_split_scratch();
long long*& debug_stamps();  // GEMM phase stamps target (debug; null = off)
GemmPlan plan_gemm_tc(const void* A, int64_t lda, const void* Wt, int64_t ldw, const float* bias,
                      void* out, int64_t ldo, int M, int N, int K, int epi,
                      const SplitScratch* scratch, int force_bn = 0, int force_splits = 0,
                      int force_lean = 0);
void launch_gemm_tc(const GemmPlan& p, cudaStream_t st);
void configure_gemm_tc();

// --- batch-1 forward_hidden as one cooperative persistent kernel (fwd_small.cu) ---
struct FwdSmallPlan {
  int M, B, S, h, f, H, L, V, causal;
  const void* host_lw;              // host array of per-layer LN / bias device pointers (8 per layer)
  const CUtensorMap* host_maps;     // host array: xn16, ff16, then Wqkv, Wo, W1, W2 per layer
  const float *tok, *pos, *lnfg, *lnfb;
  const int32_t* ids;
  int* err;
  float* x;
  __half *xn16, *ff16;
  float* scratch;            // fwd_small_workspace_floats()
  unsigned* gbar;            // kBarRegionBytes: the grid barrier counter, then per-QKV-task flags
  int embed_only = 0;        // debug: stop after the embedding stage (x = tok + pos)
};
constexpr int kFlagQkv = 16, kFlagFfn1 = kFlagQkv + 512, kFlagAttn = kFlagFfn1 + 256;  // u32 offsets
constexpr size_t kBarRegionBytes = 4 * (kFlagAttn + 4096);
bool fwd_small_supported(int64_t M, int64_t S, int64_t h, int64_t f, int64_t hd, int64_t L);
size_t fwd_small_workspace_floats(int64_t M, int64_t h, int64_t f);
int fwd_small_pair_n1(int64_t f);
void launch_fwd_small(const FwdSmallPlan& p, cudaStream_t st);
long long*& small_debug_stamps();  // [stage][grid][2] globaltimer stamps target (debug; null = off)

// --- batch-1 forward_hidden on 16-CTA clusters owning 32-row blocks (fwd_cluster.cu) ---
struct FwdClusterPlan {
  int M, S, L, V, causal;
  const void* host_lw;            // host array of per-layer {ln1g, ln1b, ln2g, ln2b, bqkv, bo, b1, b2}
  CUtensorMap ctx_map;            // ctx rows [12 kb][128 rows][64], box 32 rows x 12 kb
  const uint8_t* wstream;         // per-CTA weight streams (build_cluster_stream), L x 888 units of 16 KB
  const float *tok, *pos, *lnfg, *lnfb;
  const int32_t* ids;
  int* err;
  float* xg;
  __half* ctxg;
  __half* kvg;
  float* part;
  unsigned* flags;
  __half* xn16;
  int embed_only = 0;
};
bool fwd_cluster_supported(int64_t M, int64_t S, int64_t h, int64_t f, int64_t H, int64_t L);
size_t fwd_cluster_workspace_bytes(int64_t L);
size_t cluster_stream_bytes_per_layer();
void build_cluster_stream(const __half* wqkv, const __half* wo, const __half* w1, const __half* w2, void* dst,
                          cudaStream_t st);
void launch_fwd_cluster(const FwdClusterPlan& p, cudaStream_t st);
long long*& cluster_debug_stamps();  // [cluster][2][L][16] globaltimer phase stamps (debug; null = off)

// --- fused tensor-core attention (hybrid, head_dim 64, seq <= 512) ---
struct AttnPlan {
  CUtensorMap tmQKV;
  void* ctx;
  int B, S, H, hd, causal;
  int64_t ld_qkv, ld_ctx;
  long long* dbg = nullptr;  // phase timestamps (debug)
  int unstab = 0;            // unstabilised softmax (full_fp16 fast path, kernels.cpp:155): no max shift
  const int* fa_sched = nullptr;  // streaming kernel's balanced unit schedule (attn_fa_schedule)
  int* fa_work = nullptr;         // its dynamic-schedule counter [2] (zeroed; owned by the caller's plan)
};
bool attn_tc_supported(int S, int hd);
AttnPlan plan_attn_tc(const void* qkv, int64_t ld_qkv, void* ctx, int64_t ld_ctx, int B, int S,
                      int H, int hd, int causal);
// tap (optional): [B][H][S][S] fp32 pre-mask scores (the reference's retain_scores capture)
void launch_attn_tc(const AttnPlan& p, cudaStream_t st, float* tap = nullptr);
void configure_attn_tc();
// key-block streaming variant (attn_fa.cu: online softmax, two CTAs per SM); launch_attn_tc
// dispatches to it when no tap is requested unless PRLAB_ATTN_FA=0
bool attn_fa_enabled();
void launch_attn_fa(const AttnPlan& p, cudaStream_t st);
// device table of the streaming kernel's per-CTA unit lists (built once per shape, at plan time)
const int* attn_fa_schedule(int B, int S, int H, int causal);

// --- fp32-policy linears on the tensor cores: 3xTF32 tcgen05 GEMM (gemm_tf32.cu) ---
// lo = w - trunc19(w) (the part of each fp32 value kind::tf32 drops)
void split_lo(const float* w, float* lo, int64_t n, cudaStream_t st);
bool gemm_tf32_ok(const float* A, int64_t lda, const float* W, int64_t ldw, int64_t K);
// out = epi(A . W^T): op 0 (+bias), 1 GELU (exact erf), 2 residual (out = resid + v); fp32
void gemm_tf32(const float* A, int64_t lda, const float* W, const float* Wlo, int64_t ldw, float* out, int64_t ldo,
               int M, int N, int K, const float* bias, int op, const float* resid, float* ws, size_t ws_floats,
               cudaStream_t st);

// --- SIMT kernels (any shape, any policy; fp32 storage) ---
struct Kcfg {
  int compute, accum, stabilized;
};
// out[m,n] = epilogue( sum_k A[m,k] * Bt[n,k] ) with the reference linear_bias /
// matmul semantics under `lin`; op: 0 none, 1 gelu (act cfg), 2 residual add
// into `resid` (res cfg, written to out).
struct SimtGemmEpi {
  const float* bias;  // may be null (plain matmul)
  int op;
  Kcfg act, res;
  const float* resid;  // residual input (may alias out)
};
void simt_gemm(const float* A, int64_t lda, const float* Bt, int64_t ldb, float* out,
               int64_t ldo, int M, int N, int K, Kcfg lin, const SimtGemmEpi& epi,
               cudaStream_t st);
void simt_embed(const float* tok, int64_t vocab, const float* pos, int h, const int32_t* ids,
                int B, int S, Kcfg cfg, float* out, int* err_flag, cudaStream_t st);
void simt_layernorm(const float* x, int rows, int n, const float* gamma, const float* beta,
                    float eps, Kcfg cfg, float* out_f32, __half* out_f16, int round_out16,
                    cudaStream_t st);
// Generic attention: q/k/v columns inside row-major [B*S, ld] buffers.
void simt_attention(const float* q, const float* k, const float* v, int64_t ld_in, float* ctx,
                    int64_t ld_ctx, int B, int S, int H, int hd, float scale, int causal,
                    Kcfg att, Kcfg sm, float* tap, cudaStream_t st);
void simt_scores(const float* q, const float* k, int sq, int sk, int d, float scale, Kcfg cfg,
                 float* out, float* tap, cudaStream_t st);
void simt_softmax(const float* x, int64_t rows, int64_t n, Kcfg cfg, float* out, cudaStream_t st);
void simt_gelu(const float* x, int64_t n, Kcfg cfg, float* out, cudaStream_t st);
void simt_add(const float* a, const float* b, int64_t n, Kcfg cfg, float* out, cudaStream_t st);
void simt_tanh(const float* x, int64_t n, Kcfg cfg, float* out, cudaStream_t st);
// device logits reductions (logits_reduce.cu): per row NLL of targets[row] (skipped
// when < 0; double) and argmax; compare_logits partials [rows][7]
// fold the EPI_ROWSTAT partials of the LM head: per row NLL of the target (as row_nll)
// and the first argmax column
void rowstat_combine(const void* stat, int nslots, int64_t rows, int64_t n, const int32_t* targets,
                     const float* tval, double* nll, int32_t* amax, cudaStream_t st);
void row_nll(const void* logits, int dtype, int64_t rows, int64_t n, int64_t ld, const int32_t* targets,
             double* nll, int32_t* amax, cudaStream_t st);
void compare_rows(const void* base, int base_dtype, int64_t ldb, const void* cand, int cand_dtype, int64_t ldc,
                  int64_t rows, int64_t n, double* part, cudaStream_t st);
// classifier mean pool over the sequence (x32 or x16 [B*S, h]) -> out [B, h] fp32
void simt_pool_mean(const float* x32, const __half* x16, int B, int S, int h, Kcfg lin, float* out,
                    cudaStream_t st);
void simt_round_copy(const float* x, int64_t n, int f16, float* out, cudaStream_t st);
// fp16 padded [M, ld16] -> fp32 dense [M, N]
// Device fp16 rows (pitch ld_src halves) -> host fp32 rows (pitch ld_dst), copied in
// row chunks and widened on host threads as each chunk lands (host_widen.cpp).  Exact;
// returns once every row is in h_dst.
void d2h_widen_f16(const void* d_src, int64_t ld_src, float* h_dst, int64_t ld_dst, int64_t rows, int64_t cols,
                   cudaStream_t st);
void convert_f16_to_f32(const __half* in, int64_t ld_in, float* out, int64_t ld_out, int M, int N,
                        cudaStream_t st);
void f32_to_f16(const float* in, __half* out, int64_t n, cudaStream_t st);
void transpose_f32(const float* in, int rows, int cols, float* out, int round16, cudaStream_t st);
void transpose_to_f16(const float* in, int rows, int cols, __half* out, int64_t ld_out,
                      cudaStream_t st);
void round16_inplace(float* x, int64_t n, cudaStream_t st);

// fast-path LayerNorm for h % 128 == 0 (warp per row): fp32 x -> fp16 lattice (hybrid)
// x_round (full_fp16 fast path): x itself, rounded onto the binary16 lattice in place first
void ln_f32_to_f16(const float* x, int rows, int n, const float* gamma, const float* beta,
                   float eps, __half* out, cudaStream_t st, float* x_round = nullptr);
// fast embed for the hybrid path (fp32 add, float4)
void embed_f32(const float* tok, int64_t vocab, const float* pos, int h, const int32_t* ids,
               int B, int S, float* out, int* err_flag, cudaStream_t st);

// greedy argmax per row (lowest index wins ties, NaN never wins); dtype 0 fp32, 1 fp16
void argmax_rows(const void* logits, int dtype, int64_t rows, int64_t n, int64_t ld, int32_t* out,
                 cudaStream_t st);

}  // namespace prlab_gpu
