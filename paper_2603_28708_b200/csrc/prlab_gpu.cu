// Host runtime behind include/prlab_gpu.h: weight arena planner, device model,
// forward orchestration (fast tcgen05 path / generic SIMT path), CUDA-graph
// cache, and the C-ABI with the reference's error semantics.
//
// Reference call stack being replaced: prlab::forward -> forward_hidden
// (src/model.cpp:350-482) -> embed / layernorm_lastdim / linear_bias / matmul /
// attention_scores / softmax_lastdim / gelu / add (src/kernels.cpp).
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/prlab_gpu.h"
#include <fstream>
#include <cctype>
#include "common.cuh"
#include "internal.h"

namespace prlab_gpu {

namespace {
thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return PRLAB_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return PRLAB_EINVAL;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return PRLAB_ERANGE;
  } catch (const cuda_error& e) {
    g_last_error = e.what();
    return PRLAB_ECUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PRLAB_ERUNTIME;
  }
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
    cudaGetLastError();
    throw cuda_error("no CUDA device available (prlab_gpu has no CPU fallback)");
  }
}
}  // namespace

int current_device() {
  int dev = 0;
  PRLAB_CUDA(cudaGetDevice(&dev));
  return dev;
}

int num_sms() {
  static int n[64] = {};
  const int dev = current_device() & 63;
  if (n[dev] == 0) {
    int v = 0;
    PRLAB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    n[dev] = v;
  }
  return n[dev];
}

bool pdl_enabled() {
  static const bool on = std::getenv("PRLAB_NO_PDL") == nullptr;
  return on;
}

// ---------------------------------------------------------------------------
// TMA descriptors through the driver entry point (no -lcuda link dependency)
// ---------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    PRLAB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw cuda_error("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
}  // namespace

CUtensorMap make_tmap_f16_2d(const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_elems,
                             uint32_t box_rows, uint32_t box_cols) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_elems * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled(2d) failed: " + std::to_string(r));
  return m;
}

CUtensorMap make_tmap_f32_2d(const void* base, uint64_t rows, uint64_t cols, uint64_t pitch_elems,
                             uint32_t box_rows, uint32_t box_cols) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_elems * 4};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled(f32 2d) failed: " + std::to_string(r));
  return m;
}

CUtensorMap make_tmap_f16_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                             uint64_t pitch1_elems, uint64_t pitch2_elems, uint32_t box0,
                             uint32_t box1, uint32_t box2) {
  CUtensorMap m;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {pitch1_elems * 2, pitch2_elems * 2};
  cuuint32_t box[3] = {box0, box1, box2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled(3d) failed: " + std::to_string(r));
  return m;
}

// ---------------------------------------------------------------------------
// arena planner: one cudaMalloc, 1 KiB-aligned carve-outs (TMA / 128B swizzle)
// ---------------------------------------------------------------------------
namespace {
struct ArenaPlan {
  std::vector<size_t> offs;
  size_t total = 0;
  int add(size_t bytes) {
    total = (total + 1023) & ~static_cast<size_t>(1023);
    offs.push_back(total);
    total += bytes;
    return static_cast<int>(offs.size()) - 1;
  }
};

struct DeviceBuffer {
  void* p = nullptr;
  size_t bytes = 0;
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { reset(); }
  void alloc(size_t n) {
    reset();
    if (n) PRLAB_CUDA(cudaMalloc(&p, n));
    bytes = n;
  }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* at(size_t off) const {
    return reinterpret_cast<T*>(static_cast<uint8_t*>(p) + off);
  }
};

Kcfg K(const prlab_kcfg& c) { return Kcfg{c.compute, c.accum, c.stabilized}; }

// The built-in hybrid assignment (src/policy.cpp:59-63): Linear, AttentionScoreMatmul,
// Activation {F16E, F32}; Softmax, LayerNorm, Embedding, Residual {F32, F32}, stabilized softmax.
bool is_hybrid(const prlab_policy& p) {
  for (int i = 0; i < PRLAB_NUM_OP_CLASSES; ++i) {
    const prlab_kcfg& c = p.cls[i];
    const bool narrow = i == PRLAB_LINEAR || i == PRLAB_ATTENTION_SCORE_MATMUL || i == PRLAB_ACTIVATION;
    if (c.compute != (narrow ? 1 : 0) || c.accum != 0) return false;
    if (i == PRLAB_SOFTMAX && !c.stabilized) return false;
  }
  return true;
}
// The built-in full_fp16 assignment (src/policy.cpp:55): every class {F16E, F16E}, unstabilised.
bool is_full_fp16(const prlab_policy& p) {
  for (int i = 0; i < PRLAB_NUM_OP_CLASSES; ++i) {
    const prlab_kcfg& c = p.cls[i];
    if (c.compute != 1 || c.accum != 1 || c.stabilized) return false;
  }
  return true;
}
uint64_t policy_key(const prlab_policy& p) {
  uint64_t k = 0;
  for (int i = 0; i < PRLAB_NUM_OP_CLASSES; ++i)
    k = (k << 3) | (static_cast<uint64_t>(p.cls[i].compute & 1) << 2) |
        (static_cast<uint64_t>(p.cls[i].accum & 1) << 1) |
        static_cast<uint64_t>(p.cls[i].stabilized != 0);
  return k;
}
void validate_kcfg(const prlab_kcfg& c) {
  if ((c.compute != 0 && c.compute != 1) || (c.accum != 0 && c.accum != 1))
    throw std::invalid_argument("unknown dtype in kernel config");
  if (c.compute == 0 && c.accum == 1)  // KernelConfig::validate, src/kernels.cpp:33-38
    throw std::invalid_argument("invalid kernel config: f32 compute with f16e accumulation");
}
void validate_policy(const prlab_policy& p) {
  for (int i = 0; i < PRLAB_NUM_OP_CLASSES; ++i) validate_kcfg(p.cls[i]);
}

void validate_desc(const prlab_model_desc& c) {
  // ModelConfig::validate, src/model.cpp:101-117 (same messages)
  if (c.num_layers < 0) throw std::invalid_argument("num_layers must be >= 0");
  if (c.hidden < 1) throw std::invalid_argument("hidden must be >= 1");
  if (c.heads < 1) throw std::invalid_argument("heads must be >= 1");
  if (c.ffn < 1) throw std::invalid_argument("ffn must be >= 1");
  if (c.vocab < 1) throw std::invalid_argument("vocab must be >= 1");
  if (c.max_positions < 1) throw std::invalid_argument("max_positions must be >= 1");
  if (c.hidden % c.heads != 0)
    throw std::invalid_argument("heads (" + std::to_string(c.heads) + ") must divide hidden (" +
                                std::to_string(c.hidden) + ")");
  if (c.ffn < c.hidden)
    throw std::invalid_argument("ffn (" + std::to_string(c.ffn) + ") must be >= hidden (" +
                                std::to_string(c.hidden) + ")");
  if (c.archetype != 0 && c.archetype != 1)
    throw std::invalid_argument("unknown archetype (expected encoder_only or decoder_only)");
}

std::vector<size_t> param_sizes(const prlab_model_desc& d) {
  const size_t h = d.hidden, f = d.ffn;
  std::vector<size_t> s = {static_cast<size_t>(d.vocab) * h, static_cast<size_t>(d.max_positions) * h};
  for (int64_t l = 0; l < d.num_layers; ++l) {
    const size_t lay[16] = {h, h, h * h, h, h * h, h, h * h, h, h * h, h, h, h, h * f, f, f * h, h};
    s.insert(s.end(), lay, lay + 16);
  }
  s.push_back(h);
  s.push_back(h);
  if (d.archetype == 0) {
    s.push_back(h * h);
    s.push_back(h);
    s.push_back(h * 2);
    s.push_back(2);
  }
  return s;
}

// Model::for_each_param canonical names and shapes (src/model.cpp:178-209)
std::vector<std::pair<std::string, std::vector<int64_t>>> param_specs(const prlab_model_desc& d) {
  const int64_t h = d.hidden, f = d.ffn;
  std::vector<std::pair<std::string, std::vector<int64_t>>> s = {{"token_embedding", {d.vocab, h}},
                                                                  {"position_embedding", {d.max_positions, h}}};
  for (int64_t l = 0; l < d.num_layers; ++l) {
    const std::string p = "layers." + std::to_string(l) + ".";
    s.push_back({p + "ln1.gamma", {h}});
    s.push_back({p + "ln1.beta", {h}});
    s.push_back({p + "attn.wq", {h, h}});
    s.push_back({p + "attn.bq", {h}});
    s.push_back({p + "attn.wk", {h, h}});
    s.push_back({p + "attn.bk", {h}});
    s.push_back({p + "attn.wv", {h, h}});
    s.push_back({p + "attn.bv", {h}});
    s.push_back({p + "attn.wo", {h, h}});
    s.push_back({p + "attn.bo", {h}});
    s.push_back({p + "ln2.gamma", {h}});
    s.push_back({p + "ln2.beta", {h}});
    s.push_back({p + "ffn.w1", {h, f}});
    s.push_back({p + "ffn.b1", {f}});
    s.push_back({p + "ffn.w2", {f, h}});
    s.push_back({p + "ffn.b2", {h}});
  }
  s.push_back({"final_ln.gamma", {h}});
  s.push_back({"final_ln.beta", {h}});
  if (d.archetype == 0) {
    s.push_back({"pooler.weight", {h, h}});
    s.push_back({"pooler.bias", {h}});
    s.push_back({"classifier.weight", {h, 2}});
    s.push_back({"classifier.bias", {2}});
  }
  return s;
}

std::string shape_str(const std::vector<int64_t>& v) {  // src/tensor.cpp:27-36
  std::string o = "[";
  for (size_t i = 0; i < v.size(); ++i) o += (i ? ", " : "") + std::to_string(v[i]);
  return o + "]";
}

// binary16 -> fp32 (f16_decode, src/float16.cpp; exact for every non-NaN encoding)
float f16_decode_host(uint16_t h) {
  const uint32_t sign = (h & 0x8000u) << 16, e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
  uint32_t u;
  if (e == 0x1F) {
    u = m ? 0x7FC00000u : (sign | 0x7F800000u);
  } else if (e == 0) {
    float v = static_cast<float>(m) * 5.9604644775390625e-08f;  // m * 2^-24, exact
    std::memcpy(&u, &v, 4);
    u |= sign;
  } else {
    u = sign | ((e + 112u) << 23) | (m << 13);
  }
  float x;
  std::memcpy(&x, &u, 4);
  return x;
}

// The flat JSON object config_to_json writes (src/model.cpp:148-176): string / integer
// values only; "preset" names the reference presets (src/model.cpp:122-136).
prlab_model_desc config_from_json(const std::string& js) {
  std::map<std::string, std::string> kv;
  size_t i = 0;
  auto ws = [&] { while (i < js.size() && std::isspace(static_cast<unsigned char>(js[i]))) ++i; };
  auto str = [&]() {
    if (js[i] != '"') throw std::runtime_error("checkpoint config is not valid JSON");
    std::string o;
    for (++i; i < js.size() && js[i] != '"'; ++i) o += js[i];
    ++i;
    return o;
  };
  ws();
  if (i >= js.size() || js[i] != '{') throw std::runtime_error("checkpoint config is not a JSON object");
  ++i;
  for (ws(); i < js.size() && js[i] != '}';) {
    const std::string k = str();
    ws();
    if (js[i] != ':') throw std::runtime_error("checkpoint config is not valid JSON");
    ++i;
    ws();
    std::string v;
    if (js[i] == '"') {
      v = str();
    } else {
      while (i < js.size() && js[i] != ',' && js[i] != '}' && !std::isspace(static_cast<unsigned char>(js[i]))) v += js[i++];
    }
    kv[k] = v;
    ws();
    if (js[i] == ',') ++i;
    ws();
  }
  prlab_model_desc d{};
  auto preset = [&](const std::string& n) {
    if (n == "bert_base") d = {0, 12, 768, 12, 3072, 30522, 512, 0};
    else if (n == "gpt2_small") d = {1, 12, 768, 12, 3072, 50257, 1024, 0};
    else if (n == "encoder_toy") d = {0, 4, 128, 4, 256, 320, 160, 0};
    else if (n == "decoder_toy") d = {1, 4, 128, 4, 256, 320, 160, 0};
    else
      throw std::invalid_argument("unknown model preset '" + n + "' (valid: bert_base, gpt2_small, encoder_toy, decoder_toy)");
  };
  d = {1, 0, 0, 0, 0, 0, 0, 0};  // ModelConfig defaults (include/prlab/model.hpp:21-29)
  if (kv.count("preset")) preset(kv["preset"]);
  if (kv.count("archetype")) {
    if (kv["archetype"] == "encoder_only") d.archetype = 0;
    else if (kv["archetype"] == "decoder_only") d.archetype = 1;
    else throw std::invalid_argument("unknown archetype '" + kv["archetype"] + "' (expected encoder_only or decoder_only)");
  }
  auto num = [&](const char* k, int64_t& dst) { if (kv.count(k)) dst = std::stoll(kv[k]); };
  num("num_layers", d.num_layers);
  num("hidden", d.hidden);
  num("heads", d.heads);
  num("ffn", d.ffn);
  num("vocab", d.vocab);
  num("max_positions", d.max_positions);
  if (kv.count("seed")) d.seed = std::stoull(kv["seed"]);
  validate_desc(d);
  return d;
}

// load_checkpoint (src/checkpoint.cpp:133-162): PRLABCKP v1, config JSON, tensor records
// in canonical order; f16 payloads are decoded exactly (they land on the fp16 arena as-is).
std::vector<std::vector<float>> read_checkpoint(const std::string& path, prlab_model_desc& desc) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open checkpoint: " + path);
  auto get_u32 = [&](const std::string& what) {
    unsigned char b[4];
    if (!in.read(reinterpret_cast<char*>(b), 4)) throw std::runtime_error("checkpoint truncated while reading " + what);
    return static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) | (static_cast<uint32_t>(b[2]) << 16) |
           (static_cast<uint32_t>(b[3]) << 24);
  };
  auto get_u64 = [&](const std::string& what) {
    const uint64_t lo = get_u32(what), hi = get_u32(what);
    return lo | (hi << 32);
  };
  char magic[8];
  if (!in.read(magic, 8) || std::memcmp(magic, "PRLABCKP", 8) != 0)
    throw std::runtime_error("not a checkpoint (bad magic): " + path);
  const uint32_t version = get_u32("format version");
  if (version != 1) throw std::runtime_error("unsupported checkpoint version " + std::to_string(version));
  const uint32_t cfg_len = get_u32("config length");
  std::string cfg(cfg_len, '\0');
  if (!in.read(cfg.data(), cfg_len)) throw std::runtime_error("checkpoint truncated while reading config");
  desc = config_from_json(cfg);
  const auto specs = param_specs(desc);
  std::vector<std::vector<float>> params;
  params.reserve(specs.size());
  for (const auto& sp : specs) {
    const uint32_t name_len = get_u32("tensor name length");
    std::string name(name_len, '\0');
    if (!in.read(name.data(), name_len)) throw std::runtime_error("checkpoint truncated while reading tensor name");
    if (name != sp.first) throw std::runtime_error("unexpected tensor '" + name + "' (wanted '" + sp.first + "')");
    const int tag = in.get();
    if (tag != 0 && tag != 1)
      throw std::runtime_error("tensor '" + name + "' has unknown dtype tag " + std::to_string(tag));
    const uint32_t rank = get_u32("tensor rank");
    std::vector<int64_t> shape(rank);
    int64_t numel = 1;
    for (uint32_t r = 0; r < rank; ++r) {
      shape[r] = static_cast<int64_t>(get_u64("tensor extent"));
      numel *= shape[r];
    }
    std::vector<float> t(static_cast<size_t>(numel));
    if (tag == 0) {
      for (auto& v : t) {
        const uint32_t u = get_u32("tensor payload");
        std::memcpy(&v, &u, 4);
      }
    } else {
      std::vector<unsigned char> raw(static_cast<size_t>(numel) * 2);
      if (!in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size())))
        throw std::runtime_error("checkpoint truncated while reading tensor payload");
      for (size_t k = 0; k < t.size(); ++k)
        t[k] = f16_decode_host(static_cast<uint16_t>(raw[2 * k] | (raw[2 * k + 1] << 8)));
    }
    if (shape != sp.second)
      throw std::runtime_error("tensor '" + name + "' has shape " + shape_str(shape) + ", expected " +
                               shape_str(sp.second));
    params.push_back(std::move(t));
  }
  return params;
}
}  // namespace

}  // namespace prlab_gpu

using namespace prlab_gpu;

// ---------------------------------------------------------------------------
// device model
// ---------------------------------------------------------------------------
struct prlab_gpu_model {
  prlab_model_desc d{};
  int device = 0;
  int64_t h = 0, f = 0, H = 0, hd = 0, V = 0, P = 0, L = 0;
  std::mutex mu;
  std::vector<std::vector<float>> host;  // fp32 parameter copies (for the lazily built fp32 arena)

  // fast (hybrid) arena: fp16 K-major linear weights + fp32 tables / LN params,
  // biases pre-rounded onto the fp16 lattice (the reference's conform(b), model.cpp:73)
  DeviceBuffer arena16;
  struct L16 {
    __half *wqkv, *wo, *w1, *w2;
    float *bqkv, *bo, *b1, *b2, *ln1g, *ln1b, *ln2g, *ln2b;
  };
  std::vector<L16> l16;
  __half* emb16 = nullptr;  // tied head E [V, h] fp16 (already K-major)
  float *tok = nullptr, *pos = nullptr, *lnfg = nullptr, *lnfb = nullptr;

  // generic fp32 arena: W^T fp32 [out, in] and raw fp32 biases
  DeviceBuffer arena32;
  struct L32 {
    float *wqkv_t, *wo_t, *w1_t, *w2_t, *bqkv, *bo, *b1, *b2;
  };
  std::vector<L32> l32;
  bool have32 = false;
  // 3xTF32 residues w - trunc19(w) of the fp32 linears and the tied head (gemm_tf32.cu),
  // built with the first plan of a plain-fp32 policy
  DeviceBuffer arena32lo;
  struct L32lo {
    float *wqkv, *wo, *w1, *w2;
  };
  std::vector<L32lo> l32lo;
  float* tok_lo = nullptr;
  bool have32lo = false;

  // encoder classifier head (pooler [h,h], classifier [h,2]) as fp32 W^T + biases,
  // uploaded on the first classifier_probs call
  DeviceBuffer cls_arena;
  float *pool_wt = nullptr, *pool_b = nullptr, *cls_wt = nullptr, *cls_b = nullptr;

  DeviceBuffer cl_stream;  // batch-1 cluster kernel: per-CTA weight streams (built with its first plan)
  DeviceBuffer err;  // device error word (bad token ids)
  DeviceBuffer split_ws, split_tickets;
  SplitScratch scratch;
  cudaStream_t stream = nullptr;  // private stream of the host (drop-in) forward
  // Host forward copy-out slots (prlab_gpu_forward, hybrid, logits widened on the host): the
  // call enqueues its compute under `mu` into slot s's device logits, releases `mu`, and copies
  // slot s out on the slot's own stream -- a concurrent caller's compute overlaps that copy-out.
  // A slot's mutex is held from before its compute is enqueued until its copy-out finished.
  struct HostSlot {
    std::mutex mu;
    DeviceBuffer buf;
    cudaStream_t cs = nullptr;
    cudaEvent_t ready = nullptr;  // the slot's logits are written (recorded on the compute stream)
  };
  HostSlot hslot[2];
  uint64_t hslot_next = 0;
  // Every call shares the workspace below (activations, split-K scratch, the persistent
  // kernel's grid-barrier counter, graphs): work queued on a stream other than the previous
  // call's waits on this event, recorded after that call's work (see StreamOrder).
  cudaEvent_t last_ev = nullptr;
  cudaStream_t last_st = nullptr;
  bool have_last = false;

  // activation workspace + per-key plans
  DeviceBuffer ws;
  struct Plan {
    int64_t B = 0, S = 0;
    bool fast = false;
    bool fp16 = false;  // full_fp16 on the tensor cores (fast16_eligible)
    prlab_policy pol{};
    float* x = nullptr;
    __half *xn16 = nullptr, *big16 = nullptr, *logit16 = nullptr;
    float *xn32 = nullptr, *qkv32 = nullptr, *ctx32 = nullptr, *ff32 = nullptr;
    int32_t* ids = nullptr;
    float* out32 = nullptr;    // fp32 logits staging (host forward / generic path), allocated on first use
    int64_t ld16 = 0, outw = 0;
    DeviceBuffer lazy16, lazy32;  // the [B*S, V] logits buffers are not part of the planned workspace
    // host forward copy-out: 0 = not calibrated, 1 = fp16 rows widened on host, 2 = fp32 copy
    int copy_mode = 0;
    std::vector<GemmPlan> gemms;  // fast path: 4 per layer + head
    AttnPlan attn{};
    // batch-1 shapes: forward_hidden as one cooperative persistent kernel (fwd_small.cu)
    bool small = false;
    FwdSmallPlan sp{};
    DeviceBuffer small_buf;  // ctx16 + scratch + barrier counter
    std::vector<CUtensorMap> small_maps;
    std::vector<std::array<const void*, 12>> small_lw;
    // batch-1 shapes on 16-CTA clusters (fwd_cluster.cu); preferred over fwd_small when supported
    bool cluster = false;
    FwdClusterPlan cp{};
    DeviceBuffer cl_buf;
    std::vector<std::array<const float*, 8>> cl_lw;
    std::map<std::tuple<const void*, void*, int, int64_t>, cudaGraphExec_t> graphs;
    std::map<std::tuple<void*, int64_t, int>, GemmPlan> head_plans;  // (out, ld, epilogue)
    // fused head statistics (prlab_gpu_forward_nll_device): 0 = not planned, 1 = fused, 2 = unfused
    int rs_state = 0;
    GemmPlan rs_plan{};
    DeviceBuffer attn_work;  // the streaming attention's dynamic-schedule counter (int [2])
    DeviceBuffer rs_buf;  // float4 [nslots][M] partials + float [M] target logits
  };
  std::map<std::tuple<int64_t, int64_t, uint64_t>, std::unique_ptr<Plan>> plans;

  ~prlab_gpu_model() {
    drop_plans();
    for (auto& hs : hslot) {
      if (hs.cs) cudaStreamDestroy(hs.cs);
      if (hs.ready) cudaEventDestroy(hs.ready);
    }
    if (stream) cudaStreamDestroy(stream);
    if (last_ev) cudaEventDestroy(last_ev);
  }
  void drop_plans() {
    for (auto& kv : plans)
      for (auto& g : kv.second->graphs) cudaGraphExecDestroy(g.second);
    plans.clear();
  }
};

namespace {

// The library-side logits buffers ([B*S, V]: 1.65 GB fp16 / 3.3 GB fp32 at C4) exist only
// for callers that want the logits in the library (host forward, unfused NLL); a device
// forward into the caller's buffer or the fused NLL head never allocates them.
__half* plan_logits16(prlab_gpu_model::Plan& p) {
  if (!p.logit16) {
    p.lazy16.alloc(static_cast<size_t>(p.B * p.S * p.ld16) * 2);
    p.logit16 = static_cast<__half*>(p.lazy16.p);
  }
  return p.logit16;
}
float* plan_out32(prlab_gpu_model::Plan& p) {
  if (!p.out32) {
    p.lazy32.alloc(static_cast<size_t>(p.B * p.S * p.outw) * 4);
    p.out32 = static_cast<float*>(p.lazy32.p);
  }
  return p.out32;
}

// Stream ordering of one API call on the model's shared workspace (held under the model
// mutex): before queuing on `st`, wait for the previous call's work if that was queued on
// another stream; afterwards record the event on `st`.  Streams under the CALLER's graph
// capture are left alone (the caller orders its graph).
struct StreamOrder {
  prlab_gpu_model& m;
  cudaStream_t st;
  bool active = true;
  StreamOrder(prlab_gpu_model& mm, cudaStream_t s) : m(mm), st(s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    PRLAB_CUDA(cudaStreamIsCapturing(st, &cs));
    active = cs == cudaStreamCaptureStatusNone;
    if (active && m.have_last && m.last_st != st) PRLAB_CUDA(cudaStreamWaitEvent(st, m.last_ev, 0));
  }
  ~StreamOrder() {
    if (active && cudaEventRecord(m.last_ev, st) == cudaSuccess) {
      m.last_st = st;
      m.have_last = true;
    }
  }
};

// Fast (tensor-core) path eligibility: the hybrid policy and TMA-friendly extents.
bool tc_shape_ok(const prlab_gpu_model& m, int64_t S) {
  if (m.L < 1) return false;
  if (m.h % 128 != 0 || m.h > 1024 || m.f % 64 != 0) return false;
  if (!attn_tc_supported(static_cast<int>(S), static_cast<int>(m.hd))) return false;
  if (std::getenv("PRLAB_FORCE_GENERIC")) return false;
  return true;
}
bool fast_eligible(const prlab_gpu_model& m, int64_t S, const prlab_policy& pol) {
  return is_hybrid(pol) && tc_shape_ok(m, S);
}
// full_fp16 on the tensor cores (C5 speed arm): FP16 accumulators, the residual stream and
// every op output on the binary16 lattice, unstabilised softmax.  It rounds once per
// 16-wide MMA step instead of after every product (the reference's per-MAC emulation,
// src/kernels.cpp:56-66), so it is selected only when per-MAC exactness is not asked for:
// `exact` plans (retain_scores) and PRLAB_FP16_EXACT=1 keep the exact SIMT emulation that
// reproduces the reference's known-answer tests.
bool fast16_eligible(const prlab_gpu_model& m, int64_t S, const prlab_policy& pol, bool exact) {
  if (exact || !is_full_fp16(pol) || !tc_shape_ok(m, S)) return false;
  const char* e = std::getenv("PRLAB_FP16_EXACT");
  return e == nullptr || std::atoi(e) == 0;
}

void h2d(void* dst, const float* src, size_t n) {
  PRLAB_CUDA(cudaMemcpy(dst, src, n * sizeof(float), cudaMemcpyHostToDevice));
}

void upload_fast(prlab_gpu_model& m) {
  const int64_t h = m.h, f = m.f, V = m.V, P = m.P, L = m.L;
  ArenaPlan ap;
  const int s_tok = ap.add(V * h * 4), s_pos = ap.add(P * h * 4), s_emb = ap.add(V * h * 2);
  const int s_lnf = ap.add(2 * h * 4);
  std::vector<std::array<int, 12>> ls(L);
  for (int64_t l = 0; l < L; ++l)
    ls[l] = {ap.add(3 * h * h * 2), ap.add(h * h * 2), ap.add(f * h * 2), ap.add(h * f * 2),
             ap.add(3 * h * 4),     ap.add(h * 4),     ap.add(f * 4),     ap.add(h * 4),
             ap.add(h * 4),         ap.add(h * 4),     ap.add(h * 4),     ap.add(h * 4)};
  m.arena16.alloc(ap.total);
  auto at = [&](int s) { return ap.offs[s]; };
  m.tok = m.arena16.at<float>(at(s_tok));
  m.pos = m.arena16.at<float>(at(s_pos));
  m.emb16 = m.arena16.at<__half>(at(s_emb));
  m.lnfg = m.arena16.at<float>(at(s_lnf));
  m.lnfb = m.lnfg + h;
  cudaStream_t st = nullptr;
  h2d(m.tok, m.host[0].data(), V * h);
  h2d(m.pos, m.host[1].data(), P * h);
  f32_to_f16(m.tok, m.emb16, V * h, st);
  const size_t fin = 2 + 16 * L;
  h2d(m.lnfg, m.host[fin].data(), h);
  h2d(m.lnfb, m.host[fin + 1].data(), h);

  DeviceBuffer stage;
  stage.alloc(static_cast<size_t>(h) * std::max(h, f) * 4);
  auto rounded_bias = [&](float* dst, const std::vector<float>& src) {
    std::vector<float> tmp(src);
    for (auto& v : tmp) v = __half2float(__float2half_rn(v));
    h2d(dst, tmp.data(), tmp.size());
  };
  // W [in, out] row-major (model.cpp:229-242) -> W^T [out, in] fp16 (K-major)
  auto put = [&](const std::vector<float>& src, int64_t in, int64_t out, __half* dst) {
    h2d(stage.p, src.data(), in * out);
    transpose_to_f16(static_cast<float*>(stage.p), static_cast<int>(in), static_cast<int>(out), dst, in, st);
    PRLAB_CUDA(cudaStreamSynchronize(st));
  };
  m.l16.resize(L);
  for (int64_t l = 0; l < L; ++l) {
    const auto* p = &m.host[2 + 16 * l];
    auto& w = m.l16[l];
    w.wqkv = m.arena16.at<__half>(at(ls[l][0]));
    w.wo = m.arena16.at<__half>(at(ls[l][1]));
    w.w1 = m.arena16.at<__half>(at(ls[l][2]));
    w.w2 = m.arena16.at<__half>(at(ls[l][3]));
    w.bqkv = m.arena16.at<float>(at(ls[l][4]));
    w.bo = m.arena16.at<float>(at(ls[l][5]));
    w.b1 = m.arena16.at<float>(at(ls[l][6]));
    w.b2 = m.arena16.at<float>(at(ls[l][7]));
    w.ln1g = m.arena16.at<float>(at(ls[l][8]));
    w.ln1b = m.arena16.at<float>(at(ls[l][9]));
    w.ln2g = m.arena16.at<float>(at(ls[l][10]));
    w.ln2b = m.arena16.at<float>(at(ls[l][11]));
    h2d(w.ln1g, p[0].data(), h);
    h2d(w.ln1b, p[1].data(), h);
    h2d(w.ln2g, p[10].data(), h);
    h2d(w.ln2b, p[11].data(), h);
    put(p[2], h, h, w.wqkv);
    put(p[4], h, h, w.wqkv + h * h);
    put(p[6], h, h, w.wqkv + 2 * h * h);
    put(p[8], h, h, w.wo);
    put(p[12], h, f, w.w1);
    put(p[14], f, h, w.w2);
    rounded_bias(w.bqkv, p[3]);
    rounded_bias(w.bqkv + h, p[5]);
    rounded_bias(w.bqkv + 2 * h, p[7]);
    rounded_bias(w.bo, p[9]);
    rounded_bias(w.b1, p[13]);
    rounded_bias(w.b2, p[15]);
  }
  m.err.alloc(256);
  PRLAB_CUDA(cudaMemset(m.err.p, 0, 256));
  m.scratch.ws_floats = static_cast<size_t>(2 * num_sms()) * 128 * 128;
  m.split_ws.alloc(m.scratch.ws_floats * sizeof(float));
  m.scratch.ws = static_cast<float*>(m.split_ws.p);
  m.scratch.n_tickets = 4096;
  m.split_tickets.alloc(m.scratch.n_tickets * sizeof(int));
  PRLAB_CUDA(cudaMemset(m.split_tickets.p, 0, m.scratch.n_tickets * sizeof(int)));
  m.scratch.tickets = static_cast<int*>(m.split_tickets.p);
  PRLAB_CUDA(cudaDeviceSynchronize());
}

void ensure_f32(prlab_gpu_model& m) {
  if (m.have32) return;
  const int64_t h = m.h, f = m.f, L = m.L;
  ArenaPlan ap;
  std::vector<std::array<int, 8>> ls(L);
  for (int64_t l = 0; l < L; ++l)
    ls[l] = {ap.add(3 * h * h * 4), ap.add(h * h * 4), ap.add(f * h * 4), ap.add(h * f * 4),
             ap.add(3 * h * 4),     ap.add(h * 4),     ap.add(f * 4),     ap.add(h * 4)};
  m.arena32.alloc(std::max<size_t>(ap.total, 1024));
  DeviceBuffer stage;
  stage.alloc(static_cast<size_t>(h) * std::max(h, f) * 4);
  cudaStream_t st = nullptr;
  auto put = [&](const std::vector<float>& src, int64_t in, int64_t out, float* dst) {
    h2d(stage.p, src.data(), in * out);
    transpose_f32(static_cast<float*>(stage.p), static_cast<int>(in), static_cast<int>(out), dst, 0, st);
    PRLAB_CUDA(cudaStreamSynchronize(st));
  };
  m.l32.resize(L);
  for (int64_t l = 0; l < L; ++l) {
    const auto* p = &m.host[2 + 16 * l];
    auto& w = m.l32[l];
    auto at = [&](int i) { return m.arena32.at<float>(ap.offs[ls[l][i]]); };
    w.wqkv_t = at(0);
    w.wo_t = at(1);
    w.w1_t = at(2);
    w.w2_t = at(3);
    w.bqkv = at(4);
    w.bo = at(5);
    w.b1 = at(6);
    w.b2 = at(7);
    put(p[2], h, h, w.wqkv_t);
    put(p[4], h, h, w.wqkv_t + h * h);
    put(p[6], h, h, w.wqkv_t + 2 * h * h);
    put(p[8], h, h, w.wo_t);
    put(p[12], h, f, w.w1_t);
    put(p[14], f, h, w.w2_t);
    h2d(w.bqkv, p[3].data(), h);
    h2d(w.bqkv + h, p[5].data(), h);
    h2d(w.bqkv + 2 * h, p[7].data(), h);
    h2d(w.bo, p[9].data(), h);
    h2d(w.b1, p[13].data(), f);
    h2d(w.b2, p[15].data(), h);
  }
  PRLAB_CUDA(cudaDeviceSynchronize());
  m.have32 = true;
}

// fp32 policy on the tensor cores: linear / activation / residual classes all plain fp32
bool tf32_policy(const prlab_policy& pol) {
  auto f32 = [&](int c) { return pol.cls[c].compute == PRLAB_F32 && pol.cls[c].accum == PRLAB_F32; };
  return f32(PRLAB_LINEAR) && f32(PRLAB_ACTIVATION) && f32(PRLAB_RESIDUAL);
}

void ensure_f32lo(prlab_gpu_model& m) {
  if (m.have32lo) return;
  ensure_f32(m);
  const int64_t h = m.h, f = m.f, L = m.L;
  const int64_t per = 3 * h * h + h * h + f * h + h * f;
  m.arena32lo.alloc(static_cast<size_t>(per * L + m.V * h) * 4 + 1024);
  float* base = static_cast<float*>(m.arena32lo.p);
  m.l32lo.resize(L);
  for (int64_t l = 0; l < L; ++l) {
    float* b = base + per * l;
    auto& lo = m.l32lo[l];
    const auto& w = m.l32[l];
    lo = {b, b + 3 * h * h, b + 4 * h * h, b + 4 * h * h + f * h};
    split_lo(w.wqkv_t, lo.wqkv, 3 * h * h, nullptr);
    split_lo(w.wo_t, lo.wo, h * h, nullptr);
    split_lo(w.w1_t, lo.w1, f * h, nullptr);
    split_lo(w.w2_t, lo.w2, h * f, nullptr);
  }
  m.tok_lo = base + per * L;
  split_lo(m.tok, m.tok_lo, m.V * h, nullptr);
  PRLAB_CUDA(cudaDeviceSynchronize());
  m.have32lo = true;
}

// Batch-1 plan: tensor maps (activations box 128 x 64, weights box 32 x 64) and the
// the fp32 partials (per-head Wo, FFN2 K splits) and the grid-barrier counter live in
// one device buffer.
void plan_small(prlab_gpu_model& m, prlab_gpu_model::Plan& p, int64_t B, int64_t S) {
  const int64_t M = B * S, h = m.h, f = m.f, L = m.L;
  ArenaPlan ap;
  const int s_scr = ap.add(fwd_small_workspace_floats(M, h, f) * 4);
  const int s_bar = ap.add(kBarRegionBytes);
  p.small_buf.alloc(ap.total);
  char* base = static_cast<char*>(p.small_buf.p);
  auto& maps = p.small_maps;
  maps.clear();
  // K-major matrices viewed as [K/64 k-blocks][rows][64]: a box spans several k-blocks
  // (one TMA request per 2-4 k-blocks of A, one per task for B -- fwd_small.cu)
  auto kblk = [](const void* base, int64_t rows, int64_t K, uint32_t box_rows, uint32_t box_kb) {
    return make_tmap_f16_3d(base, 64, rows, K / 64, K, 64, 64, box_rows, box_kb);
  };
  maps.push_back(kblk(p.xn16, M, h, 128, 4));    // QKV / FFN1 A: 4 k-blocks per request
  maps.push_back(kblk(p.big16, M, f, 128, 4));   // FFN2 A (ff16 reuses the qkv/ff buffer)
  p.small_lw.assign(static_cast<size_t>(L), {});
  const int64_t kb_ffn2 = f / 64 / (f / 512);  // FFN2 split-K depth (launch_fwd_small)
  for (int64_t l = 0; l < L; ++l) {
    const auto& w = m.l16[l];
    // per-task weight boxes: QKV N = 16, FFN1 / FFN2 N = 32 (M > 128, CTA pairs: each CTA half of
    // the pair's N = 32 / 48 (64 when ffn % 48 != 0) / 64 -- fwd_small.cu)
    const bool pair = M > 128;
    maps.push_back(kblk(w.wqkv, 3 * h, h, 16, static_cast<uint32_t>(h / 64)));
    maps.push_back(make_tmap_f16_2d(w.wo, h, h, h, 256, 64));  // a head's Wo column slice, 256 rows per box
    maps.push_back(kblk(w.w1, f, h, pair ? static_cast<uint32_t>(fwd_small_pair_n1(f) / 2) : 32u,
                        static_cast<uint32_t>(h / 64)));  // (pair: each CTA half of the task's N)
    maps.push_back(kblk(w.w2, h, f, 32, static_cast<uint32_t>(kb_ffn2)));
    // (QKV / FFN2: the same boxes serve both kernels -- a pair's N is twice the single-CTA N)
    p.small_lw[l] = {w.ln1g, w.ln1b, w.ln2g, w.ln2b, w.bqkv, w.bo, w.b1, w.b2, w.wqkv, w.wo, w.w1, w.w2};
  }
  FwdSmallPlan& sp = p.sp;
  sp.M = static_cast<int>(M);
  sp.B = static_cast<int>(B);
  sp.S = static_cast<int>(S);
  sp.h = static_cast<int>(h);
  sp.f = static_cast<int>(f);
  sp.H = static_cast<int>(m.H);
  sp.L = static_cast<int>(L);
  sp.V = static_cast<int>(m.V);
  sp.causal = m.d.archetype == 1;
  sp.host_lw = p.small_lw.data();
  sp.host_maps = maps.data();
  sp.tok = m.tok;
  sp.pos = m.pos;
  sp.lnfg = m.lnfg;
  sp.lnfb = m.lnfb;
  sp.err = m.err.at<int>(0);
  sp.x = p.x;
  sp.xn16 = p.xn16;
  sp.ff16 = p.big16;
  sp.scratch = reinterpret_cast<float*>(base + ap.offs[s_scr]);
  sp.gbar = reinterpret_cast<unsigned*>(base + ap.offs[s_bar]);
  p.small = true;
}

// Cluster plan: per-layer weight maps (3D k-block views, boxes of 64 / 48 rows x one
// k-block), the ctx map (32 rows x 12 k-blocks), and the L2 exchange buffers.
void plan_cluster(prlab_gpu_model& m, prlab_gpu_model::Plan& p, int64_t B, int64_t S) {
  const int64_t M = B * S, h = m.h, L = m.L;
  if (m.cl_stream.p == nullptr) {  // once per model: every CTA rank's weights in consumption order
    const size_t per = cluster_stream_bytes_per_layer();
    m.cl_stream.alloc(per * static_cast<size_t>(L));
    for (int64_t l = 0; l < L; ++l) {
      const auto& w = m.l16[l];
      build_cluster_stream(w.wqkv, w.wo, w.w1, w.w2, static_cast<char*>(m.cl_stream.p) + per * l, nullptr);
    }
    PRLAB_CUDA(cudaDeviceSynchronize());
  }
  ArenaPlan ap;
  const int s_xg = ap.add(128 * h * 4), s_ctx = ap.add(128 * h * 2), s_kv = ap.add(L * 128 * 2 * h * 2),
            s_part = ap.add(4 * 16 * h * 32 * 4), s_flags = ap.add(L * 4 * 16 * 4);
  p.cl_buf.alloc(ap.total);
  char* base = static_cast<char*>(p.cl_buf.p);
  p.cl_lw.assign(static_cast<size_t>(L), {});
  for (int64_t l = 0; l < L; ++l) {
    const auto& w = m.l16[l];
    p.cl_lw[l] = {w.ln1g, w.ln1b, w.ln2g, w.ln2b, w.bqkv, w.bo, w.b1, w.b2};
  }
  __half* ctxg = reinterpret_cast<__half*>(base + ap.offs[s_ctx]);
  FwdClusterPlan& cp = p.cp;
  cp.ctx_map = make_tmap_f16_3d(ctxg, 64, 128, h / 64, h, 64, 64, 32, static_cast<uint32_t>(h / 64));
  cp.wstream = static_cast<const uint8_t*>(m.cl_stream.p);
  cp.M = static_cast<int>(M);
  cp.S = static_cast<int>(S);
  cp.L = static_cast<int>(L);
  cp.V = static_cast<int>(m.V);
  cp.causal = m.d.archetype == 1;
  cp.host_lw = p.cl_lw.data();
  cp.tok = m.tok;
  cp.pos = m.pos;
  cp.lnfg = m.lnfg;
  cp.lnfb = m.lnfb;
  cp.err = m.err.at<int>(0);
  cp.xg = reinterpret_cast<float*>(base + ap.offs[s_xg]);
  cp.ctxg = ctxg;
  cp.kvg = reinterpret_cast<__half*>(base + ap.offs[s_kv]);
  cp.part = reinterpret_cast<float*>(base + ap.offs[s_part]);
  cp.flags = reinterpret_cast<unsigned*>(base + ap.offs[s_flags]);
  cp.xn16 = p.xn16;
  p.cluster = true;
}

prlab_gpu_model::Plan& get_plan(prlab_gpu_model& m, int64_t B, int64_t S, const prlab_policy& pol,
                                bool exact = false) {
  const bool fast16 = fast16_eligible(m, S, pol, exact);
  const auto key = std::make_tuple(B, S, policy_key(pol) | (fast16 ? 1ull << 40 : 0ull));
  auto it = m.plans.find(key);
  if (it != m.plans.end()) return *it->second;

  const bool fast = fast_eligible(m, S, pol) || fast16;
  if (!fast) {
    ensure_f32(m);
    if (tf32_policy(pol) && !std::getenv("PRLAB_NO_TF32X3")) ensure_f32lo(m);
  }
  const int64_t M = B * S, h = m.h, f = m.f, V = m.V;
  const int64_t outw = m.L > 0 ? V : h;
  const int64_t ld16 = (V + 7) / 8 * 8;
  // Activation liveness: x (fp32 residual stream) lives throughout; xn (LN out)
  // dies at the QKV GEMM before ctx is born and ctx dies at Wo before LN2 writes
  // xn again -> one buffer.  qkv dies at attention before FFN1 writes ff -> one buffer.
  ArenaPlan ap;
  const int s_x = ap.add(M * h * 4);
  const int s_ids = ap.add(M * 4);
  int s_a, s_b, s_c = -1;
  if (fast) {
    s_a = ap.add(M * h * 2);                       // xn16 / ctx16
    s_b = ap.add(M * std::max(3 * h, f) * 2);      // qkv16 / ff16
  } else {
    s_a = ap.add(M * h * 4);                       // xn32
    s_b = ap.add(M * (3 * h + f) * 4);             // qkv32 | ff32 (attention reads qkv while ff unused)
    s_c = ap.add(M * h * 4);                       // ctx32
  }
  if (ap.total > m.ws.bytes) {
    m.drop_plans();  // every cached plan / graph points into the old workspace
    PRLAB_CUDA(cudaDeviceSynchronize());
    m.ws.alloc(ap.total);
  }
  auto plan = std::make_unique<prlab_gpu_model::Plan>();
  auto& p = *plan;
  p.B = B;
  p.S = S;
  p.pol = pol;
  p.fast = fast;
  p.fp16 = fast16;
  p.ld16 = ld16;
  auto at = [&](int s) { return ap.offs[s]; };
  p.x = m.ws.at<float>(at(s_x));
  p.ids = m.ws.at<int32_t>(at(s_ids));
  p.outw = outw;
  const int Mi = static_cast<int>(M), hi = static_cast<int>(h), fi = static_cast<int>(f);
  if (fast) {
    p.xn16 = m.ws.at<__half>(at(s_a));
    p.big16 = m.ws.at<__half>(at(s_b));
    for (int64_t l = 0; l < m.L; ++l) {
      const auto& w = m.l16[l];
      p.gemms.push_back(plan_gemm_tc(p.xn16, h, w.wqkv, h, w.bqkv, p.big16, 3 * h, Mi, 3 * hi, hi, EPI_BIAS_F16, &m.scratch));
      p.gemms.push_back(plan_gemm_tc(p.xn16, h, w.wo, h, w.bo, p.x, h, Mi, hi, hi, EPI_BIAS_RESID_F32, &m.scratch));
      p.gemms.push_back(plan_gemm_tc(p.xn16, h, w.w1, h, w.b1, p.big16, f, Mi, fi, hi, EPI_BIAS_GELU_F16, &m.scratch));
      p.gemms.push_back(plan_gemm_tc(p.big16, f, w.w2, f, w.b2, p.x, h, Mi, hi, fi, EPI_BIAS_RESID_F32, &m.scratch));
    }
    p.attn = plan_attn_tc(p.big16, 3 * h, p.xn16, h, static_cast<int>(B), static_cast<int>(S),
                          static_cast<int>(m.H), static_cast<int>(m.hd), m.d.archetype == 1);
    p.attn_work.alloc(2 * sizeof(int));
    PRLAB_CUDA(cudaMemset(p.attn_work.p, 0, 2 * sizeof(int)));
    p.attn.fa_work = static_cast<int*>(p.attn_work.p);
    if (fast16) {
      for (auto& g : p.gemms) g.acc16 = true;
      p.attn.unstab = 1;
    } else if (fwd_small_supported(M, S, h, f, m.hd, m.L)) {
      plan_small(m, p, B, S);
      if (fwd_cluster_supported(M, S, h, f, m.H, m.L)) plan_cluster(m, p, B, S);
    }
  } else {
    p.xn32 = m.ws.at<float>(at(s_a));
    p.qkv32 = m.ws.at<float>(at(s_b));
    p.ff32 = p.qkv32 + M * 3 * h;
    p.ctx32 = m.ws.at<float>(at(s_c));
  }
  auto& ref = *plan;
  m.plans[key] = std::move(plan);
  return ref;
}

// Options of one forward recording (the drop-in's retain_scores / instrumented /
// classifier variants; the default is the plain logits forward).
struct FwdOpts {
  float* tap = nullptr;      // device [L][B][H][S][S] fp32 pre-mask scores (retain_scores)
  bool hidden_only = false;  // stop after forward_hidden (classifier_probs)
  // instrumented mode: one (op class, start, end) event triple per launch
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>>* timing = nullptr;
};

// Records one forward on `st`; returns the number of kernels launched.
int64_t enqueue_forward(prlab_gpu_model& m, prlab_gpu_model::Plan& p, const int32_t* ids, void* out,
                        int out_dtype, int64_t ld, cudaStream_t st, const FwdOpts& o = FwdOpts()) {
  const int64_t B = p.B, S = p.S, M = B * S, h = m.h, f = m.f, V = m.V, L = m.L;
  const int Bi = static_cast<int>(B), Si = static_cast<int>(S), Mi = static_cast<int>(M);
  const int hi = static_cast<int>(h), fi = static_cast<int>(f), Vi = static_cast<int>(V);
  int* err = m.err.at<int>(0);
  int64_t n = 0;
  // instrumented mode: bracket each launch with events attributed to the reference op
  // class (fused kernels count for the class that produces their output; the fused
  // attention kernel for AttentionScoreMatmul)
  auto T = [&](int cls, auto&& launch) {
    if (o.timing) {
      cudaEvent_t a, b;
      PRLAB_CUDA(cudaEventCreate(&a));
      PRLAB_CUDA(cudaEventCreate(&b));
      PRLAB_CUDA(cudaEventRecord(a, st));
      launch();
      PRLAB_CUDA(cudaEventRecord(b, st));
      o.timing->emplace_back(cls, a, b);
    } else {
      launch();
    }
    ++n;
  };
  const int64_t tap_stride = B * m.H * S * S;
  if (p.fast && p.small && !o.tap && !o.timing) {
    // batch-1 shapes: embed .. final LN as one cooperative kernel (fwd_small.cu)
    if (p.cluster) {
      FwdClusterPlan cp = p.cp;
      cp.ids = ids;
      launch_fwd_cluster(cp, st);
    } else {
      FwdSmallPlan sp = p.sp;
      sp.ids = ids;
      launch_fwd_small(sp, st);
    }
    n += 1;
  } else if (p.fast) {
    float* xr = p.fp16 ? p.x : nullptr;  // full_fp16: LN rounds the residual stream in place first
    if (p.fp16)  // embed with every operand conformed to binary16 (kernels.cpp:256-294, F16E)
      T(PRLAB_EMBEDDING, [&] { simt_embed(m.tok, V, m.pos, hi, ids, Bi, Si, Kcfg{1, 1, 0}, p.x, err, st); });
    else
      T(PRLAB_EMBEDDING, [&] { embed_f32(m.tok, V, m.pos, hi, ids, Bi, Si, p.x, err, st); });
    for (int64_t l = 0; l < L; ++l) {
      const auto& w = m.l16[l];
      float* tap = o.tap ? o.tap + l * tap_stride : nullptr;
      T(PRLAB_LAYERNORM, [&] { ln_f32_to_f16(p.x, Mi, hi, w.ln1g, w.ln1b, 1e-5f, p.xn16, st, xr); });  // LN1
      T(PRLAB_LINEAR, [&] { launch_gemm_tc(p.gemms[4 * l + 0], st); });                          // QKV (+bias)
      T(PRLAB_ATTENTION_SCORE_MATMUL, [&] { launch_attn_tc(p.attn, st, tap); });                // -> ctx (xn16)
      T(PRLAB_LINEAR, [&] { launch_gemm_tc(p.gemms[4 * l + 1], st); });                          // Wo + residual
      T(PRLAB_LAYERNORM, [&] { ln_f32_to_f16(p.x, Mi, hi, w.ln2g, w.ln2b, 1e-5f, p.xn16, st, xr); });  // LN2
      T(PRLAB_LINEAR, [&] { launch_gemm_tc(p.gemms[4 * l + 2], st); });                          // FFN1 + GELU
      T(PRLAB_LINEAR, [&] { launch_gemm_tc(p.gemms[4 * l + 3], st); });                          // FFN2 + residual
    }
    T(PRLAB_LAYERNORM, [&] { ln_f32_to_f16(p.x, Mi, hi, m.lnfg, m.lnfb, 1e-5f, p.xn16, st, xr); });
  }
  if (p.fast) {
    if (o.hidden_only) return n;  // forward_hidden: r16(final LN) in xn16 (the Linear lattice)
    if (out_dtype == PRLAB_OUT_F16) {
      if (ld % 8 != 0) throw std::invalid_argument("fp16 logits need a row pitch that is a multiple of 8");
      const auto key = std::make_tuple(out, ld, static_cast<int>(EPI_F16));
      auto it = p.head_plans.find(key);
      if (it == p.head_plans.end())
        it = p.head_plans.emplace(key, plan_gemm_tc(p.xn16, h, m.emb16, h, nullptr, out, ld, Mi, Vi, hi, EPI_F16, &m.scratch)).first;
      it->second.acc16 = p.fp16;
      T(PRLAB_LINEAR, [&] { launch_gemm_tc(it->second, st); });  // tied head straight into the caller's buffer
    } else {
      // fp32 logits straight from the head's epilogue (the widened binary16 values; TMA
      // store when the rows are 16-byte aligned), no fp16 staging buffer
      const auto key = std::make_tuple(out, ld, static_cast<int>(EPI_F16_F32));
      auto it = p.head_plans.find(key);
      if (it == p.head_plans.end())
        it = p.head_plans.emplace(key, plan_gemm_tc(p.xn16, h, m.emb16, h, nullptr, out, ld, Mi, Vi, hi, EPI_F16_F32, &m.scratch)).first;
      it->second.acc16 = p.fp16;
      T(PRLAB_LINEAR, [&] { launch_gemm_tc(it->second, st); });
    }
    return n;
  }

  // ---------------- generic path (fp32 storage, per-class configs) ----------------
  const prlab_policy& pol = p.pol;
  const Kcfg lin = K(pol.cls[PRLAB_LINEAR]), att = K(pol.cls[PRLAB_ATTENTION_SCORE_MATMUL]),
             sm = K(pol.cls[PRLAB_SOFTMAX]), ln = K(pol.cls[PRLAB_LAYERNORM]),
             act = K(pol.cls[PRLAB_ACTIVATION]), emb = K(pol.cls[PRLAB_EMBEDDING]),
             res = K(pol.cls[PRLAB_RESIDUAL]);
  T(PRLAB_EMBEDDING, [&] { simt_embed(m.tok, V, m.pos, hi, ids, Bi, Si, emb, p.x, err, st); });
  const float scale = 1.0f / std::sqrt(static_cast<float>(m.hd));
  // plain-fp32 linears on the tensor cores (3xTF32, gemm_tf32.cu) when the residues exist
  const bool tc32 = m.have32lo && tf32_policy(pol) && !std::getenv("PRLAB_NO_TF32X3");
  auto lin_gemm = [&](const float* A, int64_t lda, const float* W, const float* Wlo, int64_t ldw, float* out,
                      int64_t ldo, int Mi_, int Ni_, int Ki_, const float* bias, int op, const float* resid) {
    if (tc32 && Wlo != nullptr && gemm_tf32_ok(A, lda, W, ldw, Ki_))
      gemm_tf32(A, lda, W, Wlo, ldw, out, ldo, Mi_, Ni_, Ki_, bias, op, resid, m.scratch.ws, m.scratch.ws_floats, st);
    else
      simt_gemm(A, lda, W, ldw, out, ldo, Mi_, Ni_, Ki_, lin, SimtGemmEpi{bias, op, act, res, resid}, st);
  };
  for (int64_t l = 0; l < L; ++l) {
    const auto& w16 = m.l16[l];
    const auto& w = m.l32[l];
    const auto* wl = tc32 ? &m.l32lo[l] : nullptr;
    float* tap = o.tap ? o.tap + l * tap_stride : nullptr;
    T(PRLAB_LAYERNORM, [&] { simt_layernorm(p.x, Mi, hi, w16.ln1g, w16.ln1b, 1e-5f, ln, p.xn32, nullptr, 0, st); });
    T(PRLAB_LINEAR, [&] {
      lin_gemm(p.xn32, h, w.wqkv_t, wl ? wl->wqkv : nullptr, h, p.qkv32, 3 * h, Mi, 3 * hi, hi, w.bqkv, 0, nullptr);
    });
    T(PRLAB_ATTENTION_SCORE_MATMUL, [&] {
      simt_attention(p.qkv32, p.qkv32 + h, p.qkv32 + 2 * h, 3 * h, p.ctx32, h, Bi, Si, static_cast<int>(m.H),
                     static_cast<int>(m.hd), scale, m.d.archetype == 1, att, sm, tap, st);
    });
    T(PRLAB_LINEAR, [&] { lin_gemm(p.ctx32, h, w.wo_t, wl ? wl->wo : nullptr, h, p.x, h, Mi, hi, hi, w.bo, 2, p.x); });
    T(PRLAB_LAYERNORM, [&] { simt_layernorm(p.x, Mi, hi, w16.ln2g, w16.ln2b, 1e-5f, ln, p.xn32, nullptr, 0, st); });
    T(PRLAB_LINEAR, [&] { lin_gemm(p.xn32, h, w.w1_t, wl ? wl->w1 : nullptr, h, p.ff32, f, Mi, fi, hi, w.b1, 1, nullptr); });
    T(PRLAB_LINEAR, [&] { lin_gemm(p.ff32, f, w.w2_t, wl ? wl->w2 : nullptr, f, p.x, h, Mi, hi, fi, w.b2, 2, p.x); });
  }
  if (o.hidden_only) {
    // forward_hidden: zero layers -> the embeddings (p.x), else the final LN in xn32
    if (L > 0) T(PRLAB_LAYERNORM, [&] { simt_layernorm(p.x, Mi, hi, m.lnfg, m.lnfb, 1e-5f, ln, p.xn32, nullptr, 0, st); });
    return n;
  }
  if (out_dtype != PRLAB_OUT_F32)
    throw std::invalid_argument("fp16 logits are only produced by the hybrid tensor-core path");
  float* dst = static_cast<float*>(out);
  if (L == 0) {
    // zero-layer model: the embeddings are the output (model.cpp:461-467)
    PRLAB_CUDA(cudaMemcpy2DAsync(dst, ld * 4, p.x, h * 4, h * 4, M, cudaMemcpyDeviceToDevice, st));
    ++n;
  } else {
    T(PRLAB_LAYERNORM, [&] { simt_layernorm(p.x, Mi, hi, m.lnfg, m.lnfb, 1e-5f, ln, p.xn32, nullptr, 0, st); });
    // tied head: logits = hidden . E^T, E [V, h] is already K-major (model.cpp:469-480)
    T(PRLAB_LINEAR, [&] { lin_gemm(p.xn32, h, m.tok, tc32 ? m.tok_lo : nullptr, h, dst, ld, Mi, Vi, hi, nullptr, 0, nullptr); });
  }
  return n;
}

void fill_calls(const prlab_gpu_model& m, int64_t B, const prlab_policy& pol, prlab_trace* tr) {
  // Same per-(class, dtype) counts as the reference's timed() wrappers (model.cpp:55-62).
  std::memset(tr, 0, sizeof(*tr));
  auto add = [&](int cls, uint64_t n) { tr->kernel_calls[cls][pol.cls[cls].compute] += n; };
  add(PRLAB_EMBEDDING, 1);
  const uint64_t L = static_cast<uint64_t>(m.L), BH = static_cast<uint64_t>(B * m.H);
  add(PRLAB_LAYERNORM, 2 * L + (L > 0 ? 1 : 0));
  add(PRLAB_LINEAR, 6 * L + (L > 0 ? 1 : 0));
  add(PRLAB_ATTENTION_SCORE_MATMUL, 2 * BH * L);
  add(PRLAB_SOFTMAX, BH * L);
  add(PRLAB_ACTIVATION, L);
  add(PRLAB_RESIDUAL, 2 * L);
}

void check_forward_args(const prlab_gpu_model& m, int64_t B, int64_t S) {
  // forward_hidden validation, src/model.cpp:355-362 (same messages)
  if (B < 1 || S < 1) throw std::invalid_argument("forward needs a non-empty token batch");
  if (S > m.P)
    throw std::invalid_argument("sequence length " + std::to_string(S) + " exceeds max_positions " +
                                std::to_string(m.P));
}

// Enqueue one forward on `st`, replaying a cached CUDA graph when requested.
void run_forward(prlab_gpu_model& m, prlab_gpu_model::Plan& p, const int32_t* d_ids, void* d_out, int out_dtype,
                 int64_t ld, cudaStream_t st, bool use_graph) {
  if (!use_graph) {
    enqueue_forward(m, p, d_ids, d_out, out_dtype, ld, st);
    return;
  }
  const auto key = std::make_tuple(static_cast<const void*>(d_ids), d_out, out_dtype, ld);
  auto it = p.graphs.find(key);
  if (it == p.graphs.end()) {
    // buffers the recording needs are allocated before the capture (no cudaMalloc inside it)
    if (p.fast && out_dtype == PRLAB_OUT_F32) plan_logits16(p);
    // capture on a private stream so a legacy-default caller stream still works
    cudaStream_t cap;
    PRLAB_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t g;
    PRLAB_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_forward(m, p, d_ids, d_out, out_dtype, ld, cap);
    } catch (...) {
      cudaStreamEndCapture(cap, &g);
      cudaStreamDestroy(cap);
      throw;
    }
    PRLAB_CUDA(cudaStreamEndCapture(cap, &g));
    cudaGraphExec_t ge;
    PRLAB_CUDA(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    it = p.graphs.emplace(key, ge).first;
  }
  PRLAB_CUDA(cudaGraphLaunch(it->second, st));
}

struct TmpDev {
  void* p = nullptr;
  explicit TmpDev(size_t n) { PRLAB_CUDA(cudaMalloc(&p, n ? n : 4)); }
  ~TmpDev() { cudaFree(p); }
  float* f() const { return static_cast<float*>(p); }
};

}  // namespace

namespace {
template <typename Fn>
int unary(const float* x, int64_t n, prlab_kcfg cfg, float* out, Fn fn) {
  return guarded([&] {
    validate_kcfg(cfg);
    require_device();
    if (n == 0) return;
    TmpDev dx(n * 4), dout(n * 4);
    PRLAB_CUDA(cudaMemcpy(dx.p, x, n * 4, cudaMemcpyHostToDevice));
    fn(dx.f(), n, K(cfg), dout.f());
    PRLAB_CUDA(cudaMemcpy(out, dout.p, n * 4, cudaMemcpyDeviceToHost));
  });
}
}  // namespace

// ---------------------------------------------------------------------------
// host fixture generators (reference build_model / random_tokens streams)
// ---------------------------------------------------------------------------
namespace {
// std::mt19937_64 (the engine named at src/model.cpp:23 and :292)
struct Mt64 {
  uint64_t mt[312];
  int i = 312;
  explicit Mt64(uint64_t seed) {
    mt[0] = seed;
    for (int k = 1; k < 312; ++k) mt[k] = 6364136223846793005ULL * (mt[k - 1] ^ (mt[k - 1] >> 62)) + k;
  }
  uint64_t operator()() {
    if (i >= 312) {
      static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
      for (int k = 0; k < 312; ++k) {
        const uint64_t x = (mt[k] & 0xFFFFFFFF80000000ULL) | (mt[(k + 1) % 312] & 0x7FFFFFFFULL);
        mt[k] = mt[(k + 156) % 312] ^ (x >> 1) ^ mag[x & 1];
      }
      i = 0;
    }
    uint64_t x = mt[i++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
  }
};
}  // namespace

prlab_gpu_model* create_model(const prlab_model_desc& desc, const float* const* params, int64_t n_params,
                              int device) {
  validate_desc(desc);
  const auto sizes = param_sizes(desc);
  if (static_cast<size_t>(n_params) != sizes.size())
    throw std::invalid_argument("expected " + std::to_string(sizes.size()) + " parameter tensors, got " +
                                std::to_string(n_params));
  require_device();
  PRLAB_CUDA(cudaSetDevice(device));
  auto m = std::make_unique<prlab_gpu_model>();
  m->d = desc;
  m->device = device;
  m->h = desc.hidden;
  m->f = desc.ffn;
  m->H = desc.heads;
  m->hd = desc.hidden / desc.heads;
  m->V = desc.vocab;
  m->P = desc.max_positions;
  m->L = desc.num_layers;
  m->host.resize(sizes.size());
  for (size_t i = 0; i < sizes.size(); ++i) m->host[i].assign(params[i], params[i] + sizes[i]);
  upload_fast(*m);
  configure_gemm_tc();
  configure_attn_tc();
  PRLAB_CUDA(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
  PRLAB_CUDA(cudaEventCreateWithFlags(&m->last_ev, cudaEventDisableTiming));
  return m.release();
}

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* prlab_gpu_last_error(void) { return g_last_error.c_str(); }
int prlab_gpu_abi_version(void) { return PRLAB_GPU_ABI_VERSION; }

int prlab_gpu_resolve_policy(const char* name, prlab_policy* out) {
  return guarded([&] {
    // resolve_policy, src/policy.cpp:49-67
    const std::string n = name ? name : "";
    const prlab_kcfg f32{0, 0, 1}, full{1, 1, 0}, wide{1, 0, 1};
    prlab_policy p;
    if (n == "fp32") {
      for (auto& c : p.cls) c = f32;
    } else if (n == "full_fp16") {
      for (auto& c : p.cls) c = full;
    } else if (n == "hybrid") {
      for (auto& c : p.cls) c = f32;
      p.cls[PRLAB_LINEAR] = wide;
      p.cls[PRLAB_ATTENTION_SCORE_MATMUL] = wide;
      p.cls[PRLAB_ACTIVATION] = wide;
    } else {
      throw std::invalid_argument("unknown policy '" + n + "' (valid: fp32, full_fp16, hybrid)");
    }
    *out = p;
  });
}

uint64_t prlab_gpu_param_count(const prlab_model_desc* d) {
  uint64_t n = 0;
  for (size_t s : param_sizes(*d)) n += s;
  return n;
}

int prlab_gpu_build_model(const prlab_model_desc* desc, float* out, int64_t out_len) {
  return guarded([&] {
    validate_desc(*desc);
    const auto sizes = param_sizes(*desc);
    uint64_t total = 0;
    for (size_t s : sizes) total += s;
    if (static_cast<uint64_t>(out_len) != total)
      throw std::invalid_argument("build_model: output holds " + std::to_string(out_len) + " floats, need " +
                                  std::to_string(total));
    // NormalSampler (src/model.cpp:22-44): the uniform stream is sequential; the
    // Box-Muller transform of each pair is independent, so it runs on threads.
    Mt64 rng(desc->seed);
    // per tensor: 0 = matrix (normal draws), 1 = gamma (ones), 2 = zeros
    std::vector<int> kind = {0, 0};
    for (int64_t l = 0; l < desc->num_layers; ++l) {
      const int k[16] = {1, 2, 0, 2, 0, 2, 0, 2, 0, 2, 1, 2, 0, 2, 0, 2};
      kind.insert(kind.end(), k, k + 16);
    }
    kind.push_back(1);
    kind.push_back(2);
    if (desc->archetype == 0) {
      const int k[4] = {0, 2, 0, 2};
      kind.insert(kind.end(), k, k + 4);
    }
    uint64_t n_normal = 0;
    for (size_t t = 0; t < sizes.size(); ++t)
      if (kind[t] == 0) n_normal += sizes[t];
    const uint64_t pairs = (n_normal + 1) / 2;
    std::vector<uint64_t> u(2 * pairs);
    for (auto& x : u) x = rng();
    std::vector<float> normals(2 * pairs);
    const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (uint64_t i = t; i < pairs; i += nt) {
          const double u1 = (static_cast<double>(u[2 * i] >> 11) + 0.5) * 0x1.0p-53;
          const double u2 = static_cast<double>(u[2 * i + 1] >> 11) * 0x1.0p-53;
          const double r = std::sqrt(-2.0 * std::log(u1));
          const double a = 2.0 * 3.14159265358979323846 * u2;
          normals[2 * i] = static_cast<float>(r * std::cos(a) * static_cast<double>(0.02f));
          normals[2 * i + 1] = static_cast<float>(r * std::sin(a) * static_cast<double>(0.02f));
        }
      });
    for (auto& th : pool) th.join();
    float* o = out;
    uint64_t k = 0;
    for (size_t t = 0; t < sizes.size(); ++t) {
      for (size_t i = 0; i < sizes[t]; ++i) o[i] = kind[t] == 0 ? normals[k++] : (kind[t] == 1 ? 1.0f : 0.0f);
      o += sizes[t];
    }
  });
}

int prlab_gpu_random_tokens(int64_t vocab, int64_t batch, int64_t seq, uint64_t seed, int32_t* ids) {
  return guarded([&] {
    if (vocab < 1 || batch < 1 || seq < 1)
      throw std::invalid_argument("random_tokens needs vocab, batch, seq >= 1");
    Mt64 rng(seed);
    for (int64_t i = 0; i < batch * seq; ++i) ids[i] = static_cast<int32_t>(rng() % static_cast<uint64_t>(vocab));
  });
}

int prlab_gpu_argmax_device(const void* d_logits, int32_t dtype, int64_t rows, int64_t n, int64_t ld,
                            int32_t* d_tokens, void* stream) {
  return guarded([&] {
    if (dtype != PRLAB_OUT_F32 && dtype != PRLAB_OUT_F16) throw std::invalid_argument("unknown logits dtype");
    argmax_rows(d_logits, dtype, rows, n, ld, d_tokens, static_cast<cudaStream_t>(stream));
  });
}

int prlab_gpu_row_nll_device(const void* d_logits, int32_t dtype, int64_t rows, int64_t n, int64_t ld,
                              const int32_t* d_targets, double* d_nll, int32_t* d_argmax, void* stream) {
  return guarded([&] {
    if (dtype != PRLAB_OUT_F32 && dtype != PRLAB_OUT_F16) throw std::invalid_argument("unknown logits dtype");
    if (n < 1 || ld < n) throw std::invalid_argument("logits row extent / pitch");
    row_nll(d_logits, dtype, rows, n, ld, d_targets, d_nll, d_argmax, static_cast<cudaStream_t>(stream));
  });
}

int prlab_gpu_compare_logits_device(const void* d_base, int32_t base_dtype, int64_t ld_base, const void* d_cand,
                                    int32_t cand_dtype, int64_t ld_cand, int64_t rows, int64_t n, void* stream,
                                    prlab_logit_comparison* out) {
  return guarded([&] {
    for (int d : {base_dtype, cand_dtype})
      if (d != PRLAB_OUT_F32 && d != PRLAB_OUT_F16) throw std::invalid_argument("unknown logits dtype");
    if (rows < 0 || n < 0 || ld_base < n || ld_cand < n) throw std::invalid_argument("logits extents / pitches");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<double> h(static_cast<size_t>(rows * 7));
    if (rows > 0 && n > 0) {
      TmpDev part(rows * 7 * sizeof(double));
      compare_rows(d_base, base_dtype, ld_base, d_cand, cand_dtype, ld_cand, rows, n, static_cast<double*>(part.p), st);
      PRLAB_CUDA(cudaMemcpyAsync(h.data(), part.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
      PRLAB_CUDA(cudaStreamSynchronize(st));
    }
    // fold the rows in order (compare_logits, src/fidelity.cpp:11-37)
    double mx = 0.0, se = 0.0, dot = 0.0, na = 0.0, nb = 0.0;
    uint64_t fin = 0, bad = 0;
    for (int64_t r = 0; r < rows; ++r) {
      const double* q = &h[static_cast<size_t>(r * 7)];
      mx = std::max(mx, q[0]);
      se += q[1];
      dot += q[2];
      na += q[3];
      nb += q[4];
      fin += static_cast<uint64_t>(q[5]);
      bad += static_cast<uint64_t>(q[6]);
    }
    std::memset(out, 0, sizeof(*out));
    out->max_abs_error = mx;
    out->finite_pairs = fin;
    out->candidate_nonfinite = bad;
    out->nan_affected = bad > 0;
    if (fin > 0) {
      out->mean_abs_error = se / static_cast<double>(fin);
      if (na > 0.0 && nb > 0.0) {
        out->cosine = dot / (std::sqrt(na) * std::sqrt(nb));
        out->has_cosine = 1;
      }
    }
  });
}

void enqueue_nll(prlab_gpu_model& m, prlab_gpu_model::Plan& p, const int32_t* d_ids, const int32_t* d_targets,
                 double* d_nll, int32_t* d_argmax, cudaStream_t st, int32_t* fused);

int prlab_gpu_perplexity(prlab_gpu_model* m, const int32_t* tokens, int64_t n_tokens, int64_t context_len,
                         const prlab_policy* policy, double* ppl) {
  return guarded([&] {
    // validation and messages as perplexity() (src/fidelity.cpp:248-263)
    if (m->d.archetype != 1) throw std::invalid_argument("perplexity needs a decoder_only model");
    if (context_len < 2) throw std::invalid_argument("context_len must be >= 2");
    if (context_len > m->P)
      throw std::invalid_argument("context_len " + std::to_string(context_len) + " exceeds max_positions " +
                                  std::to_string(m->P));
    if (n_tokens <= context_len)
      throw std::invalid_argument("token stream of " + std::to_string(n_tokens) +
                                  " is too short for context_len " + std::to_string(context_len) +
                                  " (need context_len + 1)");
    for (int64_t i = 0; i < n_tokens; ++i)
      if (tokens[i] < 0 || tokens[i] >= m->V)
        throw std::out_of_range("token id " + std::to_string(tokens[i]) + " outside vocab of " +
                                std::to_string(m->V));
    std::lock_guard<std::mutex> lk(m->mu);
    validate_policy(*policy);
    PRLAB_CUDA(cudaSetDevice(m->device));
    cudaStream_t st = m->stream;
    StreamOrder order(*m, st);
    const int64_t V = m->V;
    // windows [off, off + len): full ones batched (bounded logits buffer), then the tail
    const int64_t nfull = n_tokens / context_len;
    const int64_t tail = n_tokens - nfull * context_len;
    double nll_sum = 0.0;
    uint64_t predicted = 0;
    auto run = [&](int64_t off, int64_t nwin, int64_t len) {
      const int64_t rows = nwin * len;
      auto& p = get_plan(*m, nwin, len, *policy);
      std::vector<int32_t> tg(static_cast<size_t>(rows));
      for (int64_t w = 0; w < nwin; ++w)
        for (int64_t t = 0; t < len; ++t)
          tg[static_cast<size_t>(w * len + t)] = t + 1 < len ? tokens[off + w * len + t + 1] : -1;
      TmpDev dtg(rows * 4), dnll(rows * sizeof(double));
      PRLAB_CUDA(cudaMemcpyAsync(p.ids, tokens + off, rows * 4, cudaMemcpyHostToDevice, st));
      PRLAB_CUDA(cudaMemcpyAsync(dtg.p, tg.data(), rows * 4, cudaMemcpyHostToDevice, st));
      // logits stay on the device; under hybrid on the tensor-core path the head's epilogue
      // reduces them to per-row statistics and they are never written (enqueue_nll)
      enqueue_nll(*m, p, p.ids, static_cast<const int32_t*>(dtg.p), static_cast<double*>(dnll.p), nullptr, st, nullptr);
      std::vector<double> h(static_cast<size_t>(rows));
      PRLAB_CUDA(cudaMemcpyAsync(h.data(), dnll.p, rows * sizeof(double), cudaMemcpyDeviceToHost, st));
      PRLAB_CUDA(cudaStreamSynchronize(st));
      for (int64_t w = 0; w < nwin; ++w) {  // window by window, positions in order
        double win = 0.0;
        for (int64_t t = 0; t + 1 < len; ++t) win += h[static_cast<size_t>(w * len + t)];
        nll_sum += win;
        predicted += static_cast<uint64_t>(len - 1);
      }
    };
    const int64_t max_rows = std::max<int64_t>(context_len, (int64_t(1) << 31) / (V * 2));  // <= 2 GB of logits
    const int64_t per_batch = std::max<int64_t>(1, std::min<int64_t>(64, max_rows / context_len));
    for (int64_t w = 0; w < nfull; w += per_batch)
      run(w * context_len, std::min(per_batch, nfull - w), context_len);
    if (tail >= 2) run(nfull * context_len, 1, tail);
    *ppl = std::exp(nll_sum / static_cast<double>(predicted));
  });
}

int prlab_gpu_model_load_checkpoint(const char* path, int device, prlab_model_desc* desc, prlab_gpu_model** out) {
  return guarded([&] {
    prlab_model_desc d{};
    const auto params = read_checkpoint(path, d);
    std::vector<const float*> ptrs;
    for (const auto& t : params) ptrs.push_back(t.data());
    *out = create_model(d, ptrs.data(), static_cast<int64_t>(ptrs.size()), device);
    if (desc) *desc = d;
  });
}

int prlab_gpu_validate_policy(const prlab_policy* p) {
  return guarded([&] { validate_policy(*p); });
}

int prlab_gpu_model_create(const prlab_model_desc* desc, const float* const* params, int64_t n_params,
                           int device, prlab_gpu_model** out) {
  return guarded([&] { *out = create_model(*desc, params, n_params, device); });
}

int prlab_gpu_model_create_flat(const prlab_model_desc* desc, const float* flat, int device,
                                prlab_gpu_model** out) {
  return guarded([&] {
    validate_desc(*desc);
    const auto sizes = param_sizes(*desc);
    std::vector<const float*> ptrs;
    const float* p = flat;
    for (size_t s : sizes) {
      ptrs.push_back(p);
      p += s;
    }
    *out = create_model(*desc, ptrs.data(), static_cast<int64_t>(ptrs.size()), device);
  });
}

void prlab_gpu_model_destroy(prlab_gpu_model* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  delete m;
}

int prlab_gpu_model_memory(const prlab_gpu_model* m, uint64_t* weight_bytes, uint64_t* workspace_bytes) {
  return guarded([&] {
    if (weight_bytes) *weight_bytes = m->arena16.bytes + m->arena32.bytes;
    if (workspace_bytes) *workspace_bytes = m->ws.bytes;
  });
}

int prlab_gpu_model_memory_ex(prlab_gpu_model* m, prlab_memory_report* r) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(m->mu);
    std::memset(r, 0, sizeof(*r));
    r->weights_fast = m->arena16.bytes;
    r->weights_fp32 = m->arena32.bytes + m->cls_arena.bytes;
    r->weights_fast += m->cl_stream.bytes;  // the batch-1 cluster kernel's re-tiled fp16 linears
    r->workspace = m->ws.bytes;
    r->scratch = m->split_ws.bytes + m->split_tickets.bytes + m->err.bytes;
    for (const auto& kv : m->plans) {
      const auto& p = *kv.second;
      r->logits += p.lazy16.bytes + p.lazy32.bytes;
      r->scratch += p.small_buf.bytes + p.rs_buf.bytes;
    }
    r->total = r->weights_fast + r->weights_fp32 + r->workspace + r->logits + r->scratch;
  });
}

// Overlapped host forward (hybrid, logits widened on the host, calibrated plan): returns false
// (nothing done) when the call must take the serial path below.  Phase 1 under the model lock:
// ids H2D + forward into slot s's device logits on the compute stream; phase 2 outside it: the
// slot's copy-out (chunked fp16 D2H + host widening, host_widen.cpp) on the slot's stream.
bool forward_overlapped(prlab_gpu_model* m, const int32_t* ids, int64_t B, int64_t S, const prlab_policy* policy,
                        float* logits, prlab_trace* trace) {
  if (std::getenv("PRLAB_NO_HOST_OVERLAP") || std::getenv("PRLAB_NO_HOST_WIDEN") || std::getenv("PRLAB_HOST_COPY"))
    return false;
  std::unique_lock<std::mutex> lk(m->mu);
  validate_policy(*policy);
  check_forward_args(*m, B, S);
  if (m->L == 0) return false;
  auto it = m->plans.find(std::make_tuple(B, S, policy_key(*policy)));
  if (it == m->plans.end() || !it->second->fast || it->second->copy_mode != 1) return false;
  auto& p = *it->second;
  const size_t bytes = static_cast<size_t>(B * S * p.ld16) * 2;
  if (bytes > (static_cast<size_t>(512) << 20)) return false;  // C4-sized logits: one buffer, serial path
  for (int64_t i = 0; i < B * S; ++i)  // embed(), src/kernels.cpp:278-283
    if (ids[i] < 0 || ids[i] >= m->V)
      throw std::out_of_range("token id " + std::to_string(ids[i]) + " outside vocab of " + std::to_string(m->V));
  PRLAB_CUDA(cudaSetDevice(m->device));
  auto& hs = m->hslot[m->hslot_next++ & 1];
  // waits only for this slot's previous copy-out (which never takes the model lock)
  std::unique_lock<std::mutex> sl(hs.mu);
  if (!hs.cs) {
    PRLAB_CUDA(cudaStreamCreateWithFlags(&hs.cs, cudaStreamNonBlocking));
    PRLAB_CUDA(cudaEventCreateWithFlags(&hs.ready, cudaEventDisableTiming));
  }
  if (hs.buf.bytes < bytes) hs.buf.alloc(bytes);  // the slot's last copy-out completed
  __half* dlog = static_cast<__half*>(hs.buf.p);
  const int64_t w = m->V, ld16 = p.ld16;
  const bool graph = !std::getenv("PRLAB_NO_GRAPH");
  {
    cudaStream_t st = m->stream;
    StreamOrder order(*m, st);
    PRLAB_CUDA(cudaMemcpyAsync(p.ids, ids, B * S * 4, cudaMemcpyHostToDevice, st));
    run_forward(*m, p, p.ids, dlog, PRLAB_OUT_F16, ld16, st, graph);
    PRLAB_CUDA(cudaEventRecord(hs.ready, st));
  }
  if (trace) fill_calls(*m, B, *policy, trace);
  lk.unlock();
  PRLAB_CUDA(cudaStreamWaitEvent(hs.cs, hs.ready, 0));
  d2h_widen_f16(dlog, ld16, logits, w, B * S, w, hs.cs);
  return true;
}

int prlab_gpu_forward(prlab_gpu_model* m, const int32_t* ids, int64_t B, int64_t S,
                      const prlab_policy* policy, float* logits, prlab_trace* trace) {
  return guarded([&] {
    if (forward_overlapped(m, ids, B, S, policy, logits, trace)) return;
    std::lock_guard<std::mutex> lk(m->mu);
    validate_policy(*policy);
    check_forward_args(*m, B, S);
    for (int64_t i = 0; i < B * S; ++i)  // embed(), src/kernels.cpp:278-283
      if (ids[i] < 0 || ids[i] >= m->V)
        throw std::out_of_range("token id " + std::to_string(ids[i]) + " outside vocab of " +
                                std::to_string(m->V));
    PRLAB_CUDA(cudaSetDevice(m->device));
    auto& p = get_plan(*m, B, S, *policy);
    const int64_t w = m->L > 0 ? m->V : m->h;
    cudaStream_t st = m->stream;
    StreamOrder order(*m, st);
    PRLAB_CUDA(cudaMemcpyAsync(p.ids, ids, B * S * 4, cudaMemcpyHostToDevice, st));
    const bool graph = !std::getenv("PRLAB_NO_GRAPH");
    if (p.fast && m->L > 0 && !std::getenv("PRLAB_NO_HOST_WIDEN")) {
      // hybrid: the head's logits are round16'd, so the fp16 rows widened on the host are
      // the fp32 logits bit for bit -- half the PCIe bytes (host_widen.cpp), but host-thread
      // work whose speed depends on the host; the first call of a plan times both copy-outs
      // of the same logits and keeps the faster one
      run_forward(*m, p, p.ids, plan_logits16(p), PRLAB_OUT_F16, p.ld16, st, graph);
      if (const char* force = std::getenv("PRLAB_HOST_COPY"))  // "widen" / "fp32": skip the timing
        p.copy_mode = std::strcmp(force, "widen") == 0 ? 1 : 2;
      if (p.copy_mode == 0) {
        using clk = std::chrono::steady_clock;
        double t_w = 1e30, t_f = 1e30;
        for (int r = 0; r < 3; ++r) {
          const auto t0 = clk::now();
          d2h_widen_f16(p.logit16, p.ld16, logits, w, B * S, w, st);
          t_w = std::min(t_w, std::chrono::duration<double>(clk::now() - t0).count());
        }
        convert_f16_to_f32(p.logit16, p.ld16, plan_out32(p), w, static_cast<int>(B * S), static_cast<int>(w), st);
        PRLAB_CUDA(cudaStreamSynchronize(st));
        for (int r = 0; r < 3; ++r) {
          const auto t0 = clk::now();
          PRLAB_CUDA(cudaMemcpyAsync(logits, p.out32, B * S * w * 4, cudaMemcpyDeviceToHost, st));
          PRLAB_CUDA(cudaStreamSynchronize(st));
          t_f = std::min(t_f, std::chrono::duration<double>(clk::now() - t0).count());
        }
        p.copy_mode = t_w < t_f ? 1 : 2;
      } else if (p.copy_mode == 1) {
        d2h_widen_f16(p.logit16, p.ld16, logits, w, B * S, w, st);
      } else {
        convert_f16_to_f32(p.logit16, p.ld16, plan_out32(p), w, static_cast<int>(B * S), static_cast<int>(w), st);
        PRLAB_CUDA(cudaMemcpyAsync(logits, p.out32, B * S * w * 4, cudaMemcpyDeviceToHost, st));
        PRLAB_CUDA(cudaStreamSynchronize(st));
      }
    } else {
      run_forward(*m, p, p.ids, plan_out32(p), PRLAB_OUT_F32, w, st, graph);
      PRLAB_CUDA(cudaMemcpyAsync(logits, p.out32, B * S * w * 4, cudaMemcpyDeviceToHost, st));
      PRLAB_CUDA(cudaStreamSynchronize(st));
    }
    if (trace) fill_calls(*m, B, *policy, trace);
  });
}

int prlab_gpu_forward_ex(prlab_gpu_model* m, const int32_t* ids, int64_t B, int64_t S,
                         const prlab_policy* policy, int32_t flags, float* logits, prlab_trace* trace,
                         float* scores) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(m->mu);
    validate_policy(*policy);
    check_forward_args(*m, B, S);
    for (int64_t i = 0; i < B * S; ++i)  // embed(), src/kernels.cpp:278-283
      if (ids[i] < 0 || ids[i] >= m->V)
        throw std::out_of_range("token id " + std::to_string(ids[i]) + " outside vocab of " +
                                std::to_string(m->V));
    const bool retain = (flags & PRLAB_FWD_RETAIN_SCORES) != 0, timed = (flags & PRLAB_FWD_TIMED) != 0;
    if (retain && scores == nullptr) throw std::invalid_argument("retain_scores needs a scores buffer");
    PRLAB_CUDA(cudaSetDevice(m->device));
    auto& p = get_plan(*m, B, S, *policy, retain);  // the score tap needs the exact (stabilised-order) kernels
    const int64_t w = m->L > 0 ? m->V : m->h;
    cudaStream_t st = m->stream;
    StreamOrder order(*m, st);
    PRLAB_CUDA(cudaMemcpyAsync(p.ids, ids, B * S * 4, cudaMemcpyHostToDevice, st));
    FwdOpts o;
    const int64_t tap_n = m->L * B * m->H * S * S;
    TmpDev tap(retain ? static_cast<size_t>(tap_n) * 4 : 0);
    if (retain) o.tap = tap.f();
    std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> ev;
    if (timed) o.timing = &ev;
    plan_out32(p);
    if (!retain && !timed)
      run_forward(*m, p, p.ids, p.out32, PRLAB_OUT_F32, w, st, !std::getenv("PRLAB_NO_GRAPH"));
    else
      enqueue_forward(*m, p, p.ids, p.out32, PRLAB_OUT_F32, w, st, o);
    PRLAB_CUDA(cudaMemcpyAsync(logits, p.out32, B * S * w * 4, cudaMemcpyDeviceToHost, st));
    if (retain) PRLAB_CUDA(cudaMemcpyAsync(scores, tap.p, tap_n * 4, cudaMemcpyDeviceToHost, st));
    PRLAB_CUDA(cudaStreamSynchronize(st));
    if (trace) {
      fill_calls(*m, B, *policy, trace);
      for (auto& e : ev) {
        float ms = 0.0f;
        PRLAB_CUDA(cudaEventElapsedTime(&ms, std::get<1>(e), std::get<2>(e)));
        trace->seconds[std::get<0>(e)] += 1e-3 * ms;
      }
    }
    for (auto& e : ev) {
      cudaEventDestroy(std::get<1>(e));
      cudaEventDestroy(std::get<2>(e));
    }
  });
}

int prlab_gpu_classifier_probs(prlab_gpu_model* m, const int32_t* ids, int64_t B, int64_t S,
                               const prlab_policy* policy, float* probs) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(m->mu);
    if (m->d.archetype != 0) throw std::invalid_argument("classifier_probs needs an encoder_only model");
    validate_policy(*policy);
    check_forward_args(*m, B, S);
    for (int64_t i = 0; i < B * S; ++i)
      if (ids[i] < 0 || ids[i] >= m->V)
        throw std::out_of_range("token id " + std::to_string(ids[i]) + " outside vocab of " +
                                std::to_string(m->V));
    PRLAB_CUDA(cudaSetDevice(m->device));
    const int64_t h = m->h;
    if (m->pool_wt == nullptr) {
      // canonical order: ..., final_ln.{gamma,beta}, pooler.{weight [h,h], bias}, classifier.{weight [h,2], bias}
      const size_t base = 2 + 16 * static_cast<size_t>(m->L) + 2;
      const auto& pw = m->host[base];
      const auto& pb = m->host[base + 1];
      const auto& cw = m->host[base + 2];
      const auto& cb = m->host[base + 3];
      std::vector<float> buf(static_cast<size_t>(h * h + h + 2 * h + 2));
      for (int64_t r = 0; r < h; ++r)
        for (int64_t c = 0; c < h; ++c) buf[c * h + r] = pw[r * h + c];  // W^T [out, in]
      std::copy(pb.begin(), pb.end(), buf.begin() + h * h);
      for (int64_t r = 0; r < h; ++r)
        for (int64_t c = 0; c < 2; ++c) buf[h * h + h + c * h + r] = cw[r * 2 + c];
      std::copy(cb.begin(), cb.end(), buf.begin() + h * h + 3 * h);
      m->cls_arena.alloc(buf.size() * 4);
      h2d(m->cls_arena.p, buf.data(), buf.size());
      float* a = static_cast<float*>(m->cls_arena.p);
      m->pool_wt = a;
      m->pool_b = a + h * h;
      m->cls_wt = a + h * h + h;
      m->cls_b = a + h * h + 3 * h;
    }
    auto& p = get_plan(*m, B, S, *policy);
    cudaStream_t st = m->stream;
    StreamOrder order(*m, st);
    PRLAB_CUDA(cudaMemcpyAsync(p.ids, ids, B * S * 4, cudaMemcpyHostToDevice, st));
    FwdOpts o;
    o.hidden_only = true;
    enqueue_forward(*m, p, p.ids, nullptr, PRLAB_OUT_F32, 0, st, o);
    const Kcfg lin = K(policy->cls[PRLAB_LINEAR]), act = K(policy->cls[PRLAB_ACTIVATION]),
               sm = K(policy->cls[PRLAB_SOFTMAX]), res = K(policy->cls[PRLAB_RESIDUAL]);
    const int Bi = static_cast<int>(B), hi = static_cast<int>(h);
    TmpDev pooled(B * h * 4), pre(B * h * 4), logit(B * 2 * 4), pr(B * 2 * 4);
    const bool f16 = p.fast;  // fast path: r16(final LN) in fp16; generic: fp32 (or embeddings at L = 0)
    const float* x32 = f16 ? nullptr : (m->L > 0 ? p.xn32 : p.x);
    simt_pool_mean(x32, f16 ? p.xn16 : nullptr, Bi, static_cast<int>(S), hi, lin, pooled.f(), st);
    simt_gemm(pooled.f(), h, m->pool_wt, h, pre.f(), h, Bi, hi, hi, lin, SimtGemmEpi{m->pool_b, 0, act, res, nullptr}, st);
    simt_tanh(pre.f(), B * h, act, pre.f(), st);
    simt_gemm(pre.f(), h, m->cls_wt, h, logit.f(), 2, Bi, 2, hi, lin, SimtGemmEpi{m->cls_b, 0, act, res, nullptr}, st);
    simt_softmax(logit.f(), B, 2, sm, pr.f(), st);
    std::vector<float> host(static_cast<size_t>(2 * B));
    PRLAB_CUDA(cudaMemcpyAsync(host.data(), pr.p, B * 2 * 4, cudaMemcpyDeviceToHost, st));
    PRLAB_CUDA(cudaStreamSynchronize(st));
    for (int64_t b = 0; b < B; ++b) probs[b] = host[2 * b + 1];
  });
}

int prlab_gpu_forward_device(prlab_gpu_model* m, const int32_t* d_ids, int64_t B, int64_t S,
                             const prlab_policy* policy, void* d_out, int32_t out_dtype, int64_t ld,
                             void* stream, int32_t use_graph) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(m->mu);
    validate_policy(*policy);
    check_forward_args(*m, B, S);
    const int64_t w = m->L > 0 ? m->V : m->h;
    if (ld < w) throw std::invalid_argument("logits row pitch smaller than the logits width");
    if (out_dtype != PRLAB_OUT_F32 && out_dtype != PRLAB_OUT_F16)
      throw std::invalid_argument("unknown logits dtype");
    PRLAB_CUDA(cudaSetDevice(m->device));
    auto& p = get_plan(*m, B, S, *policy);
    StreamOrder order(*m, static_cast<cudaStream_t>(stream));
    run_forward(*m, p, d_ids, d_out, out_dtype, ld, static_cast<cudaStream_t>(stream), use_graph != 0);
  });
}

int prlab_gpu_forward_trunk_device(prlab_gpu_model* m, const int32_t* d_ids, int64_t B, int64_t S,
                                   const prlab_policy* policy, void* stream, int64_t* kernels) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(m->mu);
    validate_policy(*policy);
    check_forward_args(*m, B, S);
    PRLAB_CUDA(cudaSetDevice(m->device));
    auto& p = get_plan(*m, B, S, *policy);
    FwdOpts o;
    o.hidden_only = true;
    StreamOrder order(*m, static_cast<cudaStream_t>(stream));
    const int64_t n = enqueue_forward(*m, p, d_ids, nullptr, PRLAB_OUT_F32, 0, static_cast<cudaStream_t>(stream), o);
    if (kernels) *kernels = n;
  });
}

// Forward + per-row NLL / argmax (prlab_gpu_forward_nll_device, perplexity): the tied
// head's log-softmax statistics come out of the head GEMM's epilogue (EPI_ROWSTAT) when
// the head runs on CTA pairs; otherwise logits -> workspace -> row_nll.
void enqueue_nll(prlab_gpu_model& m, prlab_gpu_model::Plan& p, const int32_t* d_ids, const int32_t* d_targets,
                 double* d_nll, int32_t* d_argmax, cudaStream_t st, int32_t* fused) {
  const int64_t M = p.B * p.S, V = m.V;
  if (p.rs_state == 0) {
    p.rs_state = 2;
    if (p.fast && !std::getenv("PRLAB_NO_FUSED_NLL")) {
      // the head GEMM exactly as the logits path plans it, with the statistics epilogue
      // (planning only, never launched: any 16-byte-aligned device pointer serves as the output base)
      GemmPlan probe = plan_gemm_tc(p.xn16, m.h, m.emb16, m.h, nullptr, p.xn16, p.ld16, static_cast<int>(M),
                                    static_cast<int>(V), static_cast<int>(m.h), EPI_F16, &m.scratch);
      if (probe.pair) {
        const int nslots = (static_cast<int>(V) + probe.bn - 1) / probe.bn;  // one slot per n-block (gemm_tc.cu)
        p.rs_buf.alloc(static_cast<size_t>(nslots) * M * 16 + M * 4);
        p.rs_plan = plan_gemm_tc(p.xn16, m.h, m.emb16, m.h, nullptr, p.rs_buf.p, 8, static_cast<int>(M),
                                 static_cast<int>(V), static_cast<int>(m.h), EPI_ROWSTAT, &m.scratch, probe.bn);
        p.rs_plan.nslots = nslots;
        p.rs_plan.acc16 = p.fp16;
        p.rs_plan.tval =
            reinterpret_cast<float*>(static_cast<char*>(p.rs_buf.p) + static_cast<size_t>(nslots) * M * 16);
        p.rs_state = p.rs_plan.pair ? 1 : 2;
      }
    }
  }
  if (fused) *fused = p.rs_state == 1 ? 1 : 0;
  if (p.rs_state == 1) {
    FwdOpts o;
    o.hidden_only = true;  // forward_hidden: round16(final LN) in xn16
    enqueue_forward(m, p, d_ids, nullptr, PRLAB_OUT_F32, 0, st, o);
    GemmPlan hp = p.rs_plan;
    hp.targets = d_targets;
    launch_gemm_tc(hp, st);
    rowstat_combine(p.rs_buf.p, hp.nslots, M, V, d_targets, hp.tval, d_nll, d_argmax, st);
  } else if (p.fast) {  // unfused: logits into the workspace, then the row kernel
    enqueue_forward(m, p, d_ids, plan_logits16(p), PRLAB_OUT_F16, p.ld16, st);
    row_nll(p.logit16, 1, M, V, p.ld16, d_targets, d_nll, d_argmax, st);
  } else {
    enqueue_forward(m, p, d_ids, plan_out32(p), PRLAB_OUT_F32, V, st);
    row_nll(p.out32, 0, M, V, V, d_targets, d_nll, d_argmax, st);
  }
}

int prlab_gpu_forward_nll_device(prlab_gpu_model* m, const int32_t* d_ids, const int32_t* d_targets, int64_t B,
                                 int64_t S, const prlab_policy* policy, double* d_nll, int32_t* d_argmax,
                                 void* stream, int32_t* fused) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(m->mu);
    validate_policy(*policy);
    check_forward_args(*m, B, S);
    if (m->L == 0) throw std::invalid_argument("forward_nll needs a model with a tied head (num_layers > 0)");
    PRLAB_CUDA(cudaSetDevice(m->device));
    auto& p = get_plan(*m, B, S, *policy);
    StreamOrder order(*m, static_cast<cudaStream_t>(stream));
    enqueue_nll(*m, p, d_ids, d_targets, d_nll, d_argmax, static_cast<cudaStream_t>(stream), fused);
  });
}

int prlab_gpu_sync_status(prlab_gpu_model* m, void* stream) {
  return guarded([&] {
    PRLAB_CUDA(cudaSetDevice(m->device));
    PRLAB_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    int e = 0;
    PRLAB_CUDA(cudaMemcpy(&e, m->err.p, 4, cudaMemcpyDeviceToHost));
    if (e) {
      PRLAB_CUDA(cudaMemset(m->err.p, 0, 4));
      throw std::out_of_range("token id outside vocab of " + std::to_string(m->V));
    }
  });
}

int prlab_gpu_forward_kernel_count_ex(prlab_gpu_model* m, int64_t B, int64_t S, const prlab_policy* policy,
                                      int32_t out_dtype, int64_t* count) {
  return guarded([&] {
    check_forward_args(*m, B, S);
    if (out_dtype != PRLAB_OUT_F32 && out_dtype != PRLAB_OUT_F16) throw std::invalid_argument("unknown logits dtype");
    const bool fast = fast_eligible(*m, S, *policy) || fast16_eligible(*m, S, *policy, false);
    const int64_t L = m->L;
    const bool small = fast_eligible(*m, S, *policy) && fwd_small_supported(B * S, S, m->h, m->f, m->hd, L);
    // fast path: trunk (1 persistent kernel, or embed + 7 per layer + final LN) + the head GEMM
    // (fp16 or fp32 logits straight from its epilogue)
    *count = small ? 2 : (fast ? 1 + 7 * L + 1 + 1 : 1 + 7 * L + (L > 0 ? 2 : 1));
  });
}

int prlab_gpu_forward_kernel_count(prlab_gpu_model* m, int64_t B, int64_t S, const prlab_policy* policy,
                                   int64_t* count) {
  return prlab_gpu_forward_kernel_count_ex(m, B, S, policy, PRLAB_OUT_F16, count);
}

int prlab_gpu_debug_embedding_device(prlab_gpu_model* m, const int32_t* d_ids, int64_t B, int64_t S, int32_t path,
                                     float* d_out, void* stream) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(m->mu);
    check_forward_args(*m, B, S);
    prlab_policy pol;
    prlab_gpu_resolve_policy("hybrid", &pol);
    if (!fast_eligible(*m, S, pol)) throw std::invalid_argument("embedding debug: shape not on the tensor-core path");
    PRLAB_CUDA(cudaSetDevice(m->device));
    auto& p = get_plan(*m, B, S, pol);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder order(*m, st);
    if (path == 0) {
      embed_f32(m->tok, m->V, m->pos, static_cast<int>(m->h), d_ids, static_cast<int>(B), static_cast<int>(S), p.x,
                m->err.at<int>(0), st);
    } else if (path == 1) {
      if (!p.small) throw std::invalid_argument("embedding debug: shape not on the persistent batch-1 kernel");
      FwdSmallPlan sp = p.sp;
      sp.ids = d_ids;
      sp.embed_only = 1;
      launch_fwd_small(sp, st);
    } else {
      if (!p.cluster) throw std::invalid_argument("embedding debug: shape not on the cluster batch-1 kernel");
      FwdClusterPlan cp = p.cp;
      cp.ids = d_ids;
      cp.embed_only = 1;
      launch_fwd_cluster(cp, st);
      PRLAB_CUDA(cudaMemcpyAsync(d_out, cp.xg, B * S * m->h * 4, cudaMemcpyDeviceToDevice, st));
      return;
    }
    PRLAB_CUDA(cudaMemcpyAsync(d_out, p.x, B * S * m->h * 4, cudaMemcpyDeviceToDevice, st));
  });
}

int prlab_gpu_host_copy_mode(prlab_gpu_model* m, int64_t B, int64_t S, const prlab_policy* policy,
                             int32_t* mode) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(m->mu);
    check_forward_args(*m, B, S);
    auto it = m->plans.find(std::make_tuple(B, S, policy_key(*policy)));
    *mode = it == m->plans.end() ? 0 : (it->second->fast && m->L > 0 ? it->second->copy_mode : 2);
  });
}

// ---- per-operator entry points (host fp32 in/out, synchronous) ----
int prlab_gpu_matmul(const float* a, const float* b, int64_t m, int64_t k, int64_t n, prlab_kcfg cfg,
                     float* out) {
  return guarded([&] {
    validate_kcfg(cfg);
    if (m < 0 || k < 0 || n < 0) throw std::invalid_argument("negative extent in matmul");
    require_device();
    if (m == 0 || n == 0) return;
    TmpDev da(m * k * 4), db(k * n * 4), dbt(k * n * 4), dout(m * n * 4);
    PRLAB_CUDA(cudaMemcpy(da.p, a, m * k * 4, cudaMemcpyHostToDevice));
    PRLAB_CUDA(cudaMemcpy(db.p, b, k * n * 4, cudaMemcpyHostToDevice));
    transpose_f32(db.f(), static_cast<int>(k), static_cast<int>(n), dbt.f(), 0, nullptr);
    simt_gemm(da.f(), k, dbt.f(), k, dout.f(), n, static_cast<int>(m), static_cast<int>(n),
              static_cast<int>(k), K(cfg), SimtGemmEpi{nullptr, 0, K(cfg), K(cfg), nullptr}, nullptr);
    PRLAB_CUDA(cudaMemcpy(out, dout.p, m * n * 4, cudaMemcpyDeviceToHost));
  });
}

int prlab_gpu_attention_scores(const float* q, const float* k, int64_t sq, int64_t sk, int64_t d, float scale,
                               prlab_kcfg cfg, float* out, float* capture) {
  return guarded([&] {
    validate_kcfg(cfg);
    require_device();
    if (sq == 0 || sk == 0) return;
    TmpDev dq(sq * d * 4), dk(sk * d * 4), dout(sq * sk * 4), dtap(capture ? sq * sk * 4 : 4);
    PRLAB_CUDA(cudaMemcpy(dq.p, q, sq * d * 4, cudaMemcpyHostToDevice));
    PRLAB_CUDA(cudaMemcpy(dk.p, k, sk * d * 4, cudaMemcpyHostToDevice));
    simt_scores(dq.f(), dk.f(), static_cast<int>(sq), static_cast<int>(sk), static_cast<int>(d), scale, K(cfg),
                dout.f(), capture ? dtap.f() : nullptr, nullptr);
    PRLAB_CUDA(cudaMemcpy(out, dout.p, sq * sk * 4, cudaMemcpyDeviceToHost));
    if (capture) PRLAB_CUDA(cudaMemcpy(capture, dtap.p, sq * sk * 4, cudaMemcpyDeviceToHost));
  });
}

int prlab_gpu_softmax(const float* x, int64_t rows, int64_t n, prlab_kcfg cfg, float* out) {
  return guarded([&] {
    validate_kcfg(cfg);
    if (n < 1) throw std::invalid_argument("softmax needs a non-empty last axis");
    require_device();
    if (rows == 0) return;
    TmpDev dx(rows * n * 4), dout(rows * n * 4);
    PRLAB_CUDA(cudaMemcpy(dx.p, x, rows * n * 4, cudaMemcpyHostToDevice));
    simt_softmax(dx.f(), rows, n, K(cfg), dout.f(), nullptr);
    PRLAB_CUDA(cudaMemcpy(out, dout.p, rows * n * 4, cudaMemcpyDeviceToHost));
  });
}

int prlab_gpu_layernorm(const float* x, int64_t rows, int64_t n, const float* gamma, const float* beta,
                        float eps, prlab_kcfg cfg, float* out) {
  return guarded([&] {
    validate_kcfg(cfg);
    if (n < 1) throw std::invalid_argument("layernorm needs a non-empty last axis");
    require_device();
    if (rows == 0) return;
    TmpDev dx(rows * n * 4), dg(n * 4), db(n * 4), dout(rows * n * 4);
    PRLAB_CUDA(cudaMemcpy(dx.p, x, rows * n * 4, cudaMemcpyHostToDevice));
    PRLAB_CUDA(cudaMemcpy(dg.p, gamma, n * 4, cudaMemcpyHostToDevice));
    PRLAB_CUDA(cudaMemcpy(db.p, beta, n * 4, cudaMemcpyHostToDevice));
    simt_layernorm(dx.f(), static_cast<int>(rows), static_cast<int>(n), dg.f(), db.f(), eps, K(cfg), dout.f(),
                   nullptr, 0, nullptr);
    PRLAB_CUDA(cudaMemcpy(out, dout.p, rows * n * 4, cudaMemcpyDeviceToHost));
  });
}

int prlab_gpu_gelu(const float* x, int64_t n, prlab_kcfg cfg, float* out) {
  return unary(x, n, cfg, out, [](const float* a, int64_t nn, Kcfg c, float* o) { simt_gelu(a, nn, c, o, nullptr); });
}
int prlab_gpu_tanh(const float* x, int64_t n, prlab_kcfg cfg, float* out) {
  return unary(x, n, cfg, out, [](const float* a, int64_t nn, Kcfg c, float* o) { simt_tanh(a, nn, c, o, nullptr); });
}
int prlab_gpu_add(const float* a, const float* b, int64_t n, prlab_kcfg cfg, float* out) {
  return guarded([&] {
    validate_kcfg(cfg);
    require_device();
    if (n == 0) return;
    TmpDev da(n * 4), db(n * 4), dout(n * 4);
    PRLAB_CUDA(cudaMemcpy(da.p, a, n * 4, cudaMemcpyHostToDevice));
    PRLAB_CUDA(cudaMemcpy(db.p, b, n * 4, cudaMemcpyHostToDevice));
    simt_add(da.f(), db.f(), n, K(cfg), dout.f(), nullptr);
    PRLAB_CUDA(cudaMemcpy(out, dout.p, n * 4, cudaMemcpyDeviceToHost));
  });
}

int prlab_gpu_embed(const float* tok, int64_t vocab, const float* pos, int64_t npos, int64_t h,
                    const int32_t* ids, int64_t B, int64_t S, prlab_kcfg cfg, float* out) {
  return guarded([&] {
    validate_kcfg(cfg);
    // embed(), src/kernels.cpp:270-283 (same exception types and messages)
    if (S > npos)
      throw std::out_of_range("sequence length " + std::to_string(S) + " exceeds position table extent " +
                              std::to_string(npos));
    for (int64_t i = 0; i < B * S; ++i)
      if (ids[i] < 0 || ids[i] >= vocab)
        throw std::out_of_range("token id " + std::to_string(ids[i]) + " outside vocab of " + std::to_string(vocab));
    require_device();
    if (B * S == 0) return;
    TmpDev dt(vocab * h * 4), dp(npos * h * 4), di(B * S * 4), dout(B * S * h * 4);
    PRLAB_CUDA(cudaMemcpy(dt.p, tok, vocab * h * 4, cudaMemcpyHostToDevice));
    PRLAB_CUDA(cudaMemcpy(dp.p, pos, npos * h * 4, cudaMemcpyHostToDevice));
    PRLAB_CUDA(cudaMemcpy(di.p, ids, B * S * 4, cudaMemcpyHostToDevice));
    if (cfg.compute == 0 && h % 4 == 0)
      embed_f32(dt.f(), vocab, dp.f(), static_cast<int>(h), static_cast<int32_t*>(di.p), static_cast<int>(B),
                static_cast<int>(S), dout.f(), nullptr, nullptr);
    else
      simt_embed(dt.f(), vocab, dp.f(), static_cast<int>(h), static_cast<int32_t*>(di.p), static_cast<int>(B),
                 static_cast<int>(S), K(cfg), dout.f(), nullptr, nullptr);
    PRLAB_CUDA(cudaMemcpy(out, dout.p, B * S * h * 4, cudaMemcpyDeviceToHost));
  });
}

int prlab_gpu_linear_f16_device(const void* A, const void* Wt, const float* bias, void* out, int64_t M,
                                int64_t N, int64_t K_, int64_t ldo, int32_t epi, void* stream) {
  return guarded([&] {
    if (epi < 0 || epi > 5 || epi == EPI_ROWSTAT) throw std::invalid_argument("unknown epilogue");
    const GemmPlan p = plan_gemm_tc(A, K_, Wt, K_, bias, out, ldo, static_cast<int>(M), static_cast<int>(N),
                                    static_cast<int>(K_), epi, &global_split_scratch());
    launch_gemm_tc(p, static_cast<cudaStream_t>(stream));
  });
}

int prlab_gpu_linear_f16_device_ex(const void* A, const void* Wt, const float* bias, void* out, int64_t M,
                                   int64_t N, int64_t K_, int64_t ldo, int32_t epi, int32_t bn, int32_t splits,
                                   int32_t lean, void* stream) {
  return guarded([&] {
    if (epi < 0 || epi > 5) throw std::invalid_argument("unknown epilogue");
    if (bn != 0 && bn != 64 && bn != 128 && bn != 256) throw std::invalid_argument("bn must be 64, 128 or 256");
    const GemmPlan p = plan_gemm_tc(A, K_, Wt, K_, bias, out, ldo, static_cast<int>(M), static_cast<int>(N),
                                    static_cast<int>(K_), epi, &global_split_scratch(), bn, splits, lean);
    launch_gemm_tc(p, static_cast<cudaStream_t>(stream));
  });
}

int prlab_gpu_linear_f32_device(const float* A, const float* Wt, const float* bias, float* out, int64_t M, int64_t N,
                                int64_t K_, int32_t epi, const float* resid, void* stream) {
  return guarded([&] {
    if (epi < 0 || epi > 2) throw std::invalid_argument("unknown epilogue");
    if (M < 1 || N < 1 || K_ < 1) throw std::invalid_argument("empty linear");
    if (epi == 2 && resid == nullptr) throw std::invalid_argument("residual epilogue needs resid");
    if (!gemm_tf32_ok(A, K_, Wt, K_, K_)) throw std::invalid_argument("tf32 linear: K % 32 and 16-byte alignment");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TmpDev lo(static_cast<size_t>(N * K_) * 4);
    split_lo(Wt, lo.f(), N * K_, st);
    auto& sc = global_split_scratch();
    gemm_tf32(A, K_, Wt, lo.f(), K_, out, N, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K_), bias, epi,
              resid, sc.ws, sc.ws_floats, st);
    PRLAB_CUDA(cudaStreamSynchronize(st));  // the residue buffer is freed on return
  });
}

int prlab_gpu_debug_small_stamps(long long* dbg) {
  return guarded([&] { small_debug_stamps() = dbg; });
}

int prlab_gpu_debug_cluster_stamps(long long* dbg) {
  return guarded([&] { cluster_debug_stamps() = dbg; });
}

int prlab_gpu_debug_gemm_stamps(long long* dbg) {
  return guarded([&] { debug_stamps() = dbg; });
}

int prlab_gpu_attention_f16_device(const void* qkv, void* ctx, int64_t B, int64_t S, int64_t H, int64_t hd,
                                   int32_t causal, void* stream) {
  return prlab_gpu_attention_f16_device_dbg(qkv, ctx, B, S, H, hd, causal, stream, nullptr);
}

int prlab_gpu_attention_f16_device_dbg(const void* qkv, void* ctx, int64_t B, int64_t S, int64_t H, int64_t hd,
                                       int32_t causal, void* stream, long long* dbg) {
  return guarded([&] {
    AttnPlan p = plan_attn_tc(qkv, 3 * H * hd, ctx, H * hd, static_cast<int>(B), static_cast<int>(S),
                              static_cast<int>(H), static_cast<int>(hd), causal);
    p.dbg = dbg;
    // the dynamic-schedule counter: one per host thread and device (this building block's calls
    // from one thread are stream-ordered by contract; see prlab_gpu.h)
    thread_local std::map<int, int*> work;
    int dev = 0;
    PRLAB_CUDA(cudaGetDevice(&dev));
    int*& w = work[dev];
    if (w == nullptr) {
      PRLAB_CUDA(cudaMalloc(&w, 2 * sizeof(int)));
      PRLAB_CUDA(cudaMemset(w, 0, 2 * sizeof(int)));
    }
    p.fa_work = w;
    launch_attn_tc(p, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
