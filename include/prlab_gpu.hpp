// prlab_gpu.hpp -- C++ drop-in over the C-ABI (include/prlab_gpu.h).
//
// Mirrors the reference API (include/prlab/{kernels,model,policy}.hpp) with the
// same names, argument meaning and exception types/messages, so code written
// against `prlab::` can switch to `prlab::gpu::`:
//
//   prlab::forward(model, tokens, policy)         -> prlab::gpu::forward(model, tokens, policy)
//   prlab::matmul(a, b, cfg) / softmax_lastdim... -> prlab::gpu::matmul(a, b, cfg) / ...
//
// The header is templated on the reference's own value types (Model, Tensor,
// TokenBatch, PrecisionPolicy, KernelConfig) and only touches their public
// fields (model.hpp:21-125, tensor.hpp:32-52, kernels.hpp:16-22), so it does not
// include -- or copy -- any reference header; include it after them.
//
// Model upload is cached per Model object: the first forward uploads the
// parameters (Model::for_each_param order, model.cpp:178-209) into the device
// arena; the Model is immutable after construction.
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "prlab_gpu.h"

namespace prlab {
namespace gpu {

inline void check(int rc) {
  if (rc == PRLAB_OK) return;
  const std::string msg = prlab_gpu_last_error();
  if (rc == PRLAB_EINVAL) throw std::invalid_argument(msg);
  if (rc == PRLAB_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);  // PRLAB_ERUNTIME, PRLAB_ECUDA
}

template <class KernelConfig>
prlab_kcfg to_c(const KernelConfig& c) {
  return prlab_kcfg{static_cast<int32_t>(c.compute_dtype), static_cast<int32_t>(c.accum_dtype),
                    c.softmax_stabilized ? 1 : 0};
}

template <class PrecisionPolicy>
prlab_policy to_c_policy(const PrecisionPolicy& p) {
  prlab_policy out;
  for (int i = 0; i < PRLAB_NUM_OP_CLASSES; ++i) out.cls[i] = to_c(p.assignment[static_cast<size_t>(i)]);
  return out;
}

// RAII device model (the arena planner of the C-ABI behind it).
class DeviceModel {
 public:
  template <class Model>
  explicit DeviceModel(const Model& m, int device = 0) {
    prlab_model_desc d{};
    d.archetype = static_cast<int32_t>(m.config.archetype);
    d.num_layers = m.config.num_layers;
    d.hidden = m.config.hidden;
    d.heads = m.config.heads;
    d.ffn = m.config.ffn;
    d.vocab = m.config.vocab;
    d.max_positions = m.config.max_positions;
    d.seed = m.config.seed;
    std::vector<const float*> ptrs;
    m.for_each_param([&ptrs](const std::string&, const auto& t) { ptrs.push_back(t.data.data()); });
    prlab_gpu_model* h = nullptr;
    check(prlab_gpu_model_create(&d, ptrs.data(), static_cast<int64_t>(ptrs.size()), device, &h));
    handle_.reset(h);
    vocab_ = d.vocab;
    hidden_ = d.hidden;
    layers_ = d.num_layers;
  }
  prlab_gpu_model* get() const { return handle_.get(); }
  int64_t vocab() const { return vocab_; }
  int64_t hidden() const { return hidden_; }
  int64_t layers() const { return layers_; }

 private:
  struct Del {
    void operator()(prlab_gpu_model* m) const { prlab_gpu_model_destroy(m); }
  };
  std::unique_ptr<prlab_gpu_model, Del> handle_;
  int64_t vocab_ = 0, hidden_ = 0, layers_ = 0;
};

// Upload cache keyed by the Model's address (models are immutable once built).
template <class Model>
DeviceModel& device_model_for(const Model& m, int device = 0) {
  static std::mutex mu;
  static std::map<const void*, std::unique_ptr<DeviceModel>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto& slot = cache[static_cast<const void*>(&m)];
  if (!slot) slot = std::make_unique<DeviceModel>(m, device);
  return *slot;
}

// prlab::forward (model.cpp:456-482): same signature, same ForwardTrace fields
// (logits [B,S,V] fp32 storage; kernel_calls per class/dtype; seconds per class from
// CUDA events like the reference's timed() wrappers; layer_scores when retained).
// Filling `seconds` per op class times every kernel separately, so this path does not run the
// fused batch-1 trunk: latency / throughput callers (bench.cpp's benchmark_forward) should use
// forward_untimed below, which runs the captured fast path (and overlaps concurrent callers).
template <class Model, class TokenBatch, class PrecisionPolicy>
auto forward(const Model& model, const TokenBatch& tokens, const PrecisionPolicy& policy,
             bool retain_scores = false) {
  DeviceModel& dm = device_model_for(model);
  const prlab_policy pol = to_c_policy(policy);
  decltype(prlab::forward(model, tokens, policy)) trace;  // the reference's ForwardTrace type
  const int64_t w = dm.layers() > 0 ? dm.vocab() : dm.hidden();
  trace.logits.shape = {tokens.batch, tokens.seq, w};
  trace.logits.data.resize(static_cast<size_t>(tokens.batch * tokens.seq * w));
  prlab_trace tr{};
  const int64_t heads = model.config.heads, S = tokens.seq, B = tokens.batch;
  std::vector<float> scores;
  if (retain_scores) scores.resize(static_cast<size_t>(dm.layers() * B * heads * S * S));
  check(prlab_gpu_forward_ex(dm.get(), tokens.ids.data(), B, S, &pol,
                             PRLAB_FWD_TIMED | (retain_scores ? PRLAB_FWD_RETAIN_SCORES : 0),
                             trace.logits.data.data(), &tr, retain_scores ? scores.data() : nullptr));
  for (int c = 0; c < PRLAB_NUM_OP_CLASSES; ++c) {
    trace.seconds[static_cast<size_t>(c)] = tr.seconds[c];
    for (int d = 0; d < 2; ++d) trace.kernel_calls[static_cast<size_t>(c)][static_cast<size_t>(d)] = tr.kernel_calls[c][d];
  }
  if (retain_scores) {
    const size_t per = static_cast<size_t>(B * heads * S * S);
    for (int64_t l = 0; l < dm.layers(); ++l) {
      decltype(trace.logits) t({B, heads, S, S});
      std::copy(scores.begin() + l * per, scores.begin() + (l + 1) * per, t.data.begin());
      trace.layer_scores.push_back(std::move(t));
    }
  }
  return trace;
}

// forward() without the per-class timing: the same logits (ForwardTrace::kernel_calls filled,
// seconds left zero), through the fused / graph-captured fast path -- what a latency or
// throughput caller wants.  Safe from several threads on one model (prlab_gpu_forward).
template <class Model, class TokenBatch, class PrecisionPolicy>
auto forward_untimed(const Model& model, const TokenBatch& tokens, const PrecisionPolicy& policy) {
  DeviceModel& dm = device_model_for(model);
  const prlab_policy pol = to_c_policy(policy);
  decltype(prlab::forward(model, tokens, policy)) trace;
  const int64_t w = dm.layers() > 0 ? dm.vocab() : dm.hidden();
  trace.logits.shape = {tokens.batch, tokens.seq, w};
  trace.logits.data.resize(static_cast<size_t>(tokens.batch * tokens.seq * w));
  prlab_trace tr{};
  check(prlab_gpu_forward(dm.get(), tokens.ids.data(), tokens.batch, tokens.seq, &pol, trace.logits.data.data(), &tr));
  for (int c = 0; c < PRLAB_NUM_OP_CLASSES; ++c)
    for (int d = 0; d < 2; ++d) trace.kernel_calls[static_cast<size_t>(c)][static_cast<size_t>(d)] = tr.kernel_calls[c][d];
  return trace;
}

// prlab::classifier_probs (model.cpp:484-526): positive-class probability per batch row.
template <class Model, class TokenBatch, class PrecisionPolicy>
std::vector<float> classifier_probs(const Model& model, const TokenBatch& tokens, const PrecisionPolicy& policy) {
  DeviceModel& dm = device_model_for(model);
  const prlab_policy pol = to_c_policy(policy);
  std::vector<float> out(static_cast<size_t>(tokens.batch));
  check(prlab_gpu_classifier_probs(dm.get(), tokens.ids.data(), tokens.batch, tokens.seq, &pol, out.data()));
  return out;
}

// ---- per-operator mirrors of include/prlab/kernels.hpp:30-70 ----
template <class Tensor, class KernelConfig>
Tensor matmul(const Tensor& a, const Tensor& b, const KernelConfig& cfg) {
  if (a.rank() != 2 || b.rank() != 2)
    throw std::invalid_argument("matmul operands must be 2-D");
  if (a.shape[1] != b.shape[0]) throw std::invalid_argument("matmul inner extents differ");
  Tensor out({a.shape[0], b.shape[1]}, cfg.compute_dtype);
  check(prlab_gpu_matmul(a.data.data(), b.data.data(), a.shape[0], a.shape[1], b.shape[1], to_c(cfg),
                         out.data.data()));
  return out;
}

template <class Tensor, class KernelConfig>
Tensor softmax_lastdim(const Tensor& x, const KernelConfig& cfg) {
  if (x.rank() == 0 || x.shape.back() == 0)
    throw std::invalid_argument("softmax needs a non-empty last axis");
  Tensor out(x.shape, cfg.compute_dtype);
  const int64_t n = x.shape.back();
  check(prlab_gpu_softmax(x.data.data(), x.numel() / n, n, to_c(cfg), out.data.data()));
  return out;
}

template <class Tensor, class KernelConfig>
Tensor layernorm_lastdim(const Tensor& x, const Tensor& gamma, const Tensor& beta, float eps,
                         const KernelConfig& cfg) {
  if (x.rank() == 0 || x.shape.back() == 0)
    throw std::invalid_argument("layernorm needs a non-empty last axis");
  Tensor out(x.shape, cfg.compute_dtype);
  const int64_t n = x.shape.back();
  check(prlab_gpu_layernorm(x.data.data(), x.numel() / n, n, gamma.data.data(), beta.data.data(), eps,
                            to_c(cfg), out.data.data()));
  return out;
}

template <class Tensor, class KernelConfig>
Tensor gelu(const Tensor& x, const KernelConfig& cfg) {
  Tensor out(x.shape, cfg.compute_dtype);
  check(prlab_gpu_gelu(x.data.data(), x.numel(), to_c(cfg), out.data.data()));
  return out;
}

template <class Tensor, class KernelConfig>
Tensor add(const Tensor& a, const Tensor& b, const KernelConfig& cfg) {
  if (a.shape != b.shape) throw std::invalid_argument("add shapes differ");
  Tensor out(a.shape, cfg.compute_dtype);
  check(prlab_gpu_add(a.data.data(), b.data.data(), a.numel(), to_c(cfg), out.data.data()));
  return out;
}

template <class Tensor, class KernelConfig>
Tensor attention_scores(const Tensor& q, const Tensor& k, float scale, const KernelConfig& cfg,
                        float* capture_f32 = nullptr) {
  if (q.shape[1] != k.shape[1]) throw std::invalid_argument("attention head extents differ");
  Tensor out({q.shape[0], k.shape[0]}, cfg.compute_dtype);
  check(prlab_gpu_attention_scores(q.data.data(), k.data.data(), q.shape[0], k.shape[0], q.shape[1], scale,
                                   to_c(cfg), out.data.data(), capture_f32));
  return out;
}

template <class Tensor, class Span, class KernelConfig>
Tensor embed(const Tensor& tok, const Tensor& pos, Span ids, int64_t batch, int64_t seq,
             const KernelConfig& cfg) {
  Tensor out({batch * seq, tok.shape[1]}, cfg.compute_dtype);
  if (static_cast<int64_t>(ids.size()) != batch * seq)
    throw std::invalid_argument("expected " + std::to_string(batch * seq) + " token ids, got " +
                                std::to_string(ids.size()));
  check(prlab_gpu_embed(tok.data.data(), tok.shape[0], pos.data.data(), pos.shape[0], tok.shape[1], ids.data(),
                        batch, seq, to_c(cfg), out.data.data()));
  return out;
}

}  // namespace gpu
}  // namespace prlab
