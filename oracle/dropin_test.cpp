// Link-level drop-in check -- TEST INFRASTRUCTURE ONLY.
//
// A C++ program written against the reference API (include/prlab/*.hpp, the
// unmodified reference sources compiled beside it) that swaps prlab::forward /
// prlab::matmul for prlab::gpu::forward / prlab::gpu::matmul (include/prlab_gpu.hpp)
// and checks: same logits shape, cosine >= 0.9998 vs the CPU fp32 forward, zero
// non-finite, the reference's exception types, and the KATs of test_kernels.cpp.
// Built by oracle/Makefile into oracle/_ref/dropin_test; run on the GPU box by
// tests/test_gpu_dropin.py.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <thread>
#include <vector>

#include "prlab/fidelity.hpp"
#include "prlab/kernels.hpp"
#include "prlab/model.hpp"
#include "prlab/policy.hpp"
#include "prlab_gpu.hpp"

static int failures = 0;
#define CHECK(cond, what)                                  \
  do {                                                     \
    if (cond) {                                            \
      std::printf("[PASS] %s\n", what);                    \
    } else {                                               \
      std::printf("[FAIL] %s\n", what);                    \
      ++failures;                                          \
    }                                                      \
  } while (0)

int main() {
  using namespace prlab;
  // --- model forward drop-in (GPT-2 preset, batch 1, seq 32)
  const Model model = build_model(ModelConfig::gpt2_small());
  const TokenBatch tokens = random_tokens(model.config.vocab, 1, 32, 1234);
  const ForwardTrace cpu = forward(model, tokens, resolve_policy("fp32"));
  const auto gpu = gpu::forward(model, tokens, resolve_policy("hybrid"));
  CHECK(gpu.logits.shape == cpu.logits.shape, "logits shape matches prlab::forward");
  const LogitComparison cmp = compare_logits(cpu.logits, gpu.logits);
  std::printf("       cosine %.7f max_abs %.3e nonfinite %llu\n", cmp.cosine.value_or(0.0), cmp.max_abs_error,
              static_cast<unsigned long long>(cmp.candidate_nonfinite));
  CHECK(cmp.cosine && *cmp.cosine >= 0.9998 && cmp.candidate_nonfinite == 0, "hybrid GPU vs CPU fp32 cosine >= 0.9998");
  const auto gpu32 = gpu::forward(model, tokens, resolve_policy("fp32"));
  double max_abs = 0.0, max_ref = 0.0;
  for (size_t i = 0; i < cpu.logits.data.size(); ++i) {
    max_abs = std::fmax(max_abs, std::fabs(static_cast<double>(gpu32.logits.data[i]) - cpu.logits.data[i]));
    max_ref = std::fmax(max_ref, std::fabs(static_cast<double>(cpu.logits.data[i])));
  }
  std::printf("       fp32 rel err %.3e\n", max_abs / max_ref);
  CHECK(max_abs / max_ref <= 1e-3, "fp32 GPU vs CPU within 1e-3 relative");
  const ForwardTrace cpu_h = forward(model, tokens, resolve_policy("hybrid"));
  bool calls_equal = true;
  for (int c = 0; c < kNumOpClasses; ++c)
    for (int d = 0; d < 2; ++d) calls_equal &= cpu_h.kernel_calls[c][d] == gpu.kernel_calls[c][d];
  CHECK(calls_equal, "ForwardTrace kernel_calls identical to the reference");

  // --- ForwardTrace::seconds filled (CUDA-event time per op class, timed() wrappers)
  CHECK(gpu.seconds[static_cast<int>(OpClass::Linear)] > 0.0 &&
            gpu.seconds[static_cast<int>(OpClass::LayerNorm)] > 0.0,
        "ForwardTrace seconds per op class measured on the device");

  // --- retain_scores: layer_scores [B,H,S,S] fp32 pre-mask taps (model.cpp:393-427)
  {
    const ForwardTrace cpu_t = forward(model, tokens, resolve_policy("hybrid"), true);
    const auto gpu_t = gpu::forward(model, tokens, resolve_policy("hybrid"), true);
    bool shape_ok = gpu_t.layer_scores.size() == cpu_t.layer_scores.size();
    double md = 0.0, mref = 0.0;
    for (size_t l = 0; shape_ok && l < cpu_t.layer_scores.size(); ++l) {
      shape_ok &= gpu_t.layer_scores[l].shape == cpu_t.layer_scores[l].shape;
      for (size_t i = 0; shape_ok && i < cpu_t.layer_scores[l].data.size(); ++i) {
        md = std::max(md, std::fabs(static_cast<double>(gpu_t.layer_scores[l].data[i]) - cpu_t.layer_scores[l].data[i]));
        mref = std::max(mref, std::fabs(static_cast<double>(cpu_t.layer_scores[l].data[i])));
      }
    }
    std::printf("       layer_scores max |gpu-cpu| %.3e (max |score| %.3e)\n", md, mref);
    CHECK(shape_ok && md <= 2e-2 * std::max(mref, 1e-3), "retain_scores layer_scores match the reference taps");
  }

  // --- classifier_probs (model.cpp:484-526) on a BERT-shaped encoder
  {
    ModelConfig ec = ModelConfig::bert_base();
    ec.num_layers = 2;
    ec.vocab = 4096;
    const Model enc = build_model(ec);
    const TokenBatch et = random_tokens(ec.vocab, 3, 48, 11);
    const std::vector<float> want = classifier_probs(enc, et, resolve_policy("fp32"));
    const std::vector<float> got = gpu::classifier_probs(enc, et, resolve_policy("hybrid"));
    const std::vector<float> got32 = gpu::classifier_probs(enc, et, resolve_policy("fp32"));
    double d16 = 0.0, d32 = 0.0;
    for (size_t i = 0; i < want.size(); ++i) {
      d16 = std::max(d16, std::fabs(static_cast<double>(got[i]) - want[i]));
      d32 = std::max(d32, std::fabs(static_cast<double>(got32[i]) - want[i]));
    }
    std::printf("       classifier |hybrid-cpu32| %.3e |fp32-cpu32| %.3e\n", d16, d32);
    CHECK(got.size() == want.size() && d16 <= 2e-3 && d32 <= 1e-5, "classifier_probs matches the reference");
    bool dec = false;
    try {
      gpu::classifier_probs(model, tokens, resolve_policy("hybrid"));
    } catch (const std::invalid_argument&) {
      dec = true;
    }
    CHECK(dec, "classifier_probs on a decoder -> std::invalid_argument");
  }

  // --- concurrent callers (the reference's free functions are safe on distinct data,
  //     SPEC.md:118-119): four threads x 8 forwards on one model through forward_untimed
  //     (the fused path with the overlapped copy-out); every call equals its serial result
  {
    std::vector<TokenBatch> tb;
    std::vector<std::vector<float>> want;
    for (int t = 0; t < 4; ++t) {
      tb.push_back(random_tokens(model.config.vocab, 1, 128, 500 + t));
      want.push_back(gpu::forward_untimed(model, tb.back(), resolve_policy("hybrid")).logits.data);
    }
    std::atomic<int> mismatches{0}, errors{0};
    std::vector<std::thread> th;
    for (int t = 0; t < 4; ++t)
      th.emplace_back([&, t] {
        try {
          for (int r = 0; r < 8; ++r)
            if (gpu::forward_untimed(model, tb[t], resolve_policy("hybrid")).logits.data != want[t]) ++mismatches;
        } catch (const std::exception&) {
          ++errors;
        }
      });
    for (auto& x : th) x.join();
    const auto timed = gpu::forward(model, tb[0], resolve_policy("hybrid"));
    double md = 0.0;
    for (size_t i = 0; i < want[0].size(); ++i) md = std::max(md, std::fabs(static_cast<double>(timed.logits.data[i]) - want[0][i]));
    std::printf("       concurrent: %d mismatches, %d errors; timed vs untimed max |diff| %.3e\n", mismatches.load(),
                errors.load(), md);
    CHECK(mismatches == 0 && errors == 0, "4 concurrent callers x 8 forwards return their serial logits");
    CHECK(md <= 2e-2, "forward (instrumented) and forward_untimed (fused) agree");
  }

  // --- exceptions: same types as the reference
  TokenBatch bad = tokens;
  bad.ids[3] = static_cast<int32_t>(model.config.vocab);
  bool oor = false;
  try {
    gpu::forward(model, bad, resolve_policy("hybrid"));
  } catch (const std::out_of_range&) {
    oor = true;
  }
  CHECK(oor, "bad token id -> std::out_of_range");
  bool inv = false;
  try {
    TokenBatch longer = random_tokens(model.config.vocab, 1, 1025, 1);
    gpu::forward(model, longer, resolve_policy("hybrid"));
  } catch (const std::invalid_argument&) {
    inv = true;
  }
  CHECK(inv, "seq > max_positions -> std::invalid_argument");

  // --- operator KATs through the drop-in (test_kernels.cpp:37-60, 82-98)
  const KernelConfig f16acc{Dtype::F16E, Dtype::F16E, true}, f16wide{Dtype::F16E, Dtype::F32, true},
      f32{Dtype::F32, Dtype::F32, true}, unstable{Dtype::F16E, Dtype::F16E, false};
  Tensor a({1, 2049}), b({2049, 1});
  for (float& v : a.data) v = 1.0f;
  for (float& v : b.data) v = 1.0f;
  CHECK(gpu::matmul(a, b, f16acc).data[0] == 2048.0f && gpu::matmul(a, b, f16wide).data[0] == 2048.0f &&
            gpu::matmul(a, b, f32).data[0] == 2049.0f,
        "2049 ones: 2048 / 2048 / 2049");
  const Tensor x = Tensor::from({1, 2}, {12.0f, 0.0f});
  const Tensor y = gpu::softmax_lastdim(x, f16acc);
  const Tensor z = gpu::softmax_lastdim(x, unstable);
  CHECK(y.data[0] == 1.0f && y.data[1] == 6.139278411865234e-06f && std::isnan(z.data[0]) && z.data[1] == 0.0f,
        "softmax [12,0]: stabilized / unstabilized");
  bool cfg_bad = false;
  try {
    gpu::matmul(a, b, KernelConfig{Dtype::F32, Dtype::F16E, true});
  } catch (const std::invalid_argument&) {
    cfg_bad = true;
  }
  CHECK(cfg_bad, "f32 compute with f16e accumulation -> std::invalid_argument");
  std::printf("%s (%d failures)\n", failures ? "DROPIN FAIL" : "DROPIN OK", failures);
  return failures ? 1 : 0;
}
