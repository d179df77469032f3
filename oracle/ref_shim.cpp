// prlab reference shim -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" surface over the UNMODIFIED reference sources
// (/root/reference/proj/src/{float16,tensor,kernels,policy,model,fidelity}.cpp),
// compiled by oracle/Makefile into oracle/_ref/libprlab_ref.so.  It lets the
// Python tests and bench.py's reference arm call the reference itself:
//   * to pin the C restatement (oracle/prlab_oracle.c) bit-for-bit,
//   * to generate tests/golden/ fixtures (tests/golden/make_golden.py),
//   * as the CPU baseline (`cpu_baseline.kind = "reference"`).
// No reference source is copied here; this file only calls its public API
// (include/prlab/{kernels,model,policy,fidelity}.hpp).
#include <cstring>
#include <span>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <algorithm>
#include <vector>

#include <chrono>

#include "prlab/bench.hpp"
#include "prlab/fidelity.hpp"
#include "prlab/float16.hpp"
#include "prlab/kernels.hpp"
#include "prlab/checkpoint.hpp"
#include "prlab/model.hpp"
#include "prlab/policy.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

prlab::ModelConfig make_cfg(int archetype, int64_t L, int64_t h, int64_t H, int64_t f,
                            int64_t V, int64_t P, uint64_t seed) {
  prlab::ModelConfig c;
  c.archetype = archetype == 0 ? prlab::Archetype::EncoderOnly : prlab::Archetype::DecoderOnly;
  c.num_layers = L;
  c.hidden = h;
  c.heads = H;
  c.ffn = f;
  c.vocab = V;
  c.max_positions = P;
  c.seed = seed;
  return c;
}

// Model whose parameters are copied from a flat canonical-order buffer.
prlab::Model model_from_flat(const prlab::ModelConfig& cfg, const float* params) {
  prlab::ModelConfig zero = cfg;
  prlab::Model m = prlab::build_model(zero);  // allocates every tensor with its shape
  const float* p = params;
  m.for_each_param([&p](const std::string&, prlab::Tensor& t) {
    std::memcpy(t.data.data(), p, t.data.size() * sizeof(float));
    p += t.data.size();
  });
  return m;
}

prlab::KernelConfig kcfg(int compute, int accum, int stabilized) {
  return {compute ? prlab::Dtype::F16E : prlab::Dtype::F32,
          accum ? prlab::Dtype::F16E : prlab::Dtype::F32, stabilized != 0};
}

prlab::Tensor tensor2(const float* p, int64_t r, int64_t c) {
  prlab::Tensor t({r, c});
  std::memcpy(t.data.data(), p, static_cast<size_t>(r * c) * sizeof(float));
  return t;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

float ref_round16(float x) { return prlab::round16(x); }
uint16_t ref_f16_encode(float x) { return prlab::f16_encode(x); }
float ref_f16_decode(uint16_t h) { return prlab::f16_decode(h); }

uint64_t ref_param_count(int archetype, int64_t L, int64_t h, int64_t H, int64_t f, int64_t V,
                         int64_t P) {
  return prlab::param_count(make_cfg(archetype, L, h, H, f, V, P, 0));
}

int ref_build_model(int archetype, int64_t L, int64_t h, int64_t H, int64_t f, int64_t V,
                    int64_t P, uint64_t seed, float* out) {
  try {
    const prlab::Model m = prlab::build_model(make_cfg(archetype, L, h, H, f, V, P, seed));
    float* o = out;
    m.for_each_param([&o](const std::string&, const prlab::Tensor& t) {
      std::memcpy(o, t.data.data(), t.data.size() * sizeof(float));
      o += t.data.size();
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

void ref_random_tokens(int64_t vocab, int64_t batch, int64_t seq, uint64_t seed, int32_t* ids) {
  const prlab::TokenBatch t = prlab::random_tokens(vocab, batch, seq, seed);
  std::memcpy(ids, t.ids.data(), t.ids.size() * sizeof(int32_t));
}

// Full forward through prlab::forward.  calls: optional [7][2].
// nthreads > 1 splits the batch into per-sequence forwards on std::threads
// (batched and per-sequence logits are bit-identical).
int ref_forward(int archetype, int64_t L, int64_t h, int64_t H, int64_t f, int64_t V,
                int64_t P, const float* params, const int32_t* ids, int64_t B, int64_t S,
                const char* policy, float* logits, uint64_t* calls, int nthreads) {
  try {
    const prlab::ModelConfig cfg = make_cfg(archetype, L, h, H, f, V, P, 0);
    const prlab::Model m = model_from_flat(cfg, params);
    const prlab::PrecisionPolicy pol = prlab::resolve_policy(policy);
    const int64_t out_w = L > 0 ? V : h;
    if (nthreads <= 1 || B == 1) {
      prlab::TokenBatch tb;
      tb.batch = B;
      tb.seq = S;
      tb.ids.assign(ids, ids + B * S);
      const prlab::ForwardTrace tr = prlab::forward(m, tb, pol);
      std::memcpy(logits, tr.logits.data.data(), tr.logits.data.size() * sizeof(float));
      if (calls) {
        for (int c = 0; c < prlab::kNumOpClasses; ++c)
          for (int d = 0; d < 2; ++d) calls[c * 2 + d] = tr.kernel_calls[c][d];
      }
      return 0;
    }
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<size_t>(nthreads));
    for (int t = 0; t < nthreads; ++t) {
      pool.emplace_back([&, t] {
        try {
          for (int64_t b = t; b < B; b += nthreads) {
            prlab::TokenBatch tb;
            tb.batch = 1;
            tb.seq = S;
            tb.ids.assign(ids + b * S, ids + (b + 1) * S);
            const prlab::ForwardTrace tr = prlab::forward(m, tb, pol);
            std::memcpy(logits + b * S * out_w, tr.logits.data.data(),
                        tr.logits.data.size() * sizeof(float));
          }
        } catch (const std::exception& e) {
          errs[static_cast<size_t>(t)] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (const auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    if (calls) std::memset(calls, 0, sizeof(uint64_t) * 14);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, -1);
  } catch (const std::out_of_range& e) {
    return fail(e, -2);
  } catch (const std::exception& e) {
    return fail(e, -3);
  }
}

// ---- model handle: the reference Model built ONCE (prlab::build_model, src/model.cpp:217-265)
// outside any timed region, as src/bench.cpp:47-106 run_benchmark / benchmark_forward expect.
void* ref_model_build(int archetype, int64_t L, int64_t h, int64_t H, int64_t f, int64_t V, int64_t P,
                      uint64_t seed) {
  try {
    return new prlab::Model(prlab::build_model(make_cfg(archetype, L, h, H, f, V, P, seed)));
  } catch (const std::exception& e) {
    fail(e, -1);
    return nullptr;
  }
}

void ref_model_free(void* m) { delete static_cast<prlab::Model*>(m); }

// The reference's own benchmark of one forward configuration: prlab::benchmark_forward
// (src/bench.cpp:102-106 -> run_benchmark :47-100) with BenchProtocol{warmup, measure},
// single-threaded.  out: mean_s, p50_s, p95_s, throughput_sps; samples: measure doubles.
int ref_benchmark_forward(void* m, const int32_t* ids, int64_t B, int64_t S, const char* policy,
                          int64_t warmup, int64_t measure, double* out, double* samples) {
  try {
    prlab::TokenBatch tb;
    tb.batch = B;
    tb.seq = S;
    tb.ids.assign(ids, ids + B * S);
    prlab::BenchProtocol proto;
    proto.warmup_iters = warmup;
    proto.measure_iters = measure;
    const prlab::BenchStats st =
        prlab::benchmark_forward(*static_cast<prlab::Model*>(m), tb, prlab::resolve_policy(policy), proto);
    out[0] = st.mean_s;
    out[1] = st.p50_s;
    out[2] = st.p95_s;
    out[3] = st.throughput_sps;
    for (size_t i = 0; i < st.samples_s.size(); ++i) samples[i] = st.samples_s[i];
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

// Throughput: B independent batch-1 prlab::forward calls of S tokens on `nthreads` host
// threads over the prebuilt Model (batched and per-sequence logits are bit-identical,
// SURVEY 8(d)); *seconds = steady_clock wall time of the forwards only (threads started
// before the clock, released together).  logits may be NULL (discarded).
int ref_forward_threads(void* mp, const int32_t* ids, int64_t B, int64_t S, const char* policy,
                        int nthreads, float* logits, double* seconds) {
  try {
    const prlab::Model& m = *static_cast<prlab::Model*>(mp);
    const prlab::PrecisionPolicy pol = prlab::resolve_policy(policy);
    const int64_t out_w = m.config.num_layers > 0 ? m.config.vocab : m.config.hidden;
    nthreads = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(nthreads, B)));
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<size_t>(nthreads));
    std::atomic<int> ready{0};
    std::atomic<bool> go{false};
    for (int t = 0; t < nthreads; ++t) {
      pool.emplace_back([&, t] {
        ready.fetch_add(1);
        while (!go.load(std::memory_order_acquire)) std::this_thread::yield();
        try {
          for (int64_t b = t; b < B; b += nthreads) {
            prlab::TokenBatch tb;
            tb.batch = 1;
            tb.seq = S;
            tb.ids.assign(ids + b * S, ids + (b + 1) * S);
            const prlab::ForwardTrace tr = prlab::forward(m, tb, pol);
            if (logits)
              std::memcpy(logits + b * S * out_w, tr.logits.data.data(), tr.logits.data.size() * sizeof(float));
          }
        } catch (const std::exception& e) {
          errs[static_cast<size_t>(t)] = e.what();
        }
      });
    }
    while (ready.load() < nthreads) std::this_thread::yield();
    const auto t0 = std::chrono::steady_clock::now();
    go.store(true, std::memory_order_release);
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (const auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

// prlab::forward with retain_scores: logits + the [L][B][H][S][S] fp32 pre-mask score taps
int ref_forward_scores(int archetype, int64_t L, int64_t h, int64_t H, int64_t f, int64_t V, int64_t P,
                       const float* params, const int32_t* ids, int64_t B, int64_t S, const char* policy,
                       float* logits, float* scores) {
  try {
    const prlab::Model m = model_from_flat(make_cfg(archetype, L, h, H, f, V, P, 0), params);
    prlab::TokenBatch tb;
    tb.batch = B;
    tb.seq = S;
    tb.ids.assign(ids, ids + B * S);
    const prlab::ForwardTrace tr = prlab::forward(m, tb, prlab::resolve_policy(policy), true);
    std::memcpy(logits, tr.logits.data.data(), tr.logits.data.size() * sizeof(float));
    float* o = scores;
    for (const auto& t : tr.layer_scores) {
      std::memcpy(o, t.data.data(), t.data.size() * sizeof(float));
      o += t.data.size();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

// prlab::classifier_probs (src/model.cpp:484-526)
int ref_classifier_probs(int archetype, int64_t L, int64_t h, int64_t H, int64_t f, int64_t V, int64_t P,
                         const float* params, const int32_t* ids, int64_t B, int64_t S, const char* policy,
                         float* out) {
  try {
    const prlab::Model m = model_from_flat(make_cfg(archetype, L, h, H, f, V, P, 0), params);
    prlab::TokenBatch tb;
    tb.batch = B;
    tb.seq = S;
    tb.ids.assign(ids, ids + B * S);
    const std::vector<float> pr = prlab::classifier_probs(m, tb, prlab::resolve_policy(policy));
    std::memcpy(out, pr.data(), pr.size() * sizeof(float));
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, -1);
  } catch (const std::exception& e) {
    return fail(e, -3);
  }
}

// prlab::perplexity (src/fidelity.cpp:248-279)
int ref_perplexity(int archetype, int64_t L, int64_t h, int64_t H, int64_t f, int64_t V, int64_t P,
                   const float* params, const int32_t* stream, int64_t n, int64_t context_len, const char* policy,
                   double* out) {
  try {
    const prlab::Model m = model_from_flat(make_cfg(archetype, L, h, H, f, V, P, 0), params);
    *out = prlab::perplexity(m, std::span<const int32_t>(stream, static_cast<size_t>(n)), context_len,
                             prlab::resolve_policy(policy));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

// serialize_checkpoint (src/checkpoint.cpp:104-121) of flat canonical params; dtype 0 f32, 1 f16
int ref_serialize_checkpoint(int archetype, int64_t L, int64_t h, int64_t H, int64_t f, int64_t V, int64_t P,
                             uint64_t seed, const float* params, int dtype, const char* path) {
  try {
    const prlab::Model m = model_from_flat(make_cfg(archetype, L, h, H, f, V, P, seed), params);
    prlab::serialize_checkpoint(m, dtype ? prlab::Dtype::F16E : prlab::Dtype::F32, path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

// load_checkpoint (src/checkpoint.cpp:133-162) -> flat canonical params
int ref_load_checkpoint(const char* path, float* out, int64_t cap) {
  try {
    const prlab::Model m = prlab::load_checkpoint(path);
    int64_t n = 0;
    m.for_each_param([&](const std::string&, const prlab::Tensor& t) {
      if (n + static_cast<int64_t>(t.data.size()) > cap) throw std::runtime_error("output too small");
      std::memcpy(out + n, t.data.data(), t.data.size() * sizeof(float));
      n += static_cast<int64_t>(t.data.size());
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

// make_adversarial_model (src/fidelity.cpp:282-312) -> flat canonical params
int ref_make_adversarial_model(int archetype, int64_t L, int64_t h, int64_t H, int64_t f, int64_t V,
                               int64_t P, uint64_t seed, const int32_t* probe_ids, int64_t B, int64_t S,
                               float target, float* out) {
  try {
    prlab::TokenBatch tb;
    tb.batch = B;
    tb.seq = S;
    tb.ids.assign(probe_ids, probe_ids + B * S);
    const prlab::Model m = prlab::make_adversarial_model(make_cfg(archetype, L, h, H, f, V, P, seed), tb, target);
    float* o = out;
    m.for_each_param([&o](const std::string&, const prlab::Tensor& t) {
      std::memcpy(o, t.data.data(), t.data.size() * sizeof(float));
      o += t.data.size();
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

// --- per-operator entry points (src/kernels.cpp) for KAT cross-checks ---
int ref_matmul(const float* a, const float* b, int64_t m, int64_t k, int64_t n, int compute,
               int accum, float* out) {
  try {
    const prlab::Tensor r = prlab::matmul(tensor2(a, m, k), tensor2(b, k, n), kcfg(compute, accum, 1));
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

int ref_attention_scores(const float* q, const float* k, int64_t sq, int64_t sk, int64_t d,
                         float scale, int compute, int accum, float* out, float* tap) {
  try {
    const prlab::Tensor r = prlab::attention_scores(tensor2(q, sq, d), tensor2(k, sk, d), scale,
                                                    kcfg(compute, accum, 1), tap);
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

int ref_softmax(const float* x, int64_t rows, int64_t n, int compute, int accum, int stabilized,
                float* out) {
  try {
    const prlab::Tensor r = prlab::softmax_lastdim(tensor2(x, rows, n), kcfg(compute, accum, stabilized));
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

int ref_layernorm(const float* x, int64_t rows, int64_t n, const float* g, const float* b,
                  float eps, int compute, int accum, float* out) {
  try {
    const prlab::Tensor r = prlab::layernorm_lastdim(tensor2(x, rows, n), tensor2(g, 1, n),
                                                     tensor2(b, 1, n), eps, kcfg(compute, accum, 1));
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

int ref_gelu(const float* x, int64_t n, int compute, int accum, float* out) {
  try {
    const prlab::Tensor r = prlab::gelu(tensor2(x, 1, n), kcfg(compute, accum, 1));
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

int ref_embed(const float* tok, int64_t vocab, const float* pos, int64_t npos, int64_t h,
              const int32_t* ids, int64_t batch, int64_t seq, int compute, float* out) {
  try {
    const prlab::Tensor r = prlab::embed(tensor2(tok, vocab, h), tensor2(pos, npos, h),
                                         std::span<const int32_t>(ids, static_cast<size_t>(batch * seq)),
                                         batch, seq, kcfg(compute, compute, 1));
    std::memcpy(out, r.data.data(), r.data.size() * sizeof(float));
    return 0;
  } catch (const std::out_of_range& e) {
    return fail(e, -2);
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

}  // extern "C"
