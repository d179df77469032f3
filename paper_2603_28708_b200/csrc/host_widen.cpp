// Device fp16 rows -> host fp32 rows for the drop-in forward (prlab_gpu_forward).
//
// Under the hybrid policy the tied head's outputs are round16'd (Linear class, F16E
// compute): every logit is an fp16 value, so fp32 logits on the host are exactly the
// fp16 logits widened.  Moving the fp16 rows over PCIe and widening them on the host
// halves the device->host bytes of the call (25.7 MB -> 12.9 MB for GPT-2 at seq 128),
// which is what bounds the end-to-end call (bench.py e2e).  The copy is chunked by rows:
// the calling thread waits on each chunk's CUDA event in order and publishes it; the pool
// threads widen their share of the chunk's columns as soon as it is published, while the
// next chunks are still in flight.  Widening is exact (F16C / bit-exact scalar path).
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace prlab_gpu {

namespace {

inline float half_bits_to_float(uint16_t h) {
  const uint32_t sign = static_cast<uint32_t>(h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1Fu, man = h & 0x3FFu, bits;
  if (exp == 0x1F) {
    bits = sign | 0x7F800000u | (man << 13);  // inf / nan (payload kept)
  } else if (exp == 0) {
    if (man == 0) {
      bits = sign;
    } else {  // subnormal: normalise
      int e = -1;
      do {
        man <<= 1;
        ++e;
      } while ((man & 0x400u) == 0);
      bits = sign | (static_cast<uint32_t>(127 - 15 - e) << 23) | ((man & 0x3FFu) << 13);
    }
  } else {
    bits = sign | ((exp + 112u) << 23) | (man << 13);
  }
  float f;
  std::memcpy(&f, &bits, 4);
  return f;
}

void widen_rows_scalar(const uint16_t* src, int64_t lds, float* dst, int64_t ldd, int64_t rows, int64_t n) {
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t i = 0; i < n; ++i) dst[r * ldd + i] = half_bits_to_float(src[r * lds + i]);
}

__attribute__((target("avx2,f16c"))) void widen_rows_f16c(const uint16_t* src, int64_t lds, float* dst, int64_t ldd,
                                                          int64_t rows, int64_t n) {
  for (int64_t r = 0; r < rows; ++r) {
    const uint16_t* s = src + r * lds;
    float* d = dst + r * ldd;
    int64_t i = 0;
    while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31u) != 0) {
      d[i] = half_bits_to_float(s[i]);
      ++i;
    }
    // streaming stores: the destination is not re-read here, so skip the write-allocate
    for (; i + 8 <= n; i += 8)
      _mm256_stream_ps(d + i, _mm256_cvtph_ps(_mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i))));
    for (; i < n; ++i) d[i] = half_bits_to_float(s[i]);
  }
  _mm_sfence();
}

void widen_rows(const uint16_t* src, int64_t lds, float* dst, int64_t ldd, int64_t rows, int64_t n) {
  static const bool f16c = __builtin_cpu_supports("avx2") && __builtin_cpu_supports("f16c");
  if (f16c)
    widen_rows_f16c(src, lds, dst, ldd, rows, n);
  else
    widen_rows_scalar(src, lds, dst, ldd, rows, n);
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// Persistent worker threads; run(n, f) executes f(0..n-1) on the pool and the caller.
class Pool {
 public:
  explicit Pool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return static_cast<int>(th_.size()); }
  // start(n, f): the workers begin executing f(0..n-1); finish(): the caller joins the
  // remaining items, waits for the workers and rethrows the first error.
  void start(int n, const std::function<void(int)>& f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      njobs_ = n;
      next_.store(0);
      pending_ = static_cast<int>(th_.size());
      err_.clear();
      ++gen_;
    }
    cv_.notify_all();
  }
  void finish() {
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
    if (!err_.empty()) throw std::runtime_error(err_);
  }

 private:
  void work() {
    for (int j; (j = next_.fetch_add(1)) < njobs_;) {
      try {
        (*job_)(j);
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lk(err_mu_);
        if (err_.empty()) err_ = e.what();
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_, err_mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int njobs_ = 0, pending_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
  std::string err_;
};

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::max(1, std::atoi(v)) : dflt;
}

struct Widener {
  std::mutex mu;  // one call at a time (the staging buffer and events are shared)
  // pool threads (+ the caller); PRLAB_WIDEN_THREADS overrides (tuning)
  // half the host's hardware threads, at most 8: on the 16-core B200 host the copy-out
  // of GPT-2's 128 x 50257 logits takes 0.33 ms at 8 threads vs 0.42 at 4 and 0.50 for
  // the fp32 copy (scripts/e2e_sweep.py)
  Pool pool{env_int("PRLAB_WIDEN_THREADS",
                    std::max(1, std::min(8, static_cast<int>(std::thread::hardware_concurrency()) / 2))) - 1};
  void* staging = nullptr;
  size_t cap = 0;
  std::vector<cudaEvent_t> ev;
  ~Widener() {
    if (staging) cudaFreeHost(staging);
    for (auto e : ev) cudaEventDestroy(e);
  }
};

Widener& widener(int dev) {  // per device: the staging buffer is portable, the events are not
  static std::mutex mu;
  static std::vector<std::unique_ptr<Widener>> all;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0) throw std::invalid_argument("d2h_widen_f16: bad device");
  if (static_cast<int>(all.size()) <= dev) all.resize(dev + 1);
  if (!all[dev]) all[dev].reset(new Widener());
  return *all[dev];
}

}  // namespace

void d2h_widen_f16(const void* d_src, int64_t ld_src, float* h_dst, int64_t ld_dst, int64_t rows, int64_t cols,
                   cudaStream_t st) {
  int dev = 0;
  check(cudaGetDevice(&dev), "cudaGetDevice");
  Widener& w = widener(dev);
  std::lock_guard<std::mutex> lk(w.mu);
  const size_t bytes = static_cast<size_t>(rows) * cols * 2;
  if (bytes > w.cap) {
    if (w.staging) check(cudaFreeHost(w.staging), "cudaFreeHost");
    w.staging = nullptr;
    w.cap = 0;
    check(cudaMallocHost(&w.staging, bytes), "cudaMallocHost(widen staging)");
    w.cap = bytes;
  }
  // 8 row chunks: each D2H copy costs ~3.5 us of setup (128 x 50257 fp16: 238 us as one
  // copy, 293 us as 16 -- scripts/ubench/ubench_d2h.py), fewer chunks leave a longer widening
  // tail; measured e2e 0.686 ms at 8 vs 0.697 at 12 and 0.703 at 6 (scripts/gpu_e2e_sweep.sh).
  // Moving a slice of the rows as fp32 instead (device-widened) did not help: the host's
  // DRAM bandwidth, shared by the DMA writes and the widening, is the bound.
  static const int kChunks = env_int("PRLAB_WIDEN_CHUNKS", 8);
  const int64_t per = (rows + kChunks - 1) / kChunks;
  const int nch = static_cast<int>((rows + per - 1) / per);
  while (static_cast<int>(w.ev.size()) < nch) {
    cudaEvent_t e;
    check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    w.ev.push_back(e);
  }
  uint16_t* stg = static_cast<uint16_t*>(w.staging);
  for (int c = 0; c < nch; ++c) {
    const int64_t r0 = c * per, nr = std::min(per, rows - r0);
    check(cudaMemcpy2DAsync(stg + r0 * cols, cols * 2, static_cast<const uint16_t*>(d_src) + r0 * ld_src, ld_src * 2,
                            cols * 2, nr, cudaMemcpyDeviceToHost, st),
          "cudaMemcpy2DAsync(logits)");
    check(cudaEventRecord(w.ev[c], st), "cudaEventRecord");
  }
  // Only the caller talks to CUDA (waiting on the chunk events in order and publishing
  // `ready`); the pool threads spin on that counter and widen 1/P of every chunk's
  // columns each -- CUDA calls from several threads contend on driver locks
  // (measured: spinning cudaEventSynchronize in 8+ threads was slower than 4).
  const int P = w.pool.size() + 1;
  std::atomic<int> ready{0};
  std::atomic<bool> failed{false};
  const std::function<void(int)> job = [&](int i) {
    const int c = i / P, q = i % P;
    while (ready.load(std::memory_order_acquire) <= c) {
      if (failed.load(std::memory_order_relaxed)) return;
      _mm_pause();
    }
    const int64_t r0 = c * per, nr = std::min(per, rows - r0);
    const int64_t c0 = (cols * q / P) & ~int64_t(7), c1 = q + 1 == P ? cols : (cols * (q + 1) / P) & ~int64_t(7);
    if (c1 > c0) widen_rows(stg + r0 * cols + c0, cols, h_dst + r0 * ld_dst + c0, ld_dst, nr, c1 - c0);
  };
  w.pool.start(nch * P, job);
  try {
    for (int c = 0; c < nch; ++c) {
      check(cudaEventSynchronize(w.ev[c]), "cudaEventSynchronize");
      ready.store(c + 1, std::memory_order_release);
    }
  } catch (...) {
    failed.store(true);
    w.pool.finish();
    throw;
  }
  w.pool.finish();
}

}  // namespace prlab_gpu
