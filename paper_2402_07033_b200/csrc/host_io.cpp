// host_io.cpp — see host_io.h.  Compiled by g++ into libmoe_b200.so.
#include "host_io.h"

#include <immintrin.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace moe_host {
namespace {

// Persistent worker pool: spawning 16 threads per call cost more than the
// conversion itself.  Leaked on purpose (workers block on a condition
// variable; nothing to join at exit).
class Pool {
 public:
  static Pool& get() {
    static Pool* p = new Pool();
    return *p;
  }
  int size() const { return (int)workers_.size() + 1; }
  // fn(i) for i in [0, n) on the workers and the calling thread; blocks.
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> job(job_mu_);  // one job at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_ = 0;
      pending_ = n;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  Pool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nw = std::min(hw, 16u) - 1;
    for (unsigned i = 0; i < nw; ++i)
      workers_.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
          }
          work();
        }
      });
    for (auto& t : workers_) t.detach();
  }
  void work() {
    for (;;) {
      const std::function<void(int)>* fn;
      int i;
      {
        // grab a task of the CURRENT job atomically: while it runs,
        // pending_ > 0 keeps run() (and the job's fn) alive
        std::lock_guard<std::mutex> lk(mu_);
        if (!fn_ || next_ >= n_) return;
        fn = fn_;
        i = next_++;
      }
      (*fn)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0, pending_ = 0, next_ = 0;
  uint64_t gen_ = 0;
};

constexpr size_t kMin = 1 << 16;  // below: one thread

// [a, b) with a 16-float aligned split; pieces of `parts`
template <typename F>
void split(size_t n, F&& body) {
  if (n < 2 * kMin) {
    body(0, n);
    return;
  }
  Pool& pool = Pool::get();
  const int parts = (int)std::min<size_t>((size_t)pool.size() * 2, (n + kMin - 1) / kMin);
  pool.run(parts, [&](int t) {
    size_t a = n * t / parts, b = n * (t + 1) / parts;
    a &= ~size_t(15);
    if (t + 1 < parts) b &= ~size_t(15);
    body(a, b);
  });
}

__attribute__((target("avx2"))) void f32_nt_avx2(float* dst, const double* src, size_t a, size_t b) {
  size_t i = a;
  for (; i < b && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) dst[i] = (float)src[i];
  for (; i + 8 <= b; i += 8) {
    const __m128 lo = _mm256_cvtpd_ps(_mm256_loadu_pd(src + i));
    const __m128 hi = _mm256_cvtpd_ps(_mm256_loadu_pd(src + i + 4));
    _mm256_stream_ps(dst + i, _mm256_set_m128(hi, lo));
  }
  for (; i < b; ++i) dst[i] = (float)src[i];
  _mm_sfence();
}

}  // namespace

void to_f32_dma(float* dst, const double* src, size_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  split(n, [&](size_t a, size_t b) {
    if (avx2) {
      f32_nt_avx2(dst, src, a, b);
    } else {
      for (size_t i = a; i < b; ++i) dst[i] = (float)src[i];
    }
  });
}

void to_f64(double* dst, const float* src, size_t n) {
  split(n, [&](size_t a, size_t b) {
    for (size_t i = a; i < b; ++i) dst[i] = (double)src[i];
  });
}

}  // namespace moe_host
