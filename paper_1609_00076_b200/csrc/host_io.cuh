// host_io.cuh -- host-side transfer machinery shared by the host-pointer
// entry points (host_path.cu: one device; multi_host.cu: several devices):
// a small host thread pool for pitched copies, a pinned staging ring for
// pageable callers, and the Mover that issues pitched H2D/D2H copies on a
// given pair of streams.  Copies are pitched (width rows*8): padding rows
// are never read or written and nothing past (n-1)*ld+m is touched
// (matrix.py:5-6,42-45,58-61).
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

namespace myd {
namespace hostio {

// ---- a small fork-free host thread pool for pitched copies ----
class CopyPool {
 public:
  static CopyPool &get() {
    static CopyPool pool;
    return pool;
  }
  // Run fn(i) for i in [0, n) on the pool and the calling thread; blocks.
  // One job at a time (concurrent callers -- the per-device threads of the
  // multi-device path -- take turns).  Each job's state (index counter, done
  // count) lives in its own shared Job, which a worker snapshots under the
  // lock: a worker that wakes late for a finished job only ever sees that
  // job's exhausted counter, never the next job's indices, and never calls a
  // function whose caller has returned.
  void parallel_for(int n, const std::function<void(int)> &fn) {
    if (n <= 1 || workers_.empty()) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    std::lock_guard<std::mutex> run(run_mu_);
    auto job = std::make_shared<Job>(&fn, n);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = job;
      ++gen_;
    }
    cv_.notify_all();
    work(*job);
    {
      std::unique_lock<std::mutex> lk(job->mu);
      job->cv.wait(lk, [&] { return job->done == job->total; });
    }
    std::lock_guard<std::mutex> lk(mu_);
    job_.reset();
  }

 private:
  struct Job {
    Job(const std::function<void(int)> *f, int n) : fn(f), total(n) {}
    const std::function<void(int)> *fn;
    const int total;
    std::atomic<int> next{0};
    int done = 0;  // guarded by mu
    std::mutex mu;
    std::condition_variable cv;
  };
  CopyPool() {
    int want = 8;
    if (const char *s = getenv("MY_DGEMM_HOST_THREADS")) want = std::max(1, atoi(s));
    const int hw = (int)std::thread::hardware_concurrency();
    if (hw > 0) want = std::min(want, hw);
    for (int t = 1; t < want; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : workers_) t.join();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::shared_ptr<Job> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_); });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      work(*job);
    }
  }
  static void work(Job &job) {
    int did = 0;
    for (int i = job.next.fetch_add(1); i < job.total; i = job.next.fetch_add(1)) {
      (*job.fn)(i);
      ++did;
    }
    if (did) {
      std::lock_guard<std::mutex> lk(job.mu);
      job.done += did;
      if (job.done == job.total) job.cv.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex run_mu_, mu_;
  std::condition_variable cv_;
  std::shared_ptr<Job> job_;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// pitched host copy of `cols` columns of `rows` doubles, split over the pool
inline void host_copy_2d(double *dst, int64_t dpitch, const double *src, int64_t spitch, int64_t rows,
                         int64_t cols) {
  const int64_t bytes = rows * 8;
  const int64_t per = std::max<int64_t>(1, (4 << 20) / std::max<int64_t>(bytes, 1));  // ~4 MB per task
  const int tasks = (int)((cols + per - 1) / per);
  CopyPool::get().parallel_for(tasks, [&](int t) {
    const int64_t c0 = t * per, c1 = std::min<int64_t>(cols, c0 + per);
    for (int64_t c = c0; c < c1; ++c) memcpy(dst + c * dpitch, src + c * spitch, (size_t)bytes);
  });
}

inline bool is_pinned(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Pinned staging buffers for pageable host memory, each with the event of
// its last DMA.
struct StageRing {
  static constexpr int MAX = 8;
  static constexpr size_t BYTES = 32u << 20;
  int n = 0;
  double *buf[MAX] = {};
  cudaEvent_t ev[MAX] = {};
  cudaError_t ensure(int count) {  // on the current device
    count = std::min(count, MAX);
    cudaError_t e;
    for (; n < count; ++n) {
      if ((e = cudaMallocHost((void **)&buf[n], BYTES)) != cudaSuccess) return e;
      if ((e = cudaEventCreateWithFlags(&ev[n], cudaEventDisableTiming)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  void release() {
    for (int i = 0; i < n; ++i) {
      if (ev[i]) {
        cudaEventSynchronize(ev[i]);
        cudaEventDestroy(ev[i]);
      }
      if (buf[i]) cudaFreeHost(buf[i]);
      buf[i] = nullptr;
      ev[i] = nullptr;
    }
    n = 0;
  }
};

// Moves pitched column blocks between host and device on the given streams:
// straight DMA for pinned host memory (ring == nullptr), through the staging
// ring for pageable memory (host threads fill/drain the ring; the issuing
// thread blocks only on the copy work it must do itself).
class Mover {
 public:
  Mover(StageRing *ring, cudaStream_t up_stream, cudaStream_t down_stream)
      : ring_(ring), s_up_(up_stream), s_down_(down_stream) {}

  cudaError_t up(double *d, int64_t dpitch, const double *h, int64_t hpitch, int64_t rows, int64_t cols) {
    if (!ring_ || rows * 8 > (int64_t)StageRing::BYTES)  // a column larger than a stage: direct
      return cudaMemcpy2DAsync(d, dpitch * 8, h, (size_t)hpitch * 8, (size_t)rows * 8, cols,
                               cudaMemcpyHostToDevice, s_up_);
    const int64_t per = std::max<int64_t>(1, (int64_t)(StageRing::BYTES / 8) / rows);
    for (int64_t c0 = 0; c0 < cols; c0 += per) {
      const int64_t nc = std::min(per, cols - c0);
      const int s = next();
      cudaError_t e = drain_until_free(s);  // buffer free (pending copy-outs done, last DMA done)
      if (e != cudaSuccess) return e;
      host_copy_2d(ring_->buf[s], rows, h + c0 * hpitch, hpitch, rows, nc);
      e = cudaMemcpy2DAsync(d + c0 * dpitch, dpitch * 8, ring_->buf[s], (size_t)rows * 8, (size_t)rows * 8, nc,
                            cudaMemcpyHostToDevice, s_up_);
      if (e != cudaSuccess) return e;
      if ((e = cudaEventRecord(ring_->ev[s], s_up_)) != cudaSuccess) return e;
    }
    return cudaSuccess;
  }

  // Queue a download; staged pieces are copied out to the user buffer as
  // their DMA completes (at the latest in finish()).
  cudaError_t down(double *h, int64_t hpitch, const double *d, int64_t dpitch, int64_t rows, int64_t cols) {
    if (!ring_ || rows * 8 > (int64_t)StageRing::BYTES)
      return cudaMemcpy2DAsync(h, (size_t)hpitch * 8, d, dpitch * 8, (size_t)rows * 8, cols,
                               cudaMemcpyDeviceToHost, s_down_);
    const int64_t per = std::max<int64_t>(1, (int64_t)(StageRing::BYTES / 8) / rows);
    for (int64_t c0 = 0; c0 < cols; c0 += per) {
      const int64_t nc = std::min(per, cols - c0);
      const int s = next();
      cudaError_t e = drain_until_free(s);
      if (e != cudaSuccess) return e;
      e = cudaMemcpy2DAsync(ring_->buf[s], (size_t)rows * 8, d + c0 * dpitch, dpitch * 8, (size_t)rows * 8, nc,
                            cudaMemcpyDeviceToHost, s_down_);
      if (e != cudaSuccess) return e;
      if ((e = cudaEventRecord(ring_->ev[s], s_down_)) != cudaSuccess) return e;
      pending_.push_back({s, h + c0 * hpitch, hpitch, rows, nc});
    }
    return cudaSuccess;
  }

  cudaError_t finish() {
    while (!pending_.empty()) {
      cudaError_t e = pop();
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }

 private:
  struct Out {
    int s;
    double *h;
    int64_t hpitch, rows, cols;
  };
  int next() {
    const int s = slot_;
    slot_ = (slot_ + 1) % ring_->n;
    return s;
  }
  cudaError_t pop() {
    Out o = pending_.front();
    pending_.pop_front();
    cudaError_t e = cudaEventSynchronize(ring_->ev[o.s]);
    if (e != cudaSuccess) return e;
    host_copy_2d(o.h, o.hpitch, ring_->buf[o.s], o.rows, o.rows, o.cols);
    return cudaSuccess;
  }
  // Before reusing stage s, copy out (in queue order) every pending piece up
  // to the one that occupies s, then wait for the stage's last DMA.
  cudaError_t drain_until_free(int s) {
    auto uses = [&] {
      for (const Out &o : pending_)
        if (o.s == s) return true;
      return false;
    };
    while (uses()) {
      cudaError_t e = pop();
      if (e != cudaSuccess) return e;
    }
    return cudaEventSynchronize(ring_->ev[s]);
  }
  StageRing *ring_;
  cudaStream_t s_up_, s_down_;
  int slot_ = 0;
  std::deque<Out> pending_;
};

}  // namespace hostio
}  // namespace myd
