// hostio.cuh — host-side helpers of the streamed host I/O paths (the
// one-shot Cholesky call, the SHT batches over host buffers): a small pool
// of host threads that split a copy / conversion, and grow-only pinned
// staging buffers.
#pragma once

#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace sphemu_gpu {

// Blocking parallel-for over a fixed set of host threads (the caller runs
// share 0). Used by the packed host I/O to convert tile rows between fp64 and
// their storage width on the host side of the link.
class HostPool {
 public:
  explicit HostPool(int n) : n_(std::max(1, n)) {
    for (int t = 1; t < n_; ++t) th_.emplace_back([this, t] { loop(t); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  void run(const std::function<void(int, int)>& f) {
    std::unique_lock<std::mutex> lk(mu_);
    job_ = &f;
    pending_ = n_ - 1;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    f(0, n_);
    lk.lock();
    done_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int t) {
    uint64_t seen = 0;
    while (true) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      const auto* f = job_;
      lk.unlock();
      (*f)(t, n_);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int, int)>* job_ = nullptr;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

struct PinnedBuf {
  char* p = nullptr;
  size_t n = 0;
  void ensure(size_t bytes) {
    if (n >= bytes) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    SPH_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), bytes, cudaHostAllocDefault));
    n = bytes;
  }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};

}  // namespace sphemu_gpu
