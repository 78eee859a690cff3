// hostconv.cpp -- see hostconv.h.
#pragma GCC optimize("O3")
#include "hostconv.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "internal.h"

namespace rk {

HostPool::HostPool(int threads) {
  for (int i = 1; i < threads; ++i) workers_.emplace_back([this, i] { loop(i); });
}

HostPool::~HostPool() {
  {
    std::lock_guard<std::mutex> l(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void HostPool::loop(int) {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(size_t, size_t)>* fn;
    {
      std::unique_lock<std::mutex> l(mu_);
      cv_.wait(l, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      fn = fn_;
    }
    for (;;) {
      size_t b;
      {
        std::lock_guard<std::mutex> l(mu_);
        if (next_ >= n_) break;
        b = next_;
        next_ += chunk_;
      }
      (*fn)(b, std::min(n_, b + chunk_));
    }
    {
      std::lock_guard<std::mutex> l(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
}

void HostPool::parallel_for(size_t n, size_t min_chunk, const std::function<void(size_t, size_t)>& fn) {
  if (n == 0) return;
  std::lock_guard<std::mutex> call(call_mu_);
  const size_t parts = (size_t)size();
  const size_t chunk = std::max(min_chunk, (n + parts * 4 - 1) / (parts * 4));
  if (workers_.empty() || n <= chunk) {
    fn(0, n);
    return;
  }
  {
    std::lock_guard<std::mutex> l(mu_);
    fn_ = &fn;
    n_ = n;
    chunk_ = chunk;
    next_ = 0;
    pending_ = (int)workers_.size();
    ++gen_;
  }
  cv_.notify_all();
  for (;;) {  // the caller works too
    size_t b;
    {
      std::lock_guard<std::mutex> l(mu_);
      if (next_ >= n_) break;
      b = next_;
      next_ += chunk_;
    }
    fn(b, std::min(n, b + chunk));
  }
  std::unique_lock<std::mutex> l(mu_);
  done_cv_.wait(l, [&] { return pending_ == 0; });
  fn_ = nullptr;
}

Uploader::Uploader(int device) : device_(device), thread_([this] { loop(); }) {}

Uploader::~Uploader() {
  {
    std::lock_guard<std::mutex> l(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  thread_.join();
}

void Uploader::submit(std::function<void()> job) {
  {
    std::lock_guard<std::mutex> l(mu_);
    queue_.push_back(std::move(job));
  }
  cv_.notify_all();
}

void Uploader::loop() {
  cudaSetDevice(device_);
  for (;;) {
    std::function<void()> job;
    {
      std::unique_lock<std::mutex> l(mu_);
      cv_.wait(l, [&] { return stop_ || !queue_.empty(); });
      if (queue_.empty()) return;  // stop requested and drained
      job = std::move(queue_.front());
      queue_.erase(queue_.begin());
    }
    job();
  }
}

PinnedPool::~PinnedPool() {
  for (auto& kv : free_) cudaFreeHost(kv.second);
}

void* PinnedPool::acquire(size_t bytes, size_t* got) {
  {
    std::lock_guard<std::mutex> l(mu_);
    auto it = free_.lower_bound(bytes);
    if (it != free_.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      *got = it->first;
      free_.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  RK_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  *got = bytes;
  return p;
}

void PinnedPool::release(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> l(mu_);
  free_.emplace(bytes, p);
}

__attribute__((target_clones("arch=x86-64-v4", "avx2", "default"))) void f32_to_bf16_host(const float* src,
                                                                                      uint16_t* dst, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t u;
    std::memcpy(&u, src + i, 4);
    const uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
    const uint32_t nan = (u >> 16) | 0x40u;  // quiet NaN keeps its sign and payload top bits
    dst[i] = (uint16_t)((u & 0x7FFFFFFFu) > 0x7F800000u ? nan : r);
  }
}

}  // namespace rk
