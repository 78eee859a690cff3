// hostconv.h -- host-side helpers of the asynchronous relay-cache upload:
// a worker pool, a pinned staging pool and the fp32 -> bf16 conversion.
#pragma once
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

namespace rk {

// Fixed worker pool; parallel_for splits [0, n) into contiguous chunks run by
// the workers and the caller. Calls from several threads are serialised.
class HostPool {
 public:
  explicit HostPool(int threads);
  ~HostPool();
  void parallel_for(size_t n, size_t min_chunk, const std::function<void(size_t, size_t)>& fn);
  int size() const { return (int)workers_.size() + 1; }

 private:
  void loop(int id);
  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t, size_t)>* fn_ = nullptr;
  size_t n_ = 0, chunk_ = 0;
  size_t next_ = 0;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// One background thread running queued jobs in order (the host side of the
// asynchronous relay-cache uploads).
class Uploader {
 public:
  explicit Uploader(int device);
  ~Uploader();
  void submit(std::function<void()> job);

 private:
  void loop();
  int device_;
  std::thread thread_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<std::function<void()>> queue_;
  bool stop_ = false;
};

// Page-locked host blocks, reused (cudaHostAlloc is slow).
class PinnedPool {
 public:
  ~PinnedPool();
  void* acquire(size_t bytes, size_t* got);
  void release(void* p, size_t bytes);

 private:
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
};

// bf16 = round-to-nearest-even of fp32 (== __float2bfloat16_rn for non-NaN).
void f32_to_bf16_host(const float* src, uint16_t* dst, size_t n);

}  // namespace rk
