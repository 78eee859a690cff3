// prof.h -- optional per-launch timing of the hot kernels (CUDA events on the
// engine stream) with their algorithmic work, for roofline reporting.
#pragma once
#include <set>
#include <string>
#include <vector>

#include "internal.h"

namespace rk {

struct ProfRec {
  const char* name;
  int ev0, ev1;        // indices into the engine's profiling event pool
  double flops, bytes;  // algorithmic work when known on the host
  // deferred work (sparse passes: live rows / positions only on the device)
  const int* rows_dev = nullptr;
  const int* pos = nullptr;
  int rows_max = 0;
  int kind = 0;        // 0 fixed, 1 gemm (2*M*N*K), 2 attention (4*dh*H*sum(pos+1))
  int N = 0, K = 0, H = 0, dh = 0;
};

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<ProfRec> recs;
  int next = 0;
  int ev(cudaStream_t st) {
    if (next >= (int)pool.size()) {
      cudaEvent_t e;
      RK_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    RK_CUDA(cudaEventRecord(pool[next], st));
    return next++;
  }
};

Profiler& profiler(rk_engine* e);
// Stable storage for generated kernel labels.
const char* intern(const std::string& s);

// RAII scope around one launch.
struct ProfScope {
  rk_engine* e;
  ProfRec rec;
  bool on;
  ProfScope(rk_engine* eng, const char* name, double flops, double bytes);
  ~ProfScope();
};

}  // namespace rk
