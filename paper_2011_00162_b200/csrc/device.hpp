// Small RAII helpers for device memory, streams and graphs.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "plan.hpp"

namespace pdd {

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define PDD_CUDA(call) ::pdd::cuda_check((call), #call)

// Page-locked download staging (common.cuh HostStage), reserved ahead of use.
void host_stage_reserve();

// Untyped device allocation.  Freed on destruction.
class DevMem {
  static void keep_pool_mapped() {
    static thread_local int done_for = -1;  // device whose pool is configured (per thread: cheap check)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_for) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    done_for = dev;
  }

 public:
  DevMem() = default;
  explicit DevMem(size_t bytes) { alloc(bytes); }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  DevMem(DevMem&& o) noexcept : p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DevMem& operator=(DevMem&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  ~DevMem() { release(); }
  // Stream-ordered allocations from the device's default pool, which keeps
  // freed memory mapped (release threshold raised once per device): a solver
  // built after another was destroyed reuses its multi-GB buffers instead of
  // paying cudaMalloc's page mapping again (3-150 ms per solve on c4).  Both
  // calls synchronise like cudaMalloc/cudaFree did, so buffers are usable from
  // any stream on return and are freed only after all device work completes.
  void alloc(size_t bytes) {
    release();
    if (bytes == 0) return;
    keep_pool_mapped();
    PDD_CUDA(cudaMallocAsync(&p_, bytes, cudaStreamLegacy));
    PDD_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    n_ = bytes;
  }
  void release() {
    if (p_) {
      cudaDeviceSynchronize();
      cudaFreeAsync(p_, cudaStreamLegacy);
      cudaStreamSynchronize(cudaStreamLegacy);
    }
    p_ = nullptr;
    n_ = 0;
  }
  template <typename U>
  U* as() const {
    return static_cast<U*>(p_);
  }
  void* get() const { return p_; }
  size_t bytes() const { return n_; }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

template <typename U>
DevMem upload(const std::vector<U>& v, cudaStream_t st) {
  DevMem m(sizeof(U) * (v.empty() ? 1 : v.size()));
  if (!v.empty()) PDD_CUDA(cudaMemcpyAsync(m.get(), v.data(), sizeof(U) * v.size(), cudaMemcpyHostToDevice, st));
  return m;
}

class Stream {
 public:
  Stream() { PDD_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking)); }
  ~Stream() {
    if (s_) cudaStreamDestroy(s_);
  }
  Stream(const Stream&) = delete;
  Stream& operator=(const Stream&) = delete;
  cudaStream_t get() const { return s_; }
  void sync() const { PDD_CUDA(cudaStreamSynchronize(s_)); }

 private:
  cudaStream_t s_ = nullptr;
};

class Graph {
 public:
  Graph() = default;
  ~Graph() { reset(); }
  Graph(const Graph&) = delete;
  Graph& operator=(const Graph&) = delete;
  void reset() {
    if (exec_) cudaGraphExecDestroy(exec_);
    if (graph_) cudaGraphDestroy(graph_);
    exec_ = nullptr;
    graph_ = nullptr;
  }
  bool ready() const { return exec_ != nullptr; }
  template <class F>
  void capture(cudaStream_t st, F&& body) {
    reset();
    PDD_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    try {
      body();
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    PDD_CUDA(cudaStreamEndCapture(st, &graph_));
    PDD_CUDA(cudaGraphInstantiate(&exec_, graph_, 0));
  }
  void launch(cudaStream_t st) const { PDD_CUDA(cudaGraphLaunch(exec_, st)); }

 private:
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t exec_ = nullptr;
};

// Scoped device selection.
class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    PDD_CUDA(cudaGetDevice(&prev_));
    if (dev != prev_) PDD_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev_); }

 private:
  int prev_ = 0;
};

}  // namespace pdd
