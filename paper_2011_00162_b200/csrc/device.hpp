// Small RAII helpers for device memory, streams and graphs.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <functional>
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

// Library-private stream-ordered memory pool per device (device.cpp): freed
// blocks stay mapped for the next solver (repeated solves skip cudaMalloc's
// page mapping); pdd_release_cached_memory() returns them, as does the
// destruction of the last solver on a device with PDD_POOL_TRIM_ON_IDLE=1.
// The device's default pool and every other allocator in the process are
// left alone.
cudaMemPool_t device_pool(int dev);
void pool_retain(int dev);
void pool_release(int dev);   // last user on dev: trim if PDD_POOL_TRIM_ON_IDLE=1
void release_cached_memory();  // all devices

// The stream on which DevMem allocations of this thread are ordered (set by
// AllocStream scopes: a solver's stream, an operator call's stream).
cudaStream_t& alloc_stream_tl();
class AllocStream {
 public:
  explicit AllocStream(cudaStream_t s) : prev_(alloc_stream_tl()) { alloc_stream_tl() = s; }
  ~AllocStream() { alloc_stream_tl() = prev_; }
  AllocStream(const AllocStream&) = delete;
  AllocStream& operator=(const AllocStream&) = delete;

 private:
  cudaStream_t prev_;
};

// Keeps the device pool mapped for the lifetime of its owner (declare it
// before any DevMem so it is destroyed after them).
class PoolUser {
 public:
  explicit PoolUser(int dev) : dev_(dev) { pool_retain(dev); }
  ~PoolUser() { pool_release(dev_); }
  PoolUser(const PoolUser&) = delete;
  PoolUser& operator=(const PoolUser&) = delete;

 private:
  int dev_;
};

// Untyped device allocation, stream-ordered on the stream of the enclosing
// AllocStream scope: allocated with cudaMallocFromPoolAsync and freed with
// cudaFreeAsync on that stream, so neither call waits for unrelated device
// work.  All uses must be ordered on that stream (or after a host
// synchronisation of it).  Outside any scope (none on the solver paths) the
// allocation is made complete before return and the free waits for the
// device, as cudaMalloc/cudaFree would.
class DevMem {
 public:
  DevMem() = default;
  explicit DevMem(size_t bytes) { alloc(bytes); }
  DevMem(size_t bytes, cudaStream_t st) { alloc(bytes, st); }
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  DevMem(DevMem&& o) noexcept : p_(o.p_), n_(o.n_), st_(o.st_), ordered_(o.ordered_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DevMem& operator=(DevMem&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      st_ = o.st_;
      ordered_ = o.ordered_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  ~DevMem() { release(); }
  void alloc(size_t bytes) {
    cudaStream_t s = alloc_stream_tl();
    if (s) {
      alloc(bytes, s);
      return;
    }
    release();
    if (bytes == 0) return;
    int dev = 0;
    PDD_CUDA(cudaGetDevice(&dev));
    PDD_CUDA(cudaMallocFromPoolAsync(&p_, bytes, device_pool(dev), cudaStreamPerThread));
    PDD_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
    n_ = bytes;
    st_ = cudaStreamPerThread;
    ordered_ = false;
  }
  void alloc(size_t bytes, cudaStream_t st) {
    release();
    if (bytes == 0) return;
    int dev = 0;
    PDD_CUDA(cudaGetDevice(&dev));
    PDD_CUDA(cudaMallocFromPoolAsync(&p_, bytes, device_pool(dev), st));
    n_ = bytes;
    st_ = st;
    ordered_ = true;
  }
  void release() noexcept {
    if (p_) {
      if (!ordered_) cudaDeviceSynchronize();
      if (cudaFreeAsync(p_, st_) != cudaSuccess) {
        // the stream is gone or broken: wait for the device, free in order
        cudaGetLastError();
        cudaDeviceSynchronize();
        cudaFreeAsync(p_, cudaStreamPerThread);
        cudaGetLastError();
      }
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
  cudaStream_t st_ = nullptr;
  bool ordered_ = false;
};

template <typename U>
DevMem upload(const std::vector<U>& v, cudaStream_t st) {
  DevMem m(sizeof(U) * (v.empty() ? 1 : v.size()), st);
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

// A captured CUDA graph -- or, in eager mode, the recorded body itself,
// re-run on every launch (for transports whose calls block on the host and so
// cannot be captured; Comm::capturable()).
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
    eager_ = nullptr;
  }
  bool ready() const { return exec_ != nullptr || eager_ != nullptr; }
  // body must stay valid for the graph's lifetime in eager mode (capture by value)
  void capture(cudaStream_t st, std::function<void()> body, bool eager = false) {
    reset();
    if (eager) {
      eager_ = std::move(body);
      return;
    }
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
  void launch(cudaStream_t st) const {
    if (eager_) {
      eager_();
      return;
    }
    PDD_CUDA(cudaGraphLaunch(exec_, st));
  }

 private:
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t exec_ = nullptr;
  std::function<void()> eager_;
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
