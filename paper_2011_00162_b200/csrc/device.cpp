// Library-private device memory pools (device.hpp).
#include "device.hpp"

#include <cstdlib>
#include <mutex>

namespace pdd {
namespace {

constexpr int kMaxDevices = 64;

struct PoolRegistry {
  std::mutex mu;
  cudaMemPool_t pool[kMaxDevices] = {};
  int live[kMaxDevices] = {};
  static PoolRegistry& get() {
    static PoolRegistry r;
    return r;
  }
  void set_threshold(int dev, uint64_t v) {
    cudaMemPoolSetAttribute(pool[dev], cudaMemPoolAttrReleaseThreshold, &v);
  }
};

void check_dev(int dev) {
  if (dev < 0 || dev >= kMaxDevices) throw InvalidArgument("device ordinal out of range");
}

}  // namespace

cudaStream_t& alloc_stream_tl() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

// Created on first use.  Freed blocks stay mapped (release threshold "keep
// everything"): a solver built after another was destroyed -- the usual
// pattern of a caller running several solves -- reuses its buffers instead of
// paying the page mapping again (the first 30 GB of config 4 cost ~0.1-0.4 s).
// The memory is returned by pdd_release_cached_memory(), or automatically
// when the last solver on the device is destroyed if PDD_POOL_TRIM_ON_IDLE=1.
// Only this private pool is configured; the device's default pool and other
// allocators (torch, NCCL) are untouched.
cudaMemPool_t device_pool(int dev) {
  check_dev(dev);
  auto& r = PoolRegistry::get();
  std::lock_guard<std::mutex> lock(r.mu);
  if (!r.pool[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    PDD_CUDA(cudaMemPoolCreate(&r.pool[dev], &props));
    r.set_threshold(dev, UINT64_MAX);
  }
  return r.pool[dev];
}

void pool_retain(int dev) {
  device_pool(dev);  // creates it
  auto& r = PoolRegistry::get();
  std::lock_guard<std::mutex> lock(r.mu);
  ++r.live[dev];
}

void pool_release(int dev) {
  if (dev < 0 || dev >= kMaxDevices) return;
  static const bool trim_on_idle = [] {
    const char* e = std::getenv("PDD_POOL_TRIM_ON_IDLE");
    return e && e[0] == '1';
  }();
  auto& r = PoolRegistry::get();
  std::lock_guard<std::mutex> lock(r.mu);
  if (r.live[dev] > 0 && --r.live[dev] == 0 && r.pool[dev] && trim_on_idle) {
    // blocks whose stream-ordered free is still pending stay until the next trim
    cudaMemPoolTrimTo(r.pool[dev], 0);
    cudaGetLastError();
  }
}

void release_cached_memory() {
  auto& r = PoolRegistry::get();
  std::lock_guard<std::mutex> lock(r.mu);
  for (int dev = 0; dev < kMaxDevices; ++dev)
    if (r.pool[dev]) {
      DeviceGuard g(dev);
      PDD_CUDA(cudaDeviceSynchronize());
      PDD_CUDA(cudaMemPoolTrimTo(r.pool[dev], 0));
    }
}

}  // namespace pdd
