// Library-private device memory pools (device.hpp).
#include "device.hpp"

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

// Created on first use with release threshold 0 (cudaMalloc-like: freed
// memory goes back to the OS at the next synchronisation) and raised to
// "keep everything" while solvers live on the device.
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
    r.set_threshold(dev, r.live[dev] > 0 ? UINT64_MAX : 0);
  }
  return r.pool[dev];
}

void pool_retain(int dev) {
  device_pool(dev);  // creates it
  auto& r = PoolRegistry::get();
  std::lock_guard<std::mutex> lock(r.mu);
  if (r.live[dev]++ == 0) r.set_threshold(dev, UINT64_MAX);
}

void pool_release(int dev) {
  if (dev < 0 || dev >= kMaxDevices) return;
  auto& r = PoolRegistry::get();
  std::lock_guard<std::mutex> lock(r.mu);
  if (r.live[dev] > 0 && --r.live[dev] == 0 && r.pool[dev]) {
    // frees still pending in stream order are returned at the next
    // synchronisation (threshold 0); the rest goes back now
    r.set_threshold(dev, 0);
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
