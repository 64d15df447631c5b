// Developer probe: device->host download strategies for the e2e result copy
// (2.2 GB of complex128 on config 4).  nvcc -O2 -std=c++17 -o scripts/bin/d2h_probe scripts/d2h_probe.cu -lpthread
#include <cuda_runtime.h>
#include <sys/mman.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static char* prefaulted(size_t n) {
  char* p = static_cast<char*>(aligned_alloc(4096, n));
  madvise(p, n, MADV_HUGEPAGE);
  for (size_t o = 0; o < n; o += 4096) p[o] = 0;
  return p;
}

int main(int argc, char** argv) {
  const size_t n = (argc > 1 ? atol(argv[1]) : 1024) << 20;
  const int nth = argc > 2 ? atoi(argv[2]) : 8;
  printf("bytes %zu, host threads %d, hw threads %u\n", n, nth, std::thread::hardware_concurrency());
  char* dev;
  CK(cudaMalloc(&dev, n));
  CK(cudaMemset(dev, 1, n));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaDeviceSynchronize());

  // 1. pageable copy into prefaulted memory
  {
    char* h = prefaulted(n);
    double t0 = now();
    CK(cudaMemcpyAsync(h, dev, n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double t1 = now();
    printf("pageable          : %.1f ms  %.1f GB/s\n", (t1 - t0) * 1e3, n / (t1 - t0) / 1e9);
    free(h);
  }
  // 2. pageable, nth threads each copying a slice on its own stream
  {
    char* h = prefaulted(n);
    double t0 = now();
    std::vector<std::thread> th;
    for (int k = 0; k < nth; ++k)
      th.emplace_back([&, k] {
        cudaStream_t s;
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        const size_t a = n / nth * k, b = k + 1 == nth ? n : n / nth * (k + 1);
        CK(cudaMemcpyAsync(h + a, dev + a, b - a, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaStreamDestroy(s));
      });
    for (auto& x : th) x.join();
    double t1 = now();
    printf("pageable x%-2d      : %.1f ms  %.1f GB/s\n", nth, (t1 - t0) * 1e3, n / (t1 - t0) / 1e9);
    free(h);
  }
  // 3. cudaHostRegister cost + registered copy
  {
    char* h = prefaulted(n);
    double t0 = now();
    CK(cudaHostRegister(h, n, cudaHostRegisterDefault));
    double t1 = now();
    CK(cudaMemcpyAsync(h, dev, n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double t2 = now();
    CK(cudaHostUnregister(h));
    double t3 = now();
    printf("register %.1f ms, copy %.1f ms (%.1f GB/s), unregister %.1f ms\n", (t1 - t0) * 1e3, (t2 - t1) * 1e3,
           n / (t2 - t1) / 1e9, (t3 - t2) * 1e3);
    free(h);
  }
  // 4. pinned staging ring (2 x chunk) + nth host threads copying out
  for (size_t chunk : {size_t(16) << 20, size_t(64) << 20}) {
    char* h = prefaulted(n);
    double ta = now();
    char* stg;
    CK(cudaMallocHost(&stg, 2 * chunk));
    double t0 = now();
    cudaEvent_t ev[2];
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    const size_t nc = (n + chunk - 1) / chunk;
    auto issue = [&](size_t c) {
      const size_t o = c * chunk, m = std::min(chunk, n - o);
      CK(cudaMemcpyAsync(stg + (c & 1) * chunk, dev + o, m, cudaMemcpyDeviceToHost, st));
      CK(cudaEventRecord(ev[c & 1], st));
    };
    issue(0);
    for (size_t c = 0; c < nc; ++c) {
      CK(cudaEventSynchronize(ev[c & 1]));
      // the other slot was consumed in the previous round: refill it while this one drains
      if (c + 1 < nc) issue(c + 1);
      const size_t o = c * chunk, m = std::min(chunk, n - o);
      std::vector<std::thread> th;
      for (int k = 0; k < nth; ++k)
        th.emplace_back([&, k] {
          const size_t a = m / nth * k, b = k + 1 == nth ? m : m / nth * (k + 1);
          memcpy(h + o + a, stg + (c & 1) * chunk + a, b - a);
        });
      for (auto& x : th) x.join();
    }
    double t1 = now();
    printf("staging %3zu MB x%-2d: alloc %.1f ms, copy %.1f ms  %.1f GB/s\n", chunk >> 20, nth, (t0 - ta) * 1e3,
           (t1 - t0) * 1e3, n / (t1 - t0) / 1e9);
    CK(cudaFreeHost(stg));
    free(h);
  }
  return 0;
}
