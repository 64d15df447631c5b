// Per-rank device resources shared by the nonblind and blind drivers:
// measured amplitudes, frame/tile/pair tables, reduction scratch, iteration
// control, and the setup computations of the reference constructors
// (frame partitioning, pins, R-factor denominator).
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "device.hpp"
#include "engine.hpp"
#include "frame_kernel.cuh"
#include "kernels.hpp"
#include "layout.hpp"
#include "ptya.hpp"

namespace pdd {

template <typename T>
std::vector<cx<T>> to_cx(const double* p, int64_t n) {
  std::vector<cx<T>> v(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) v[i] = cx<T>{static_cast<T>(p[2 * i]), static_cast<T>(p[2 * i + 1])};
  return v;
}

template <typename T>
void from_cx(const std::vector<cx<T>>& v, double* out) {
  for (size_t i = 0; i < v.size(); ++i) {
    out[2 * i] = static_cast<double>(v[i].x);
    out[2 * i + 1] = static_cast<double>(v[i].y);
  }
}

template <typename T>
std::vector<cx<T>> twiddles(int S) {
  std::vector<cx<T>> w(static_cast<size_t>(S));
  for (int k = 0; k < S; ++k) {
    const double a = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(S);
    w[k] = cx<T>{static_cast<T>(std::cos(a)), static_cast<T>(std::sin(a))};
  }
  return w;
}

template <typename T>
std::vector<cx<T>> download_cx(const void* dev, int64_t n, cudaStream_t st) {
  std::vector<cx<T>> h(static_cast<size_t>(n));
  if (n > 0) PDD_CUDA(cudaMemcpyAsync(h.data(), dev, sizeof(cx<T>) * n, cudaMemcpyDeviceToHost, st));
  PDD_CUDA(cudaStreamSynchronize(st));
  return h;
}

// PDD_TIMING=1: setup phase timings on stderr (developer aid).
struct SetupTimer {
  bool on = std::getenv("PDD_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pdd] %-24s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};

// Large device -> host result copies (the e2e downloads: sub-solutions, merged
// image, state).  A plain cudaMemcpy into pageable memory runs at ~17 GB/s on
// the B200 hosts (the driver bounces through its own staging buffer on one
// thread).  Here W host threads each own a slice of a page-locked staging
// buffer and a stream: a thread DMAs its next chunk of T-precision data (at
// the full ~57 GB/s shared by all threads), then widens it to complex128 into
// the caller's buffer while the other threads' DMAs proceed.  float data thus
// crosses PCIe at half the bytes and is widened on the host (exact).
struct HostStage {
  static constexpr size_t kBytes = size_t(32) << 20;  // total page-locked staging
  std::mutex mu;
  void* buf = nullptr;
  int workers = 0;  // the buffer lives for the process (no CUDA calls in static destructors)
  void reserve_locked() {
    if (buf) return;
    PDD_CUDA(cudaHostAlloc(&buf, kBytes, cudaHostAllocPortable));
    // half the host threads (at most 8): the copy saturates at ~8 threads, and
    // leaving cores free keeps a descheduled worker from stalling the drain
    workers = static_cast<int>(std::clamp(std::thread::hardware_concurrency() / 2, 2u, 8u));
  }
  void reserve() {
    std::lock_guard<std::mutex> lock(mu);
    reserve_locked();
  }
  // At solver construction: the first page-locked allocation of a process
  // takes tens of ms, so it runs on a helper thread while the amplitudes
  // upload and the device loop execute (errors resurface at the first use).
  void reserve_async(int device) {
    if (started.exchange(true)) return;
    std::thread([this, device] {
      try {
        PDD_CUDA(cudaSetDevice(device));
        reserve();
      } catch (...) {
        cudaGetLastError();
      }
    }).detach();
  }
  std::atomic<bool> started{false};
  static HostStage& get() {
    static HostStage s;
    return s;
  }
};

template <typename T>
void download_c128_staged(const cx<T>* dev, int64_t n, double* out, cudaStream_t st) {
  PDD_CUDA(cudaStreamSynchronize(st));  // the producer's work is complete
  SetupTimer tm;
  int device = 0;
  PDD_CUDA(cudaGetDevice(&device));
  HostStage& hs = HostStage::get();
  std::lock_guard<std::mutex> lock(hs.mu);
  hs.reserve_locked();
  tm.mark("staged: lock+alloc");
  const int W = hs.workers;
  const int64_t chunk = static_cast<int64_t>(HostStage::kBytes / W / sizeof(cx<T>));
  const int64_t nchunks = (n + chunk - 1) / chunk;
  std::vector<cudaError_t> err(W, cudaSuccess);
  std::vector<std::thread> th;
  std::atomic<int64_t> next{0};  // chunks handed out on demand: a slow worker takes fewer
  for (int k = 0; k < W; ++k)
    th.emplace_back([&, k] {
      cudaError_t e = cudaSetDevice(device);
      cudaStream_t s = nullptr;
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      cx<T>* stage = reinterpret_cast<cx<T>*>(static_cast<char*>(hs.buf) + HostStage::kBytes / W * k);
      for (int64_t c = next.fetch_add(1); c < nchunks && e == cudaSuccess; c = next.fetch_add(1)) {
        const int64_t o = c * chunk, m = std::min(chunk, n - o);
        e = cudaMemcpyAsync(stage, dev + o, sizeof(cx<T>) * m, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) break;
        if constexpr (sizeof(T) == sizeof(double)) {
          std::memcpy(out + 2 * o, stage, sizeof(cx<T>) * m);
        } else {
          double* q = out + 2 * o;
          for (int64_t i = 0; i < m; ++i) {
            q[2 * i] = static_cast<double>(stage[i].x);
            q[2 * i + 1] = static_cast<double>(stage[i].y);
          }
        }
      }
      if (s) cudaStreamDestroy(s);
      err[k] = e;
    });
  for (auto& x : th) x.join();
  tm.mark("staged: copy");
  for (cudaError_t e : err) PDD_CUDA(e);
}

// Device complex<T> -> host complex128.  Large copies go through the staged
// multi-threaded path above; small ones widen on the device and copy directly.
template <typename T>
void download_c128(const void* dev, int64_t n, double* out, cudaStream_t st) {
  if (n <= 0) return;
  static const bool staged = [] {
    const char* e = std::getenv("PDD_STAGED_D2H");
    return !(e && e[0] == '0');
  }();
  if (staged && n >= (int64_t(1) << 20)) {
    download_c128_staged<T>(static_cast<const cx<T>*>(dev), n, out, st);
    return;
  }
  if constexpr (sizeof(T) == sizeof(double)) {
    PDD_CUDA(cudaMemcpyAsync(out, dev, sizeof(cx<double>) * n, cudaMemcpyDeviceToHost, st));
  } else {
    const int64_t chunk = std::min<int64_t>(n, int64_t(32) << 20);
    DevMem tmp(sizeof(cx<double>) * chunk);
    for (int64_t o = 0; o < n; o += chunk) {
      const int64_t m = std::min(chunk, n - o);
      PDD_CUDA(launch_widen_cx(static_cast<const cx<float>*>(dev) + o, tmp.as<cx<double>>(), m, st));
      PDD_CUDA(cudaMemcpyAsync(out + 2 * o, tmp.get(), sizeof(cx<double>) * m, cudaMemcpyDeviceToHost, st));
      PDD_CUDA(cudaStreamSynchronize(st));
    }
  }
  PDD_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void upload_cx(void* dev, const double* src, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  auto h = to_cx<T>(src, n);
  PDD_CUDA(cudaMemcpyAsync(dev, h.data(), sizeof(cx<T>) * n, cudaMemcpyHostToDevice, st));
  PDD_CUDA(cudaStreamSynchronize(st));
}


// Page-locks a caller's pageable host buffer for the duration of one upload
// (DMA at full PCIe/C2C rate instead of staged pageable copies).  Process-wide
// registry: concurrent uploads from the same buffer share one registration,
// which is dropped by the last of them only after its stream has drained;
// buffers page-locked by someone else are used as they are.  The destructor
// covers the exception paths.
class HostPin {
 public:
  HostPin(const void* p, size_t bytes, cudaStream_t st) : p_(p), st_(st) {
    if (!p) return;
    std::lock_guard<std::mutex> lock(mu());
    auto& reg = table();
    if (auto it = reg.find(p); it != reg.end()) {
      if (it->second.bytes >= bytes) {
        ++it->second.users;
        mine_ = true;
      }
      return;
    }
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeUnregistered &&
        cudaHostRegister(const_cast<void*>(p), bytes, cudaHostRegisterReadOnly) == cudaSuccess) {
      reg[p] = Entry{bytes, 1};
      mine_ = true;
    }
    cudaGetLastError();
  }
  ~HostPin() { done(); }
  HostPin(const HostPin&) = delete;
  HostPin& operator=(const HostPin&) = delete;
  // Drain this upload's stream, then drop this user's share of the registration.
  void done() noexcept {
    if (!mine_) return;
    mine_ = false;
    cudaStreamSynchronize(st_);
    std::lock_guard<std::mutex> lock(mu());
    auto& reg = table();
    auto it = reg.find(p_);
    if (it != reg.end() && --it->second.users == 0) {
      cudaHostUnregister(const_cast<void*>(p_));
      reg.erase(it);
    }
    cudaGetLastError();
  }

 private:
  struct Entry {
    size_t bytes;
    int users;
  };
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::map<const void*, Entry>& table() {
    static std::map<const void*, Entry> t;
    return t;
  }
  const void* p_;
  cudaStream_t st_;
  bool mine_ = false;
};

// Streams run() records to a RecordFn as the device completes them.
struct RecordFeed {
  const RecordFn* cb = nullptr;
  int64_t start = 0;      // iteration count before this run
  int64_t delivered = 0;  // absolute iteration of the last record handed out
  // Hand out records start+1.. last (absolute).  rec: the device record ring
  // [rec_cap][2] (rf, re); ms: device ms per 2-iteration launch so far.
  void upto(const double* dev_rec, int rec_cap, cudaStream_t st, int64_t last, const std::vector<double>& ms,
            const std::vector<double>* lag = nullptr) {
    if (!cb || !*cb) return;
    if (delivered < start) delivered = start;
    if (last <= delivered) return;
    std::vector<double> rec(2 * static_cast<size_t>(rec_cap));
    PDD_CUDA(cudaMemcpyAsync(rec.data(), dev_rec, sizeof(double) * rec.size(), cudaMemcpyDeviceToHost, st));
    PDD_CUDA(cudaStreamSynchronize(st));
    for (int64_t n = delivered + 1; n <= last; ++n) {
      const int64_t k = (n - 1) % rec_cap, i = n - start;
      const double t = ms.empty() ? 0.0 : ms[std::min<size_t>(static_cast<size_t>((i - 1) / 2), ms.size() - 1)] / 2.0;
      const double L = lag && i - 1 < static_cast<int64_t>(lag->size()) ? (*lag)[i - 1] : NAN;
      (*cb)(i, rec[2 * k], rec[2 * k + 1], t, L);
    }
    delivered = last;
  }
};

// Device ms between consecutive events (all recorded work complete).
inline std::vector<double> event_ms(const std::vector<cudaEvent_t>& ev) {
  std::vector<double> ms;
  for (size_t i = 1; i < ev.size(); ++i) {
    float t = 0.f;
    PDD_CUDA(cudaEventElapsedTime(&t, ev[i - 1], ev[i]));
    ms.push_back(t);
  }
  return ms;
}

template <typename T>
struct RankData {
  Layout L;
  int S = 0, device = 0;
  Comm* comm = nullptr;
  Stream stream;
  Stream side;  // the forked consensus branch of the iteration (fork_consensus)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  DevMem amp, tw;
  DevMem fr_off, fr_pitch, fr_r, fr_c, fr_sub;
  DevMem tiles, tile_frames, sub_off, sub_h, sub_w, sub_pbeg, psides, pgeom;
  DevMem sub_fr_beg, sub_tile_beg, local_map;
  DevMem pc_beg, pc_pos, pc_ofs, pc_rec, it_r, it_c, it_h, it_base, tile_items, tile_item_beg;  // back-projection pieces
  DevMem fmeta_beg, fmeta, fmeta_base, imeta_beg, imeta, imeta_base, tps_beg, tps;  // flattened gather lists
  DevMem rf_part, re_part, sums;  // sums: [3][D] = rf, diff, norm per subdomain
  DevMem fin_counter;
  DevMem scratch;  // global transpose tiles of the streamed kernel (complex128 128^2 frames)
  DevMem ctl, rec;
  DevMem pin_dev;  // uint8 per local image pixel
  double l1 = 0.0;
  int D = 0;
  bool rows_al16 = false;  // every window row 16-byte aligned in the image buffers
  int rec_cap = 0;

  cudaStream_t st() const { return stream.get(); }
  int64_t SS() const { return static_cast<int64_t>(S) * S; }
  double* rf_sub() const { return sums.as<double>(); }
  double* diff_sub() const { return sums.as<double>() + D; }
  double* norm_sub() const { return sums.as<double>() + 2 * D; }
  RunCtl* ctlp() const { return ctl.as<RunCtl>(); }
  int* skipA() const { return &ctl.as<RunCtl>()->skipA; }
  int* skipB() const { return &ctl.as<RunCtl>()->skipB; }
  int* skipC() const { return &ctl.as<RunCtl>()->skipC; }

  // piece_len > 1: multi-frame back-projection pieces for the streamed sweep (layout.hpp)
  void build(const Plan& plan, const DataSpec& data, const double* pin_ones, int dev, Comm* c, int max_iters,
             const char* who, int piece_len = 1) {
    device = dev;
    comm = c;
    const int rank = c ? c->rank() : 0, world = c ? c->world() : 1;
    SetupTimer tm;
    HostStage::get().reserve_async(dev);  // result-download staging, off the critical path
    L = Layout::build(plan, rank, world, sizeof(T) == 4, piece_len);
    tm.mark("layout");
    S = L.S;
    D = plan.D;
    if (!frame_supported<T>(S))
      throw InvalidArgument(std::string(who) + ": frame side " + std::to_string(S) +
                            " not supported by the CUDA path (powers of two up to " +
                            "128)");
    cudaStream_t s = st();
    tw = upload(twiddles<T>(S), s);
    fr_off = upload(L.fr_off, s);
    rows_al16 = ((sizeof(cx<T>) >= 16) ||
                 (std::all_of(L.fr_off.begin(), L.fr_off.end(), [](int64_t o) { return o % 2 == 0; }) &&
                  std::all_of(L.fr_pitch.begin(), L.fr_pitch.end(), [](int32_t p) { return p % 2 == 0; }))) &&
                !std::getenv("PDD_NO_TMA_ROWS");  // debug: plain loads for the patch rows
    fr_pitch = upload(L.fr_pitch, s);
    fr_r = upload(L.fr_r, s);
    fr_c = upload(L.fr_c, s);
    fr_sub = upload(L.fr_sub, s);
    tiles = upload(L.tiles, s);
    tile_frames = upload(L.tile_frames, s);
    sub_off = upload(L.sub_img_off, s);
    sub_h = upload(L.sub_h, s);
    sub_w = upload(L.sub_w, s);
    sub_pbeg = upload(L.sub_pbeg, s);
    psides = upload(L.psides, s);
    pgeom = upload(L.pgeom, s);
    sub_fr_beg = upload(L.sub_fr_beg, s);
    sub_tile_beg = upload(L.sub_tile_beg, s);
    local_map = upload(L.local_subs, s);
    if (const size_t b = stream_scratch_bytes<T>(S)) scratch.alloc(b, s);
    if (const int G = sweep_stream_ctas<T>(S); G > 0) {  // the streamed sweep's schedule
      L.schedule(G);
      pc_beg = upload(L.cta_beg, s);
      pc_pos = upload(L.cta_pos, s);
      pc_ofs = upload(L.cta_ofs, s);
      std::vector<PosRec> rec(L.cta_pos.size());
      for (size_t k = 0; k < rec.size(); ++k) {
        const int4 q = L.cta_pos[k];
        rec[k] = PosRec{q.x, q.y, q.z | (q.w << 16), L.fr_pitch[q.x], L.cta_ofs[k], L.fr_off[q.x]};
      }
      pc_rec = upload(rec, s);
    }
    fmeta_beg = upload(L.fmeta_beg, s);
    fmeta = upload(L.fmeta, s);
    fmeta_base = upload(L.fmeta_base, s);
    tps_beg = upload(L.tps_beg, s);
    tps = upload(L.tps, s);
    if (L.chained) {
      imeta_beg = upload(L.imeta_beg, s);
      imeta = upload(L.imeta, s);
      imeta_base = upload(L.imeta_base, s);
      it_r = upload(L.it_r, s);
      it_c = upload(L.it_c, s);
      it_h = upload(L.it_h, s);
      it_base = upload(L.it_base, s);
      tile_items = upload(L.tile_items, s);
      tile_item_beg = upload(L.tile_item_beg, s);
    }
    rf_part.alloc(sizeof(double) * std::max<int64_t>(L.nfr, 1));
    re_part.alloc(sizeof(double) * 2 * std::max(L.ntiles(), 1));
    sums.alloc(sizeof(double) * 3 * D);
    PDD_CUDA(cudaMemsetAsync(sums.get(), 0, sums.bytes(), s));
    ctl.alloc(sizeof(RunCtl));
    PDD_CUDA(cudaMemsetAsync(ctl.get(), 0, sizeof(RunCtl), s));
    fin_counter.alloc(sizeof(unsigned));  // segsum_finalize_kernel's last-block counter (self-resetting)
    PDD_CUDA(cudaMemsetAsync(fin_counter.get(), 0, sizeof(unsigned), s));
    rec_cap = max_iters + 2;
    rec.alloc(sizeof(double) * 2 * static_cast<size_t>(rec_cap));

    tm.mark("tables");
    upload_amplitudes(plan, data);
    tm.mark("amplitudes+l1");
    build_pins(plan, pin_ones);
    tm.mark("pins");
  }

  // Measured data -> T amplitudes in local frame order, plus the R-factor
  // denominator sum sqrt(f) (solver.cpp:80-93).
  void upload_amplitudes(const Plan& plan, const DataSpec& data) {
    cudaStream_t s = st();
    const int64_t per = SS();
    amp.alloc(sizeof(T) * std::max<int64_t>(L.nfr * per, 1));
    const size_t esz = data.kind == kAmplitudeF32 ? 4 : 8;
    DevMem neg(sizeof(unsigned long long));
    PDD_CUDA(cudaMemsetAsync(neg.get(), 0, neg.bytes(), s));
    if (data.kind == kPtyaFramesF64) {  // frames.ptya streamed from disk (ptya.hpp)
      std::vector<int32_t> g2l(static_cast<size_t>(plan.g.J()), -1);
      for (int64_t f = 0; f < L.nfr; ++f) g2l[L.fr_global[f]] = static_cast<int32_t>(f);
      DevMem dg2l = upload(g2l, s);
      DevMem stage[2];
      int64_t k = 0;
      ptya_stream_frames(static_cast<const char*>(data.ptr), plan.g.J(), S, s,
                         [&](int64_t first, int64_t count, const double* host) {
                           DevMem& dst = stage[k++ & 1];
                           const size_t bytes = sizeof(double) * static_cast<size_t>(count * per);
                           if (dst.bytes() < bytes) dst.alloc(bytes, s);
                           PDD_CUDA(cudaMemcpyAsync(dst.get(), host, bytes, cudaMemcpyHostToDevice, s));
                           PDD_CUDA(launch_scatter_amp<T>(dst.as<double>(), first, count, per,
                                                          dg2l.as<int32_t>(), amp.as<T>(),
                                                          neg.as<unsigned long long>(), s));
                         });
    } else {
    const cudaMemcpyKind kind = data.device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const char* src = static_cast<const char*>(data.ptr);
    // Pageable host input: page-lock it for the duration of the upload (DMA at
    // full PCIe/C2C rate instead of staged pageable copies).
    const size_t total = static_cast<size_t>(plan.g.J()) * per * esz;
    HostPin pin_src(data.device || total < (size_t(64) << 20) ? nullptr : src, total, s);
    auto runs = [&](int64_t f0, int64_t f1, char* dst) {  // runs of consecutive global frames
      int64_t f = f0;
      while (f < f1) {
        int64_t e = f + 1;
        while (e < f1 && L.fr_global[e] == L.fr_global[e - 1] + 1) ++e;
        PDD_CUDA(cudaMemcpyAsync(dst + (f - f0) * per * esz, src + L.fr_global[f] * per * esz, (e - f) * per * esz,
                                 kind, s));
        f = e;
      }
    };
    const bool same = (data.kind == kAmplitudeF32 && sizeof(T) == 4) || (data.kind == kAmplitudeF64 && sizeof(T) == 8);
    if (same) {  // straight into place, then the non-negativity check in place
      runs(0, L.nfr, amp.as<char>());
      PDD_CUDA(launch_convert_amp<T>(amp.get(), data.kind, amp.as<T>(), L.nfr * per, neg.as<unsigned long long>(), s));
      PDD_CUDA(cudaStreamSynchronize(s));
    } else {
      const int64_t chunk = std::max<int64_t>(1, (int64_t(256) << 20) / (per * static_cast<int64_t>(esz)));
      DevMem stage(esz * static_cast<size_t>(std::min(chunk, std::max<int64_t>(L.nfr, 1)) * per));
      for (int64_t f0 = 0; f0 < L.nfr; f0 += chunk) {
        const int64_t f1 = std::min(L.nfr, f0 + chunk);
        runs(f0, f1, stage.as<char>());
        PDD_CUDA(launch_convert_amp<T>(stage.get(), data.kind, amp.as<T>() + f0 * per, (f1 - f0) * per,
                                       neg.as<unsigned long long>(), s));
        PDD_CUDA(cudaStreamSynchronize(s));  // stage reuse
      }
    }
    pin_src.done();
    }
    unsigned long long nneg = 0;
    PDD_CUDA(cudaMemcpyAsync(&nneg, neg.get(), sizeof(nneg), cudaMemcpyDeviceToHost, s));
    PDD_CUDA(cudaStreamSynchronize(s));
    if (nneg) throw InvalidArgument("FrameStack: negative intensity");
    // l1 = sum_d sum_j sum_i sqrt(f)
    DevMem fs(sizeof(double) * std::max<int64_t>(L.nfr, 1));
    PDD_CUDA(launch_frame_sums<T>(amp.as<T>(), L.nfr, per, fs.as<double>(), s));
    PDD_CUDA(launch_segsum(fs.as<double>(), 1, 0, sub_fr_beg.as<int64_t>(), L.nls(), local_map.as<int>(),
                           rf_sub(), nullptr, s));
    if (comm) comm->allreduce_sum_f64(rf_sub(), D, s);
    std::vector<double> per_sub(D);
    PDD_CUDA(cudaMemcpyAsync(per_sub.data(), rf_sub(), sizeof(double) * D, cudaMemcpyDeviceToHost, s));
    PDD_CUDA(cudaStreamSynchronize(s));
    l1 = 0.0;
    for (double x : per_sub) l1 += x;
    PDD_CUDA(cudaMemsetAsync(sums.get(), 0, sums.bytes(), s));
  }

  // Pixels never covered by a window, plus the caller's vacuum mask
  // (solver.cpp:43-48, 64-69): coverage from the gather tiles on the device.
  void build_pins(const Plan& plan, const double* pin_ones) {
    cudaStream_t s = st();
    pin_dev.alloc(std::max<int64_t>(L.img_elems, 1));
    DevMem user;
    // Raster block plans: a subdomain's own windows tile its rectangle, so the
    // global coverage (scan.cpp:36-44) is zero exactly where the local one is.
    // General plans take the global coverage from the host.
    const bool host_cov = !plan.raster_blocks;
    if (pin_ones || host_cov) {
      std::vector<int32_t> cov;
      if (host_cov) cov = scan_coverage(plan.g);
      std::vector<uint8_t> up(static_cast<size_t>(L.img_elems));
      for (int ld = 0; ld < L.nls(); ++ld) {
        const Rect& sub = plan.subs[L.local_subs[ld]];
        for (int64_t r = 0; r < sub.h(); ++r)
          for (int64_t c = 0; c < sub.w(); ++c) {
            const int64_t gi = (sub.r0 + r) * plan.g.W + sub.c0 + c;
            up[L.sub_img_off[ld] + r * sub.w() + c] =
                (pin_ones && pin_ones[gi] > 0.5) || (host_cov && cov[gi] == 0);
          }
      }
      user = upload(up, s);
    }
    PDD_CUDA(launch_pins(tiles.as<int4>(), L.ntiles(), L.tile_h, L.tile_w, tile_frames.as<int32_t>(), fr_r.as<int32_t>(),
                         fr_c.as<int32_t>(), S, sub_off.as<int64_t>(), sub_h.as<int32_t>(), sub_w.as<int32_t>(),
                         (pin_ones || host_cov) ? user.as<uint8_t>() : nullptr, pin_dev.as<uint8_t>(), s));
    PDD_CUDA(cudaStreamSynchronize(s));
  }
  const uint8_t* pins_of(int ld) const { return pin_dev.as<uint8_t>() + L.sub_img_off[ld]; }

  FrameArgs<T> frame_args() const {
    FrameArgs<T> a;
    a.nframes = static_cast<int>(L.nfr);
    a.tw = tw.as<cx<T>>();
    a.off = fr_off.as<int64_t>();
    a.pitch = fr_pitch.as<int32_t>();
    a.amp = amp.as<T>();
    a.scale = static_cast<T>(1.0 / static_cast<double>(S));
    a.rows_al16 = rows_al16 ? 1 : 0;
    a.img_elems = L.img_elems;
    a.scratch = scratch.as<cx<T>>();
    return a;
  }

  // The streamed sweep's pieces / the update gather's partial images (chained layouts only).
  void set_pieces(FrameArgs<T>& a) const {
    if (!L.ncta) return;
    a.cta_beg = pc_beg.as<int32_t>();
    a.ncta = L.ncta;
    a.pc_pos = pc_pos.as<int4>();
    a.pc_ofs = pc_ofs.as<int64_t>();
    a.pc_rec = pc_rec.as<PosRec>();
  }
  void set_pieces(GatherArgs<T>& g) const {
    if (!L.chained) return;
    g.mbeg = imeta_beg.as<int32_t>();
    g.meta = imeta.as<int4>();
    g.mbase = imeta_base.as<int64_t>();
    g.tile_items = tile_items.as<int32_t>();
    g.tile_item_beg = tile_item_beg.as<int32_t>();
    g.it_r = it_r.as<int32_t>();
    g.it_c = it_c.as<int32_t>();
    g.it_h = it_h.as<int32_t>();
    g.it_base = it_base.as<int64_t>();
  }

  GatherArgs<T> gather_args(int mode) const {
    GatherArgs<T> g;
    g.mode = mode;
    g.ntiles = L.ntiles();
    g.tile_h = L.tile_h;
    g.tile_w = L.tile_w;
    g.tiles = tiles.as<int4>();
    g.tile_frames = tile_frames.as<int32_t>();
    g.fr_r = fr_r.as<int32_t>();
    g.fr_c = fr_c.as<int32_t>();
    g.fr_sub = fr_sub.as<int32_t>();
    g.S = S;
    g.sub_off = sub_off.as<int64_t>();
    g.sub_h = sub_h.as<int32_t>();
    g.sub_w = sub_w.as<int32_t>();
    g.sub_pbeg = sub_pbeg.as<int32_t>();
    g.ps = psides.as<PairSide>();
    // covering frames, flattened (set_pieces switches to the pieces); chained
    // layouts keep no flattened frame lists: the kernel then walks tile_frames
    g.mbeg = L.fmeta_beg.empty() ? nullptr : fmeta_beg.as<int32_t>();
    g.meta = fmeta.as<int4>();
    g.mbase = fmeta_base.as<int64_t>();
    g.tps_beg = tps_beg.as<int32_t>();
    g.tps = tps.as<int32_t>();
    return g;
  }

  // Per-subdomain R-factor numerators from rf_part (+ all-reduce over ranks).
  void reduce_rf(bool gated) {
    cudaStream_t s = st();
    if (comm) PDD_CUDA(cudaMemsetAsync(rf_sub(), 0, sizeof(double) * D, s));
    PDD_CUDA(launch_segsum(rf_part.as<double>(), 1, 0, sub_fr_beg.as<int64_t>(), L.nls(), local_map.as<int>(),
                           rf_sub(), gated ? skipA() : nullptr, s));
    if (comm) comm->allreduce_sum_f64(rf_sub(), D, s);
  }
  // reduce + finalize of the iteration's R-factor / RE.  Single-rank solvers
  // run them as one launch each (segsum_finalize_kernel); with a communicator
  // the all-reduce sits between the sums and the finalize step.
  bool fused_finalize() const { return !comm && D <= fused_finalize_max_subdomains(); }
  void reduce_rf_finalize() {
    cudaStream_t s = st();
    if (!fused_finalize()) {
      reduce_rf(true);
      PDD_CUDA(launch_rf_finalize(ctlp(), rf_sub(), D, rec.template as<double>(), s));
      return;
    }
    PDD_CUDA(launch_segsum_finalize(1, rf_part.as<double>(), sub_fr_beg.as<int64_t>(), L.nls(), local_map.as<int>(),
                                    rf_sub(), nullptr, skipA(), fin_counter.as<unsigned>(), ctlp(), D,
                                    rec.template as<double>(), s));
  }
  void reduce_re_finalize() {
    cudaStream_t s = st();
    if (!fused_finalize()) {
      reduce_re();
      PDD_CUDA(launch_re_finalize(ctlp(), diff_sub(), norm_sub(), D, rec.template as<double>(), s));
      return;
    }
    PDD_CUDA(launch_segsum_finalize(2, re_part.as<double>(), sub_tile_beg.as<int64_t>(), L.nls(), local_map.as<int>(),
                                    diff_sub(), norm_sub(), skipB(), fin_counter.as<unsigned>(), ctlp(), D,
                                    rec.template as<double>(), s));
  }
  void reduce_re() {
    cudaStream_t s = st();
    if (comm) PDD_CUDA(cudaMemsetAsync(diff_sub(), 0, sizeof(double) * 2 * D, s));
    PDD_CUDA(launch_segsum(re_part.as<double>(), 2, 0, sub_tile_beg.as<int64_t>(), L.nls(), local_map.as<int>(),
                           diff_sub(), skipB(), s));
    PDD_CUDA(launch_segsum(re_part.as<double>(), 2, 1, sub_tile_beg.as<int64_t>(), L.nls(), local_map.as<int>(),
                           norm_sub(), skipB(), s));
    if (comm) comm->allreduce_sum_f64(diff_sub(), 2 * D, s);
  }

  ~RankData() {
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }

  // The overlap consensus of iteration n+1 needs only u^n and Lambda^n, so
  // it runs as a branch forked off the iteration's start, concurrent with the
  // frame pass (K1), and joins before the update gather that consumes v.
  // Its skip flag is the gate's snapshot of earlier iterations' stops (skipC):
  // a stop decided inside this iteration only discards what the branch wrote.
  void fork_consensus(const cx<T>* u, const cx<T>* lam, cx<T>* sbuf, cx<T>* v) {
    if (!ev_fork) {
      PDD_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      PDD_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    PDD_CUDA(cudaEventRecord(ev_fork, st()));
    PDD_CUDA(cudaStreamWaitEvent(side.get(), ev_fork, 0));
    consensus(u, lam, sbuf, v, skipC(), side.get());
    PDD_CUDA(cudaEventRecord(ev_join, side.get()));
  }
  void join_consensus() { PDD_CUDA(cudaStreamWaitEvent(st(), ev_join, 0)); }

  // v = (s_1 + s_2)/2 with s_side = u_side + Lambda_side exchanged across ranks.
  void consensus(const cx<T>* u, const cx<T>* lam, cx<T>* sbuf, cx<T>* v, const int* skip,
                 cudaStream_t s = nullptr) {
    if (!s) s = st();
    const int np = static_cast<int>(L.lpairs.size());
    PDD_CUDA(launch_pack<T>(pgeom.as<PairGeom>(), np, L.max_pair_pix, u, lam, sbuf, skip, s));
    if (comm && !L.exch.empty()) {
      comm->group_start();
      for (const auto& e : L.exch) {
        const PairGeom& pg = L.pgeom[e.lp];
        const int64_t n = static_cast<int64_t>(pg.h) * pg.w;
        comm->send(sbuf + pg.s_off + e.my_side * n, sizeof(cx<T>) * n, e.peer, s);
        comm->recv(sbuf + pg.s_off + (1 - e.my_side) * n, sizeof(cx<T>) * n, e.peer, s);
      }
      comm->group_end();
    }
    PDD_CUDA(launch_vstep<T>(pgeom.as<PairGeom>(), np, L.max_pair_pix, sbuf, v, skip, s));
  }

  StateLayout state_layout(const Plan& plan) const {
    StateLayout sl;
    sl.local_subs = L.local_subs;
    for (int ld = 0; ld < L.nls(); ++ld) {
      sl.sub_h.push_back(L.sub_h[ld]);
      sl.sub_w.push_back(L.sub_w[ld]);
      sl.sub_frames.push_back(L.sub_fr_beg[ld + 1] - L.sub_fr_beg[ld]);
    }
    sl.local_pairs = L.lpairs;
    for (const auto& pg : L.pgeom) {
      sl.pair_h.push_back(pg.h);
      sl.pair_w.push_back(pg.w);
    }
    sl.S = S;
    return sl;
  }

  // merge (ddplan.cpp:104-121) of the device sub-solutions into a host image.
  // scratch: optional device buffer free at this point (>= H*W complex128),
  // e.g. the nonblind back-projection scratch -- a fresh 1 GB cudaMalloc here
  // cost 1-90 ms (and ~0.4 s on a process's first large allocation).
  void merge_to_host(const Plan& plan, const cx<T>* u, double* out, void* scratch = nullptr,
                     size_t scratch_bytes = 0) {
    if (L.nls() != plan.D) throw InvalidArgument("merge: this rank does not own every subdomain");
    cudaStream_t s = st();
    std::vector<int64_t> rect;
    for (const auto& r : plan.subs) {
      rect.push_back(r.r0);
      rect.push_back(r.r1);
      rect.push_back(r.c0);
      rect.push_back(r.c1);
    }
    DevMem drect = upload(rect, s);
    const int64_t n = plan.g.H * plan.g.W;
    SetupTimer tm;
    DevMem img;
    cx<double>* dst = static_cast<cx<double>*>(scratch);
    if (!dst || scratch_bytes < sizeof(cx<double>) * n) {
      img.alloc(sizeof(cx<double>) * n);
      dst = img.as<cx<double>>();
    }
    tm.mark("merge: alloc");
    PDD_CUDA(launch_merge<T>(u, drect.as<int64_t>(), sub_off.as<int64_t>(), plan.D, plan.g.H, plan.g.W, dst, s));
    download_c128<double>(dst, n, out, s);
    tm.mark("merge: kernel+download");
  }

  void reset_ctl(int iter, int max_iters, int rule, double tol_rf, double tol_re) {
    RunCtl c{};
    c.iter = iter;
    c.max_iters = max_iters;
    c.rule = rule;
    c.tol_rf = tol_rf;
    c.tol_re = tol_re;
    c.l1 = l1;
    c.rec_cap = rec_cap;
    PDD_CUDA(cudaMemcpyAsync(ctl.get(), &c, sizeof(c), cudaMemcpyHostToDevice, st()));
    PDD_CUDA(cudaStreamSynchronize(st()));
  }
  RunCtl read_ctl() {
    RunCtl c{};
    PDD_CUDA(cudaMemcpyAsync(&c, ctl.get(), sizeof(c), cudaMemcpyDeviceToHost, st()));
    PDD_CUDA(cudaStreamSynchronize(st()));
    return c;
  }
};

}  // namespace pdd
