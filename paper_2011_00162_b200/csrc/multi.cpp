// One handle driving G ranks of one process: the reference's worker pool
// (parallel.hpp:14-90; NonblindConfig::threads, solver.hpp:25) mapped onto
// GPUs (SURVEY.md sec. 8(b) "Threading").
//
// Rank r owns subdomains d with floor(d * G / D) == r (layout.hpp owner_of),
// runs on devices[r] with its own stream, CUDA graphs and solver state, and is
// driven by its own host thread; the ranks talk through a Comm exactly as the
// one-process-per-GPU mode does -- NCCL when the devices are distinct,
// otherwise the host-staged in-process transport (transport.cpp), which lets
// several ranks share one device (the multi-rank code paths on one GPU).
// Iterates are bit-identical for every G at fixed D (single-owner exact
// reductions, per-subdomain schedules).
//
// State crosses this wrapper in the single-handle (global) layout of
// ptychodd_cuda.h: subdomains in ascending d, frames in frames_of order,
// overlap variables per pair in ascending p (Lambda side 0 from the owner of
// d1, side 1 from the owner of d2).
#include <array>
#include <condition_variable>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>

#include "device.hpp"
#include "engine.hpp"
#include "layout.hpp"

namespace pdd {
namespace {

// One persistent worker thread per rank (bound to its device once).
class RankThreads {
 public:
  explicit RankThreads(const std::vector<int>& devices) : n_(static_cast<int>(devices.size())), err_(n_) {
    for (int r = 0; r < n_; ++r) th_.emplace_back([this, r, dev = devices[r]] { loop(r, dev); });
  }
  ~RankThreads() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      quit_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // f(r) on every rank concurrently; the first failure in rank order is rethrown.
  void all(const std::function<void(int)>& f) {
    {
      std::unique_lock<std::mutex> lock(mu_);
      job_ = &f;
      done_ = 0;
      for (auto& e : err_) e = nullptr;
      ++gen_;
    }
    cv_.notify_all();
    {
      std::unique_lock<std::mutex> lock(mu_);
      done_cv_.wait(lock, [&] { return done_ == n_; });
      job_ = nullptr;
    }
    for (auto& e : err_)
      if (e) std::rethrow_exception(e);
  }

 private:
  void loop(int r, int dev) {
    uint64_t seen = 0;
    const cudaError_t bind = cudaSetDevice(dev);
    for (;;) {
      const std::function<void(int)>* job = nullptr;
      {
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [&] { return gen_ != seen; });
        seen = gen_;
        if (quit_) return;
        job = job_;
      }
      std::exception_ptr e;
      try {
        if (bind != cudaSuccess) throw CudaError(std::string("cudaSetDevice: ") + cudaGetErrorString(bind));
        (*job)(r);
      } catch (...) {
        e = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lock(mu_);
        err_[r] = e;
        ++done_;
      }
      done_cv_.notify_all();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  uint64_t gen_ = 0;
  int done_ = 0;
  bool quit_ = false;
  std::vector<std::exception_ptr> err_;
};

// Global (single-handle) state offsets of a plan.
struct GlobalLayout {
  StateLayout sl;
  std::vector<int64_t> img_off, fr_off, pair_off;  // per d (elements), per d (frames), per p (elements)
  int64_t img_elems = 0, frames = 0, pair_elems = 0;
  explicit GlobalLayout(const Plan& plan) {
    sl.S = plan.g.s;
    for (int d = 0; d < plan.D; ++d) {
      sl.local_subs.push_back(d);
      sl.sub_h.push_back(plan.subs[d].h());
      sl.sub_w.push_back(plan.subs[d].w());
      sl.sub_frames.push_back(static_cast<int64_t>(plan.frames_of[d].size()));
      img_off.push_back(img_elems);
      fr_off.push_back(frames);
      img_elems += plan.subs[d].area();
      frames += static_cast<int64_t>(plan.frames_of[d].size());
    }
    for (size_t p = 0; p < plan.overlaps.size(); ++p) {
      sl.local_pairs.push_back(static_cast<int>(p));
      sl.pair_h.push_back(plan.overlaps[p].region.h());
      sl.pair_w.push_back(plan.overlaps[p].region.w());
      pair_off.push_back(pair_elems);
      pair_elems += plan.overlaps[p].region.area();
    }
  }
};

// Per-rank overlap variables (rank-local pair order) <-> global arrays.
// complex128 values as interleaved doubles.
struct PairMap {
  const Plan* plan;
  const GlobalLayout* g;
  int D, G;
  // rank-local element offsets of each local pair
  static std::vector<int64_t> local_offsets(const StateLayout& l) {
    std::vector<int64_t> o;
    int64_t a = 0;
    for (size_t k = 0; k < l.local_pairs.size(); ++k) {
      o.push_back(a);
      a += l.pair_h[k] * l.pair_w[k];
    }
    o.push_back(a);
    return o;
  }
  // v: taken from the rank owning d1; Lambda side s from the owner of d_s
  void gather(int r, const StateLayout& l, const double* v_r, const double* lam_r, double* v, double* lam) const {
    const auto lo = local_offsets(l);
    const int64_t lv = lo.back();
    for (size_t k = 0; k < l.local_pairs.size(); ++k) {
      const int p = l.local_pairs[k];
      const auto& pr = plan->overlaps[p];
      const int64_t n = pr.region.area(), go = g->pair_off[p];
      if (v && owner_of(pr.d1, D, G) == r) std::copy(v_r + 2 * lo[k], v_r + 2 * (lo[k] + n), v + 2 * go);
      if (lam) {
        // rank-local Lambda: per local pair, side 0 then side 1 (2n elements)
        const double* src = lam_r + 2 * (2 * lo[k]);
        (void)lv;
        for (int side = 0; side < 2; ++side)
          if (owner_of(side ? pr.d2 : pr.d1, D, G) == r)
            std::copy(src + 2 * side * n, src + 2 * (side + 1) * n, lam + 2 * (2 * go + side * n));
      }
    }
  }
  void scatter(const StateLayout& l, const double* v, const double* lam, double* v_r, double* lam_r) const {
    const auto lo = local_offsets(l);
    for (size_t k = 0; k < l.local_pairs.size(); ++k) {
      const int p = l.local_pairs[k];
      const int64_t n = plan->overlaps[p].region.area(), go = g->pair_off[p];
      if (v) std::copy(v + 2 * go, v + 2 * (go + n), v_r + 2 * lo[k]);
      if (lam) std::copy(lam + 2 * (2 * go), lam + 2 * (2 * go + 2 * n), lam_r + 2 * (2 * lo[k]));
    }
  }
};

int64_t pair_elems_of(const StateLayout& l) {
  int64_t a = 0;
  for (size_t k = 0; k < l.local_pairs.size(); ++k) a += l.pair_h[k] * l.pair_w[k];
  return a;
}

// merge (ddplan.cpp:104-121) of global sub-solutions on the host.
void merge_host(const Plan& plan, const GlobalLayout& g, const double* u, double* out) {
  const int64_t H = plan.g.H, W = plan.g.W;
  std::vector<double> cnt(static_cast<size_t>(H * W), 0.0);
  std::fill(out, out + 2 * H * W, 0.0);
  for (int d = 0; d < plan.D; ++d) {
    const Rect& s = plan.subs[d];
    const double* ud = u + 2 * g.img_off[d];
    for (int64_t r = 0; r < s.h(); ++r)
      for (int64_t c = 0; c < s.w(); ++c) {
        const int64_t gi = (s.r0 + r) * W + s.c0 + c, li = r * s.w() + c;
        out[2 * gi] += ud[2 * li];
        out[2 * gi + 1] += ud[2 * li + 1];
        cnt[gi] += 1.0;
      }
  }
  for (int64_t i = 0; i < H * W; ++i) {
    if (cnt[i] > 0.0) {
      out[2 * i] /= cnt[i];
      out[2 * i + 1] /= cnt[i];
    } else {
      out[2 * i] = 1.0;
      out[2 * i + 1] = 0.0;
    }
  }
}

template <class Gpu>
struct RankSet {
  std::vector<int> devices;
  std::vector<std::unique_ptr<Comm>> comms;
  std::vector<std::unique_ptr<Gpu>> ranks;
  std::unique_ptr<RankThreads> pool;
  int G = 0;

  template <class Make>
  void build(const Plan& plan, const std::vector<int>& devs, Make&& make) {
    devices = devs;
    G = static_cast<int>(devs.size());
    if (G < 1) throw InvalidArgument("multi-GPU solver: at least one device");
    if (G > plan.D) throw InvalidArgument("multi-GPU solver: more ranks than subdomains (D = " +
                                          std::to_string(plan.D) + ")");
    bool distinct = true;
    for (int a = 0; a < G; ++a)
      for (int b = a + 1; b < G; ++b) distinct = distinct && devs[a] != devs[b];
    char id[128];
    if (G == 1) {
      // a single rank needs no transport
    } else if (distinct) {
      nccl_unique_id(id);
    } else {
      host_hub_id(id);
    }
    comms.resize(G);
    ranks.resize(G);
    pool = std::make_unique<RankThreads>(devs);
    pool->all([&](int r) {
      if (G > 1) comms[r] = distinct ? make_nccl_comm(id, r, G, devs[r]) : make_host_comm(id, r, G);
      ranks[r] = make(devs[r], comms[r].get());
    });
  }
  ~RankSet() {
    if (pool)  // each rank (and its communicator) torn down on its own thread
      pool->all([&](int r) {
        ranks[r].reset();
        comms[r].reset();
      });
    pool.reset();
  }
  // run on every rank's thread with its device and allocation stream current
  void all(const std::function<void(int)>& f) {
    pool->all([&](int r) {
      DeviceGuard dg(devices[r]);
      AllocStream as(static_cast<cudaStream_t>(ranks[r]->stream()));
      f(r);
    });
  }
};

class MultiNonblind final : public NonblindGpu {
 public:
  MultiNonblind(const Plan& plan, const DataSpec& data, const double* probe, const NonblindConfig& cfg,
                const double* pin_ones, int dtype, const std::vector<int>& devices)
      : plan_(plan), g_(plan) {
    R_.build(plan, devices, [&](int dev, Comm* c) {
      return make_nonblind(plan, data, probe, cfg, pin_ones, dtype, dev, c);
    });
  }
  const StateLayout& layout() const override { return g_.sl; }
  void init_state() override { R_.all([&](int r) { R_.ranks[r]->init_state(); }); }
  void step(bool store_z) override { R_.all([&](int r) { R_.ranks[r]->step(store_z); }); }
  RunRecords run(const RecordFn& on_record) override {
    std::vector<RunRecords> rr(R_.G);
    // records are identical on every rank (all-reduced): rank 0 streams them
    R_.all([&](int r) { rr[r] = R_.ranks[r]->run(r == 0 ? on_record : RecordFn{}); });
    RunRecords out = rr[0];
    for (int r = 1; r < R_.G; ++r)
      for (size_t n = 0; n < out.t_ms.size() && n < rr[r].t_ms.size(); ++n)
        out.t_ms[n] = std::max(out.t_ms[n], rr[r].t_ms[n]);
    return out;
  }
  void iterate(int n) override { R_.all([&](int r) { R_.ranks[r]->iterate(n); }); }
  double iterate_timed(int n) override {
    std::vector<double> ms(R_.G);
    R_.all([&](int r) { ms[r] = R_.ranks[r]->iterate_timed(n); });
    return *std::max_element(ms.begin(), ms.end());
  }
  void profile(int n, double* ms) override {
    std::vector<std::array<double, 3>> m(R_.G);
    R_.all([&](int r) { R_.ranks[r]->profile(n, m[r].data()); });
    for (int k = 0; k < 3; ++k) {
      ms[k] = 0.0;
      for (int r = 0; r < R_.G; ++r) ms[k] = std::max(ms[k], m[r][k]);
    }
  }
  double last_rf() override {
    double rf = 0.0;
    R_.all([&](int r) {
      if (r == 0) rf = R_.ranks[0]->last_rf();
    });
    return rf;
  }
  void get_state(double* u, double* z, double* gamma, double* v, double* lam, int64_t* iteration) override {
    const PairMap pm{&plan_, &g_, plan_.D, R_.G};
    std::vector<int64_t> it(R_.G);
    R_.all([&](int r) {
      const StateLayout& l = R_.ranks[r]->layout();
      const int d0 = l.local_subs.front();
      const int64_t S2 = g_.sl.S * g_.sl.S, np = pair_elems_of(l);
      std::vector<double> v_r(v ? 2 * std::max<int64_t>(np, 1) : 0), lam_r(lam ? 4 * std::max<int64_t>(np, 1) : 0);
      R_.ranks[r]->get_state(u ? u + 2 * g_.img_off[d0] : nullptr, z ? z + 2 * S2 * g_.fr_off[d0] : nullptr,
                             gamma ? gamma + 2 * S2 * g_.fr_off[d0] : nullptr, v ? v_r.data() : nullptr,
                             lam ? lam_r.data() : nullptr, &it[r]);
      pm.gather(r, l, v_r.data(), lam_r.data(), v, lam);  // disjoint global ranges per rank
    });
    if (iteration) *iteration = it[0];
  }
  void set_state(const double* u, const double* z, const double* gamma, const double* v, const double* lam,
                 int64_t iteration) override {
    const PairMap pm{&plan_, &g_, plan_.D, R_.G};
    R_.all([&](int r) {
      const StateLayout& l = R_.ranks[r]->layout();
      const int d0 = l.local_subs.front();
      const int64_t S2 = g_.sl.S * g_.sl.S, np = pair_elems_of(l);
      std::vector<double> v_r(v ? 2 * std::max<int64_t>(np, 1) : 0), lam_r(lam ? 4 * std::max<int64_t>(np, 1) : 0);
      pm.scatter(l, v, lam, v_r.data(), lam_r.data());
      R_.ranks[r]->set_state(u ? u + 2 * g_.img_off[d0] : nullptr, z ? z + 2 * S2 * g_.fr_off[d0] : nullptr,
                             gamma ? gamma + 2 * S2 * g_.fr_off[d0] : nullptr, v ? v_r.data() : nullptr,
                             lam ? lam_r.data() : nullptr, iteration);
    });
  }
  void forward_frames(double* au) override {
    R_.all([&](int r) {
      const int d0 = R_.ranks[r]->layout().local_subs.front();
      R_.ranks[r]->forward_frames(au + 2 * g_.sl.S * g_.sl.S * g_.fr_off[d0]);
    });
  }
  double lagrangian() override {
    std::vector<double> L(R_.G);
    R_.all([&](int r) { L[r] = R_.ranks[r]->lagrangian(); });  // all-reduced: identical on every rank
    return L[0];
  }
  std::vector<double> lagrangian_history() const override { return R_.ranks[0]->lagrangian_history(); }
  void merged(double* out) override {
    std::vector<double> u(2 * static_cast<size_t>(g_.img_elems));
    get_state(u.data(), nullptr, nullptr, nullptr, nullptr, nullptr);
    merge_host(plan_, g_, u.data(), out);
  }
  void sync() override { R_.all([&](int r) { R_.ranks[r]->sync(); }); }
  void* stream() const override { return R_.ranks[0]->stream(); }
  int64_t kernel_launches_per_iteration() const override { return R_.ranks[0]->kernel_launches_per_iteration(); }

 private:
  Plan plan_;
  GlobalLayout g_;
  RankSet<NonblindGpu> R_;
};

class MultiBlind final : public BlindGpu {
 public:
  MultiBlind(const Plan& plan, const DataSpec& data, const BlindConfig& cfg, const double* mask,
             const double* pin_ones, int dtype, const std::vector<int>& devices)
      : plan_(plan), g_(plan) {
    R_.build(plan, devices, [&](int dev, Comm* c) {
      return make_blind(plan, data, cfg, mask, pin_ones, dtype, dev, c);
    });
  }
  const StateLayout& layout() const override { return g_.sl; }
  void init_state(const double* w0) override { R_.all([&](int r) { R_.ranks[r]->init_state(w0); }); }
  void step(bool store_z) override { R_.all([&](int r) { R_.ranks[r]->step(store_z); }); }
  RunRecords run(const RecordFn& on_record) override {
    std::vector<RunRecords> rr(R_.G);
    // records are identical on every rank (all-reduced): rank 0 streams them
    R_.all([&](int r) { rr[r] = R_.ranks[r]->run(r == 0 ? on_record : RecordFn{}); });
    RunRecords out = rr[0];
    for (int r = 1; r < R_.G; ++r)
      for (size_t n = 0; n < out.t_ms.size() && n < rr[r].t_ms.size(); ++n)
        out.t_ms[n] = std::max(out.t_ms[n], rr[r].t_ms[n]);
    return out;
  }
  void iterate(int n) override { R_.all([&](int r) { R_.ranks[r]->iterate(n); }); }
  double iterate_timed(int n) override {
    std::vector<double> ms(R_.G);
    R_.all([&](int r) { ms[r] = R_.ranks[r]->iterate_timed(n); });
    return *std::max_element(ms.begin(), ms.end());
  }
  void profile(int n, double* ms) override {
    std::vector<std::array<double, 3>> m(R_.G);
    R_.all([&](int r) { R_.ranks[r]->profile(n, m[r].data()); });
    for (int k = 0; k < 3; ++k) {
      ms[k] = 0.0;
      for (int r = 0; r < R_.G; ++r) ms[k] = std::max(ms[k], m[r][k]);
    }
  }
  void get_state(double* w, double* w_copies, double* delta, double* u, double* z, double* gamma, double* v,
                 double* lam, int64_t* iteration) override {
    const PairMap pm{&plan_, &g_, plan_.D, R_.G};
    std::vector<int64_t> it(R_.G);
    R_.all([&](int r) {
      const StateLayout& l = R_.ranks[r]->layout();
      const int d0 = l.local_subs.front();
      const int64_t S2 = g_.sl.S * g_.sl.S, np = pair_elems_of(l);
      std::vector<double> v_r(v ? 2 * std::max<int64_t>(np, 1) : 0), lam_r(lam ? 4 * std::max<int64_t>(np, 1) : 0);
      R_.ranks[r]->get_state(r == 0 ? w : nullptr, w_copies ? w_copies + 2 * S2 * d0 : nullptr,
                             delta ? delta + 2 * S2 * d0 : nullptr, u ? u + 2 * g_.img_off[d0] : nullptr,
                             z ? z + 2 * S2 * g_.fr_off[d0] : nullptr, gamma ? gamma + 2 * S2 * g_.fr_off[d0] : nullptr,
                             v ? v_r.data() : nullptr, lam ? lam_r.data() : nullptr, &it[r]);
      pm.gather(r, l, v_r.data(), lam_r.data(), v, lam);
    });
    if (iteration) *iteration = it[0];
  }
  void set_state(const double* w, const double* w_copies, const double* delta, const double* u, const double* z,
                 const double* gamma, const double* v, const double* lam, int64_t iteration) override {
    const PairMap pm{&plan_, &g_, plan_.D, R_.G};
    R_.all([&](int r) {
      const StateLayout& l = R_.ranks[r]->layout();
      const int d0 = l.local_subs.front();
      const int64_t S2 = g_.sl.S * g_.sl.S, np = pair_elems_of(l);
      std::vector<double> v_r(v ? 2 * std::max<int64_t>(np, 1) : 0), lam_r(lam ? 4 * std::max<int64_t>(np, 1) : 0);
      pm.scatter(l, v, lam, v_r.data(), lam_r.data());
      R_.ranks[r]->set_state(w, w_copies ? w_copies + 2 * S2 * d0 : nullptr, delta ? delta + 2 * S2 * d0 : nullptr,
                             u ? u + 2 * g_.img_off[d0] : nullptr, z ? z + 2 * S2 * g_.fr_off[d0] : nullptr,
                             gamma ? gamma + 2 * S2 * g_.fr_off[d0] : nullptr, v ? v_r.data() : nullptr,
                             lam ? lam_r.data() : nullptr, iteration);
    });
  }
  void get_probe(double* probe, double* probe_fourier, double* mask, double* w0) override {
    R_.all([&](int r) {
      if (r == 0) R_.ranks[0]->get_probe(probe, probe_fourier, mask, w0);
    });
  }
  void merged(double* out) override {
    std::vector<double> u(2 * static_cast<size_t>(g_.img_elems));
    get_state(nullptr, nullptr, nullptr, u.data(), nullptr, nullptr, nullptr, nullptr, nullptr);
    merge_host(plan_, g_, u.data(), out);
  }
  void sync() override { R_.all([&](int r) { R_.ranks[r]->sync(); }); }
  void* stream() const override { return R_.ranks[0]->stream(); }
  int64_t kernel_launches_per_iteration() const override { return R_.ranks[0]->kernel_launches_per_iteration(); }

 private:
  Plan plan_;
  GlobalLayout g_;
  RankSet<BlindGpu> R_;
};

}  // namespace

std::unique_ptr<NonblindGpu> make_nonblind_multi(const Plan& plan, const DataSpec& data, const double* probe,
                                                 const NonblindConfig& cfg, const double* pin_ones, int dtype,
                                                 const std::vector<int>& devices) {
  return std::make_unique<MultiNonblind>(plan, data, probe, cfg, pin_ones, dtype, devices);
}

std::unique_ptr<BlindGpu> make_blind_multi(const Plan& plan, const DataSpec& data, const BlindConfig& cfg,
                                           const double* mask, const double* pin_ones, int dtype,
                                           const std::vector<int>& devices) {
  return std::make_unique<MultiBlind>(plan, data, cfg, mask, pin_ones, dtype, devices);
}

}  // namespace pdd
