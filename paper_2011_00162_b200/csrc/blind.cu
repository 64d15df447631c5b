// Blind OD²BP driver: BlindSolver (proj/src/blind.cpp) on the GPU.
//
// Per iteration (blind.cpp:194-296), one graph node chain per rank:
//   gate -> frame BLIND pass (B(W_d^n, u^n) -> prox -> Gamma, q_j = IFFT(resid);
//           plus the shared-probe R-factor of u^n, blind.cpp:320-332)
//        -> rf_finalize
//        -> w-step: avg_d (Delta_d + W_d) -> FFT -> support mask -> IFFT
//           (blind.cpp:200-206, 159-167)
//        -> v-step (pack / [NCCL] / vstep)
//        -> probe reduction sum_j conj(u|w_j) q_j, sum_j |u|w_j|^2 (chunked,
//           ordered) -> W_d^{n+1}, Delta_d^{n+1} (blind.cpp:246-251, 276-277)
//        -> gather: u^{n+1} with conj(W^{n+1}) q_j, |W^{n+1}|^2, gamma-prox
//           anchor, Lambda update, RE partials (blind.cpp:253-272, 282-292)
//        -> re_finalize
// The reference recomputes 4 FFTs per frame; here 3 (the W- and u-steps share
// q_j).  The frame pass runs before the w-step (it does
// not depend on w^{n+1}) so it can use w^n for the lagged R-factor.
#include <algorithm>

#include "blind_kernels.hpp"
#include "common.cuh"
#include "ops.hpp"

namespace pdd {

void BlindConfig::validate(int64_t s, const double* mask) const {  // blind.cpp:30-44
  if (!(epsilon > 0.0 && epsilon < 1.0)) throw InvalidArgument("stagm: epsilon must lie in (0,1)");
  if (eta <= 0.0 || r <= 0.0 || mu <= 0.0 || gamma <= 0.0)
    throw InvalidArgument("BlindConfig: eta, r, mu, gamma must be > 0");
  if (max_iters < 1) throw InvalidArgument("BlindConfig: max_iters >= 1");
  if (tol_rf <= 0.0 || tol_re <= 0.0) throw InvalidArgument("BlindConfig: tolerances must be > 0");
  if (mask)
    for (int64_t i = 0; i < s * s; ++i)
      if (mask[i] != 0.0 && mask[i] != 1.0) throw InvalidArgument("BlindConfig: support mask entries must be 0 or 1");
}

namespace {

double freq_radius(int64_t k, int64_t l, int64_t side) {  // blind.cpp:22-27
  const double kk = static_cast<double>(std::min(k, side - k));
  const double ll = static_cast<double>(std::min(l, side - l));
  return std::sqrt(kk * kk + ll * ll);
}

}  // namespace

std::vector<double> disk_mask(int64_t side, double radius) {  // blind.cpp:46-52
  std::vector<double> m(static_cast<size_t>(side * side), 0.0);
  for (int64_t k = 0; k < side; ++k)
    for (int64_t l = 0; l < side; ++l)
      if (freq_radius(k, l, side) <= radius) m[k * side + l] = 1.0;
  return m;
}

// estimate_support_mask (blind.cpp:54-75); the spectrum comes from the GPU FFT.
std::vector<double> estimate_mask(const std::vector<double>& w0, int64_t side, double frac) {
  std::vector<double> spec = w0;
  if (side <= 64) op_fft2<double>(spec.data(), side, side, false);
  else op_fft2<float>(spec.data(), side, side, false);
  std::vector<std::pair<double, double>> by_radius;
  double total = 0.0;
  for (int64_t k = 0; k < side; ++k)
    for (int64_t l = 0; l < side; ++l) {
      const int64_t i = k * side + l;
      const double e = spec[2 * i] * spec[2 * i] + spec[2 * i + 1] * spec[2 * i + 1];
      by_radius.emplace_back(freq_radius(k, l, side), e);
      total += e;
    }
  std::sort(by_radius.begin(), by_radius.end());
  double acc = 0.0, radius = 0.0;
  for (const auto& [rad, e] : by_radius) {
    acc += e;
    radius = rad;
    if (acc >= frac * total) break;
  }
  return disk_mask(side, radius);
}

namespace {

template <typename T>
class Blind final : public BlindGpu {
 public:
  Blind(const Plan& plan, const DataSpec& data, const BlindConfig& cfg, const double* mask, const double* pin_ones,
        int device, Comm* comm)
      : plan_(plan), cfg_(cfg), pool_(device) {
    AllocStream alloc_scope(R.st());  // every buffer is stream-ordered on the solver stream
    cfg_.validate(plan.g.s, mask);
    plan.g.validate();
    R.build(plan, data, pin_ones, device, comm, cfg.max_iters, "BlindSolver");
    if (R.l1 <= 0.0) throw InvalidArgument("BlindSolver: all-zero measurements");
    cudaStream_t s = R.st();
    const int64_t SS = R.SS(), nf = R.L.nfr * SS;
    const int nls = R.L.nls();
    for (auto* m : {&gamma_[0], &gamma_[1], &q_}) m->alloc(sizeof(cx<T>) * std::max<int64_t>(nf, 1));
    u_.alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.img_elems, 1));
    v_.alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.v_elems, 1));
    lam_.alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.lam_elems, 1));
    s_.alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.s_elems, 1));
    wc_.alloc(sizeof(cx<T>) * std::max(nls, 1) * SS);
    delta_.alloc(sizeof(cx<T>) * std::max(nls, 1) * SS);
    num_.alloc(sizeof(cx<T>) * std::max(nls, 1) * SS);
    den_.alloc(sizeof(T) * std::max(nls, 1) * SS);
    w_.alloc(sizeof(cx<T>) * SS);
    avg_.alloc(sizeof(cx<T>) * SS);
    spec_.alloc(sizeof(cx<T>) * SS);
    wd_all_.alloc(sizeof(cx<T>) * R.D * SS);
    std::vector<cx<T>> ones(static_cast<size_t>(SS), cx<T>{T(1), T(0)});
    ones_ = upload(ones, s);
    one_off_ = upload(std::vector<int64_t>{0}, s);
    one_pitch_ = upload(std::vector<int32_t>{R.S}, s);

    // rpen = r per covering pair, pinned -> -1 (blind.cpp:100-107)
    rpen_.alloc(sizeof(T) * std::max<int64_t>(R.L.img_elems, 1));
    for (int ld = 0; ld < nls; ++ld) {
      PDD_CUDA(launch_rpen_sub<T>(R.pins_of(ld), R.psides.template as<PairSide>() + R.L.sub_pbeg[ld],
                                  R.L.sub_pbeg[ld + 1] - R.L.sub_pbeg[ld], R.L.sub_h[ld], R.L.sub_w[ld],
                                  static_cast<T>(cfg_.r), rpen_.as<T>() + R.L.sub_img_off[ld], s));
    }
    build_chunks();
    initial_probe();
    mask_h_ = mask ? std::vector<double>(mask, mask + SS) : estimate_mask(w0_, R.S, cfg_.support_energy);
    std::vector<T> mt(mask_h_.begin(), mask_h_.end());
    mask_ = upload(mt, s);
    PDD_CUDA(cudaStreamSynchronize(s));
    layout_ = R.state_layout(plan);
    init_state(nullptr);
  }

  const StateLayout& layout() const override { return layout_; }

  // Fixed frame chunks per local subdomain for the probe-side reductions.
  void build_chunks() {
    constexpr int kChunk = 32;
    std::vector<int32_t> f0, f1, beg{0};
    for (int ld = 0; ld < R.L.nls(); ++ld) {
      for (int64_t f = R.L.sub_fr_beg[ld]; f < R.L.sub_fr_beg[ld + 1]; f += kChunk) {
        f0.push_back(static_cast<int32_t>(f));
        f1.push_back(static_cast<int32_t>(std::min<int64_t>(f + kChunk, R.L.sub_fr_beg[ld + 1])));
      }
      beg.push_back(static_cast<int32_t>(f0.size()));
    }
    nchunks_ = static_cast<int>(f0.size());
    chunk_f0_ = upload(f0, R.st());
    chunk_f1_ = upload(f1, R.st());
    chunk_beg_ = upload(beg, R.st());
    num_part_.alloc(sizeof(cx<T>) * std::max(nchunks_, 1) * R.SS());
    den_part_.alloc(sizeof(T) * std::max(nchunks_, 1) * R.SS());
  }

  // w0 = gain * mean_j IFFT(checkerboard o sqrt f_j), gain^2 = max_j sum f_j / ||.||^2
  // (blind.cpp:123-153).
  void initial_probe() {
    cudaStream_t s = R.st();
    const int64_t SS = R.SS();
    PDD_CUDA(launch_checker<T>(R.amp.template as<T>(), R.L.nfr, R.S, q_.as<cx<T>>(), s));
    FrameArgs<T> a = R.frame_args();
    a.probe = ones_.as<cx<T>>();
    a.frames_in = q_.as<cx<T>>();
    a.bp_out = gamma_[1].as<cx<T>>();
    PDD_CUDA(launch_frame<T>(kAdj, R.S, a, s));
    PDD_CUDA(launch_probe_partials<T>(nullptr, nullptr, nullptr, gamma_[1].as<cx<T>>(), chunk_f0_.as<int32_t>(),
                                      chunk_f1_.as<int32_t>(), nchunks_, R.S, 1, num_part_.as<cx<T>>(), nullptr,
                                      nullptr, s));
    PDD_CUDA(launch_chunk_reduce<T>(num_part_.as<cx<T>>(), nullptr, chunk_beg_.as<int32_t>(), R.L.nls(),
                                    static_cast<int>(SS), num_.as<cx<T>>(), nullptr, nullptr, s));
    // per-subdomain sums -> all ranks (D-array, exact because one owner per entry)
    PDD_CUDA(cudaMemsetAsync(wd_all_.get(), 0, wd_all_.bytes(), s));
    for (int ld = 0; ld < R.L.nls(); ++ld)
      PDD_CUDA(cudaMemcpyAsync(wd_all_.as<cx<T>>() + static_cast<int64_t>(R.L.local_subs[ld]) * SS,
                               num_.as<cx<T>>() + static_cast<int64_t>(ld) * SS, sizeof(cx<T>) * SS,
                               cudaMemcpyDeviceToDevice, s));
    DevMem flux(sizeof(double) * std::max<int64_t>(R.L.nfr, 1));
    PDD_CUDA(launch_frame_flux<T>(R.amp.template as<T>(), R.L.nfr, SS, flux.as<double>(), s));
    std::vector<double> fl(static_cast<size_t>(R.L.nfr));
    PDD_CUDA(cudaMemcpyAsync(fl.data(), flux.get(), sizeof(double) * R.L.nfr, cudaMemcpyDeviceToHost, s));
    PDD_CUDA(cudaStreamSynchronize(s));
    std::vector<double> subflux(R.D, 0.0);
    for (int ld = 0; ld < R.L.nls(); ++ld)
      for (int64_t f = R.L.sub_fr_beg[ld]; f < R.L.sub_fr_beg[ld + 1]; ++f)
        subflux[R.L.local_subs[ld]] = std::max(subflux[R.L.local_subs[ld]], fl[f]);
    if (R.comm) {
      DevMem d(sizeof(double) * R.D);
      PDD_CUDA(cudaMemcpyAsync(d.get(), subflux.data(), sizeof(double) * R.D, cudaMemcpyHostToDevice, s));
      R.comm->allreduce_sum_f64(d.as<double>(), R.D, s);
      PDD_CUDA(cudaMemcpyAsync(subflux.data(), d.get(), sizeof(double) * R.D, cudaMemcpyDeviceToHost, s));
      allreduce_wd();
    }
    std::vector<cx<T>> sums = download_cx<T>(wd_all_.get(), R.D * SS, s);
    w0_.assign(static_cast<size_t>(2 * SS), 0.0);
    for (int d = 0; d < R.D; ++d)
      for (int64_t i = 0; i < SS; ++i) {
        w0_[2 * i] += static_cast<double>(sums[d * SS + i].x);
        w0_[2 * i + 1] += static_cast<double>(sums[d * SS + i].y);
      }
    const double count = static_cast<double>(plan_.g.J());
    double norm = 0.0, flux_max = 0.0;
    for (auto& x : w0_) x /= count;
    for (int64_t i = 0; i < SS; ++i) norm += w0_[2 * i] * w0_[2 * i] + w0_[2 * i + 1] * w0_[2 * i + 1];
    for (double x : subflux) flux_max = std::max(flux_max, x);
    const double gain = std::sqrt(flux_max / norm);
    for (auto& x : w0_) x *= gain;
  }

  void init_state(const double* w_init) override {  // blind.cpp:169-192
    cudaStream_t s = R.st();
    const int64_t SS = R.SS();
    const double* w = w_init ? w_init : w0_.data();
    upload_cx<T>(w_.get(), w, SS, s);
    for (int ld = 0; ld < R.L.nls(); ++ld)
      PDD_CUDA(cudaMemcpyAsync(wc_.as<cx<T>>() + ld * SS, w_.get(), sizeof(cx<T>) * SS, cudaMemcpyDeviceToDevice, s));
    for (int d = 0; d < R.D; ++d)
      PDD_CUDA(cudaMemcpyAsync(wd_all_.as<cx<T>>() + d * SS, w_.get(), sizeof(cx<T>) * SS, cudaMemcpyDeviceToDevice, s));
    PDD_CUDA(cudaMemsetAsync(delta_.get(), 0, delta_.bytes(), s));
    PDD_CUDA(launch_fill<T>(u_.as<cx<T>>(), R.L.img_elems, cx<T>{T(1), T(0)}, s));
    PDD_CUDA(cudaMemsetAsync(gamma_[0].get(), 0, gamma_[0].bytes(), s));
    PDD_CUDA(cudaMemsetAsync(lam_.get(), 0, lam_.bytes(), s));
    R.consensus(u_.as<cx<T>>(), lam_.as<cx<T>>(), s_.as<cx<T>>(), v_.as<cx<T>>(), nullptr);
    iter_ = 0;
    z_valid_ = false;
    if (z_.bytes()) {
      FrameArgs<T> a = R.frame_args();
      a.probe = wc_.as<cx<T>>();
      a.probe_idx = R.fr_sub.template as<int32_t>();
      a.img = u_.as<cx<T>>();
      a.frames_out = z_.as<cx<T>>();
      PDD_CUDA(launch_frame<T>(kFwd, R.S, a, s));
      z_valid_ = true;
    }
    PDD_CUDA(cudaStreamSynchronize(s));
  }

  // Delta_d + W_d for every d (after a state change outside the graphs).
  void refresh_wd() {
    cudaStream_t s = R.st();
    const int64_t SS = R.SS();
    if (R.comm) PDD_CUDA(cudaMemsetAsync(wd_all_.get(), 0, wd_all_.bytes(), s));
    std::vector<cx<T>> wc = download_cx<T>(wc_.get(), R.L.nls() * SS, s), dl = download_cx<T>(delta_.get(), R.L.nls() * SS, s);
    for (int ld = 0; ld < R.L.nls(); ++ld) {
      std::vector<cx<T>> t(static_cast<size_t>(SS));
      for (int64_t i = 0; i < SS; ++i) t[i] = dl[ld * SS + i] + wc[ld * SS + i];
      PDD_CUDA(cudaMemcpyAsync(wd_all_.as<cx<T>>() + static_cast<int64_t>(R.L.local_subs[ld]) * SS, t.data(),
                               sizeof(cx<T>) * SS, cudaMemcpyHostToDevice, s));
      PDD_CUDA(cudaStreamSynchronize(s));
    }
    allreduce_wd();
    PDD_CUDA(cudaStreamSynchronize(s));
  }

  void allreduce_wd() {
    if (!R.comm) return;
    // exact: every entry has a single non-zero contributor
    if constexpr (sizeof(T) == 8) R.comm->allreduce_sum_f64(reinterpret_cast<double*>(wd_all_.get()), 2 * R.D * R.SS(), R.st());
    else R.comm->allreduce_sum_f32(reinterpret_cast<float*>(wd_all_.get()), 2 * R.D * R.SS(), R.st());
  }

  void enqueue_iteration(int parity, bool store_z, cudaEvent_t* ev = nullptr) {
    cudaStream_t s = R.st();
    const int64_t SS = R.SS();
    // (the pass switches were set by reset_ctl or by the previous iteration's RE finalize step)
    if (ev) PDD_CUDA(cudaEventRecord(ev[0], s));
    FrameArgs<T> a = R.frame_args();
    a.probe = wc_.as<cx<T>>();
    a.probe_idx = R.fr_sub.template as<int32_t>();
    a.probe2 = w_.as<cx<T>>();
    a.img = u_.as<cx<T>>();
    a.gamma_in = gamma_[parity].as<cx<T>>();
    a.gamma_out = gamma_[1 - parity].as<cx<T>>();
    a.z_out = store_z ? z_.as<cx<T>>() : nullptr;
    a.bp_out = q_.as<cx<T>>();
    a.rf_part = R.rf_part.template as<double>();
    a.stop_flag = R.skipA();
    a.lam = static_cast<T>(cfg_.eta);
    a.eps = static_cast<T>(cfg_.epsilon);
    a.fast_prox = cfg_.eta <= (1.0 - cfg_.epsilon) / cfg_.epsilon;
    R.set_pieces(a);  // streamed sweep schedule (one piece per frame: q_j stays per frame)
    PDD_CUDA(launch_frame<T>(kBlind, R.S, a, s));
    if (ev) PDD_CUDA(cudaEventRecord(ev[1], s));
    R.reduce_rf_finalize();
    // w-step (blind.cpp:194-208): one launch where the frame fits a single-CTA engine
    const cudaError_t we = launch_wstep<T>(R.S, wd_all_.as<cx<T>>(), R.D, mask_.as<T>(), R.tw.template as<cx<T>>(),
                                           static_cast<T>(1.0 / static_cast<double>(R.S)), w_.as<cx<T>>(), R.skipB(), s);
    if (we != cudaErrorNotSupported) {
      PDD_CUDA(we);
    } else {
    PDD_CUDA(launch_probe_avg<T>(wd_all_.as<cx<T>>(), R.D, static_cast<int>(SS), avg_.as<cx<T>>(), R.skipB(), s));
    FrameArgs<T> p1 = R.frame_args();
    p1.nframes = 1;
    p1.off = one_off_.as<int64_t>();
    p1.pitch = one_pitch_.as<int32_t>();
    p1.probe = ones_.as<cx<T>>();
    p1.img = avg_.as<cx<T>>();
    p1.frames_out = spec_.as<cx<T>>();
    p1.stop_flag = R.skipB();
    PDD_CUDA(launch_frame<T>(kFwd, R.S, p1, s));
    PDD_CUDA(launch_apply_mask<T>(spec_.as<cx<T>>(), mask_.as<T>(), static_cast<int>(SS), R.skipB(), s));
    FrameArgs<T> p2 = p1;
    p2.img = nullptr;
    p2.frames_out = nullptr;
    p2.frames_in = spec_.as<cx<T>>();
    p2.bp_out = w_.as<cx<T>>();
    PDD_CUDA(launch_frame<T>(kAdj, R.S, p2, s));
    }
    // v-step from u^n, Lambda^n (blind.cpp:209-218).  Sequential here: the
    // blind image-side state is single-buffered (only Gamma ping-pongs), so
    // the v-step must see this iteration's stop decision (skipB).
    R.consensus(u_.as<cx<T>>(), lam_.as<cx<T>>(), s_.as<cx<T>>(), v_.as<cx<T>>(), R.skipB());
    // W-step with u^n
    PDD_CUDA(launch_probe_partials<T>(u_.as<cx<T>>(), R.fr_off.template as<int64_t>(), R.fr_pitch.template as<int32_t>(),
                                      q_.as<cx<T>>(), chunk_f0_.as<int32_t>(), chunk_f1_.as<int32_t>(), nchunks_, R.S, 0,
                                      num_part_.as<cx<T>>(), den_part_.as<T>(), R.skipB(), s));
    PDD_CUDA(launch_chunk_reduce<T>(num_part_.as<cx<T>>(), den_part_.as<T>(), chunk_beg_.as<int32_t>(), R.L.nls(),
                                    static_cast<int>(SS), num_.as<cx<T>>(), den_.as<T>(), R.skipB(), s));
    if (R.comm) PDD_CUDA(cudaMemsetAsync(wd_all_.get(), 0, wd_all_.bytes(), s));
    PDD_CUDA(launch_probe_update<T>(num_.as<cx<T>>(), den_.as<T>(), w_.as<cx<T>>(), wc_.as<cx<T>>(),
                                    delta_.as<cx<T>>(), wd_all_.as<cx<T>>(), R.local_map.template as<int>(), R.L.nls(),
                                    static_cast<int>(SS), static_cast<T>(cfg_.eta), static_cast<T>(cfg_.mu), R.skipB(),
                                    s));
    allreduce_wd();
    // u-step with W^{n+1}
    GatherArgs<T> g = R.gather_args(kGatherBlind);
    g.bp = q_.as<cx<T>>();
    g.probe = wc_.as<cx<T>>();
    g.u = u_.as<cx<T>>();
    g.rpen = rpen_.as<T>();
    g.v = v_.as<cx<T>>();
    g.lam = lam_.as<cx<T>>();
    g.eta = static_cast<T>(cfg_.eta);
    g.r = static_cast<T>(cfg_.r);
    g.gamma = static_cast<T>(cfg_.gamma);
    g.re_part = R.re_part.template as<double>();
    g.stop_flag = R.skipB();
    if (ev) PDD_CUDA(cudaEventRecord(ev[2], s));
    PDD_CUDA(launch_gather<T>(g, s));
    if (ev) PDD_CUDA(cudaEventRecord(ev[3], s));
    R.reduce_re_finalize();
  }

  void enqueue_tail() {  // R-factor of the current iterate with the shared probe
    cudaStream_t s = R.st();
    PDD_CUDA(launch_gate(R.ctlp(), s));
    FrameArgs<T> a = R.frame_args();
    a.probe = w_.as<cx<T>>();
    a.img = u_.as<cx<T>>();
    a.rf_part = R.rf_part.template as<double>();
    a.stop_flag = R.skipA();
    PDD_CUDA(launch_frame<T>(kFwd, R.S, a, s));
    R.reduce_rf_finalize();
  }

  void ensure_graphs() {
    if (full_[0].ready()) return;
    // a host-blocking transport (test transport, Comm::capturable) runs the
    // same bodies eagerly
    const bool eager = R.comm && !R.comm->capturable();
    for (int p = 0; p < 2; ++p) {
      full_[p].capture(R.st(), [this, p] {
        enqueue_iteration(p, false);
        enqueue_iteration(1 - p, false);
      }, eager);
      one_[p].capture(R.st(), [this, p] { enqueue_iteration(p, false); }, eager);
    }
    tail_.capture(R.st(), [this] { enqueue_tail(); }, eager);
  }

  void ensure_z() {
    if (!z_.bytes()) z_.alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.nfr * R.SS(), 1));
  }

  void step(bool store_z) override {
    if (store_z) ensure_z();
    R.reset_ctl(static_cast<int>(iter_), static_cast<int>(iter_) + 1, 2, cfg_.tol_rf, cfg_.tol_re);
    enqueue_iteration(static_cast<int>(iter_ & 1), store_z);
    R.stream.sync();
    PDD_CUDA(cudaStreamSynchronize(R.st()));
    ++iter_;
    z_valid_ = store_z;
  }

  // on_poll(ctl, per-launch ms so far) at every poll (the stream is idle then).
  std::vector<double> drive(int max_total, bool poll, bool tail = true,
                            const std::function<void(const RunCtl&, const std::vector<double>&)>& on_poll = {}) {
    ensure_graphs();
    constexpr int kPoll = 8;
    cudaStream_t s = R.st();
    std::vector<cudaEvent_t> ev;
    int launched = 0;
    const int parity = static_cast<int>(iter_ & 1);
    cudaEvent_t e0;
    PDD_CUDA(cudaEventCreate(&e0));
    PDD_CUDA(cudaEventRecord(e0, s));
    ev.push_back(e0);
    while (launched < max_total) {
      const int batch = std::min(kPoll, (max_total - launched + 1) / 2);
      for (int b = 0; b < batch; ++b) {
        if (!tail && launched + 2 * b + 1 == max_total)
          one_[parity].launch(s);  // odd count, no trailing R-factor pass (nonblind.cu drive)
        else
          full_[parity].launch(s);
        cudaEvent_t e;
        PDD_CUDA(cudaEventCreate(&e));
        PDD_CUDA(cudaEventRecord(e, s));
        ev.push_back(e);
      }
      launched += 2 * batch;
      if (launched >= max_total) break;
      if (poll) {
        const RunCtl c = R.read_ctl();
        if (on_poll) on_poll(c, event_ms(ev));
        if (c.stop) break;
      }
    }
    PDD_CUDA(cudaStreamSynchronize(s));
    std::vector<double> ms;
    for (size_t i = 1; i < ev.size(); ++i) {
      float t = 0.f;
      PDD_CUDA(cudaEventElapsedTime(&t, ev[i - 1], ev[i]));
      ms.push_back(t);
    }
    for (auto e : ev) cudaEventDestroy(e);
    iter_ = R.read_ctl().iter;
    if (tail) {  // R-factor of the final iterate
      tail_.launch(s);
      PDD_CUDA(cudaStreamSynchronize(s));
    }
    return ms;
  }

  RunRecords run(const RecordFn& on_record) override {  // blind.cpp:298-358, from the current state
    refresh_wd();
    R.reset_ctl(static_cast<int>(iter_), static_cast<int>(iter_) + cfg_.max_iters, cfg_.stop_rule, cfg_.tol_rf,
                cfg_.tol_re);
    const int64_t start = iter_;
    RecordFeed feed{&on_record, start, start};
    const auto ms = drive(cfg_.max_iters, true, true, [&](const RunCtl& c, const std::vector<double>& ms_now) {
      feed.upto(R.rec.template as<double>(), R.rec_cap, R.st(), c.stop ? c.stop : c.iter - 1, ms_now);
    });
    const RunCtl c = R.read_ctl();
    RunRecords out;
    const int64_t last = c.stop ? c.stop : c.iter;
    out.iterations = last - start;
    out.diverged_at = c.diverged ? c.diverged - start : 0;
    std::vector<double> rec(2 * static_cast<size_t>(R.rec_cap));
    PDD_CUDA(cudaMemcpyAsync(rec.data(), R.rec.get(), sizeof(double) * rec.size(), cudaMemcpyDeviceToHost, R.st()));
      PDD_CUDA(cudaStreamSynchronize(R.st()));
    for (int64_t n = start + 1; n <= last; ++n) {
      const int64_t k = (n - 1) % R.rec_cap;
      out.rf.push_back(rec[2 * k]);
      out.re.push_back(rec[2 * k + 1]);
      const size_t li = static_cast<size_t>((n - start - 1) / 2);
      out.t_ms.push_back(ms.empty() ? 0.0 : ms[std::min(li, ms.size() - 1)] / 2.0);
    }
    feed.upto(R.rec.template as<double>(), R.rec_cap, R.st(), last, ms);
    iter_ = last;
    z_valid_ = false;
    return out;
  }

  void iterate(int n) override {
    if (n <= 0) return;
    refresh_wd();
    R.reset_ctl(static_cast<int>(iter_), static_cast<int>(iter_) + n, 2, cfg_.tol_rf, cfg_.tol_re);
    drive(n, false);
    z_valid_ = false;
  }

  double iterate_timed(int n) override {  // exactly n iterations, CUDA events on the solver stream
    if (n <= 0) return 0.0;
    refresh_wd();
    R.reset_ctl(static_cast<int>(iter_), static_cast<int>(iter_) + n, 2, cfg_.tol_rf, cfg_.tol_re);
    ensure_graphs();
    cudaEvent_t e0, e1;
    PDD_CUDA(cudaEventCreate(&e0));
    PDD_CUDA(cudaEventCreate(&e1));
    PDD_CUDA(cudaEventRecord(e0, R.st()));
    drive(n, false, false);
    PDD_CUDA(cudaEventRecord(e1, R.st()));
    PDD_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PDD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    z_valid_ = false;
    return ms;
  }

  // n eager iterations: ms[0] frame kernel (BLIND mode), ms[1] u-gather, ms[2] whole iteration.
  void profile(int n, double* out) override {
    cudaEvent_t ev[4], e_start, e_end;
    for (auto& e : ev) PDD_CUDA(cudaEventCreate(&e));
    PDD_CUDA(cudaEventCreate(&e_start));
    PDD_CUDA(cudaEventCreate(&e_end));
    refresh_wd();
    R.reset_ctl(static_cast<int>(iter_), static_cast<int>(iter_) + n, 2, cfg_.tol_rf, cfg_.tol_re);
    double fr = 0.0, ga = 0.0;
    PDD_CUDA(cudaEventRecord(e_start, R.st()));
    for (int i = 0; i < n; ++i) {
      enqueue_iteration(static_cast<int>(iter_ & 1), false, ev);
      PDD_CUDA(cudaEventSynchronize(ev[3]));
      float a = 0.f, b = 0.f;
      PDD_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
      PDD_CUDA(cudaEventElapsedTime(&b, ev[2], ev[3]));
      fr += a;
      ga += b;
      ++iter_;
    }
    PDD_CUDA(cudaEventRecord(e_end, R.st()));
    PDD_CUDA(cudaEventSynchronize(e_end));
    float tot = 0.f;
    PDD_CUDA(cudaEventElapsedTime(&tot, e_start, e_end));
    out[0] = fr / n;
    out[1] = ga / n;
    out[2] = tot / n;
    for (auto& e : ev) cudaEventDestroy(e);
    cudaEventDestroy(e_start);
    cudaEventDestroy(e_end);
    z_valid_ = false;
  }

  void get_state(double* w, double* wc, double* delta, double* u, double* z, double* gamma, double* v, double* lam,
                 int64_t* iteration) override {
    cudaStream_t s = R.st();
    const int64_t SS = R.SS(), nf = R.L.nfr * SS;
    if (w) download_c128<T>(w_.get(), SS, w, s);
    if (wc) download_c128<T>(wc_.get(), R.L.nls() * SS, wc, s);
    if (delta) download_c128<T>(delta_.get(), R.L.nls() * SS, delta, s);
    if (u) download_c128<T>(u_.get(), R.L.img_elems, u, s);
    if (gamma) download_c128<T>(gamma_[iter_ & 1].get(), nf, gamma, s);
    if (z) {
      if (z_valid_) download_c128<T>(z_.get(), nf, z, s);
      else std::fill(z, z + 2 * nf, NAN);
    }
    if (v) download_c128<T>(v_.get(), R.L.v_elems, v, s);
    if (lam) download_c128<T>(lam_.get(), R.L.lam_elems, lam, s);
    if (iteration) *iteration = iter_;
  }

  void set_state(const double* w, const double* wc, const double* delta, const double* u, const double* z,
                 const double* gamma, const double* v, const double* lam, int64_t iteration) override {
    cudaStream_t s = R.st();
    const int64_t SS = R.SS(), nf = R.L.nfr * SS;
    iter_ = iteration;
    if (w) upload_cx<T>(w_.get(), w, SS, s);
    if (wc) upload_cx<T>(wc_.get(), wc, R.L.nls() * SS, s);
    if (delta) upload_cx<T>(delta_.get(), delta, R.L.nls() * SS, s);
    if (u) upload_cx<T>(u_.get(), u, R.L.img_elems, s);
    if (gamma) upload_cx<T>(gamma_[iter_ & 1].get(), gamma, nf, s);
    if (z) {
      ensure_z();
      upload_cx<T>(z_.get(), z, nf, s);
      z_valid_ = true;
    }
    if (v) upload_cx<T>(v_.get(), v, R.L.v_elems, s);
    if (lam) upload_cx<T>(lam_.get(), lam, R.L.lam_elems, s);
    refresh_wd();
  }

  // result.probe / probe_fourier = project_support(state.w) (blind.cpp:440)
  void get_probe(double* probe, double* probe_fourier, double* mask, double* w0) override {
    const int64_t SS = R.SS();
    std::vector<double> w(static_cast<size_t>(2 * SS));
    from_cx(download_cx<T>(w_.get(), SS, R.st()), w.data());
    std::vector<double> spec = w;
    if (sizeof(T) == 8) op_fft2<double>(spec.data(), R.S, R.S, false);
    else op_fft2<float>(spec.data(), R.S, R.S, false);
    for (int64_t i = 0; i < SS; ++i)
      if (mask_h_[i] == 0.0) spec[2 * i] = spec[2 * i + 1] = 0.0;
    if (probe_fourier) std::copy(spec.begin(), spec.end(), probe_fourier);
    if (probe) {
      std::vector<double> back = spec;
      if (sizeof(T) == 8) op_fft2<double>(back.data(), R.S, R.S, true);
      else op_fft2<float>(back.data(), R.S, R.S, true);
      std::copy(back.begin(), back.end(), probe);
    }
    if (mask) std::copy(mask_h_.begin(), mask_h_.end(), mask);
    if (w0) std::copy(w0_.begin(), w0_.end(), w0);
  }

  void merged(double* out) override { R.merge_to_host(plan_, u_.as<cx<T>>(), out); }
  void sync() override { R.stream.sync(); }
  // float32 s = 64: the BLIND frame pass is two streamed launches (kernels.cu)
  void* stream() const override { return R.st(); }
  // frame pass (two launches only for complex128 128^2); R-factor sums + finalize (1 fused / 2);
  // w-step (1 where wstep_kernel applies, else 4); pack, vstep; probe partials, chunk reduce, probe
  // update; update pass; RE sums + finalize (1 fused / 3)
  int64_t kernel_launches_per_iteration() const override {
    const int frame = (std::is_same_v<T, double> && R.S == 128) ? 2 : 1;
    const int wstep = (R.S == 16 || R.S == 32 || R.S == 64) ? 1 : 4;
    return frame + (R.fused_finalize() ? 1 : 2) + wstep + 2 + 3 + 1 + (R.fused_finalize() ? 1 : 3);
  }

 private:
  Plan plan_;
  BlindConfig cfg_;
  PoolUser pool_;  // before every DevMem: the pool outlives them
  RankData<T> R;
  StateLayout layout_;
  DevMem gamma_[2], q_, u_, v_, lam_, s_, rpen_, z_, wc_, delta_, num_, den_, w_, avg_, spec_, wd_all_, ones_, mask_;
  DevMem one_off_, one_pitch_, chunk_f0_, chunk_f1_, chunk_beg_, num_part_, den_part_;
  int nchunks_ = 0;
  std::vector<double> w0_, mask_h_;
  Graph full_[2], one_[2], tail_;
  int64_t iter_ = 0;
  bool z_valid_ = false;
};

}  // namespace

std::unique_ptr<BlindGpu> make_blind(const Plan& plan, const DataSpec& data, const BlindConfig& cfg, const double* mask,
                                     const double* pin_ones, int dtype, int device, Comm* comm) {
  DeviceGuard guard(device);
  if (dtype == 2) return std::make_unique<Blind<double>>(plan, data, cfg, mask, pin_ones, device, comm);
  return std::make_unique<Blind<float>>(plan, data, cfg, mask, pin_ones, device, comm);
}

}  // namespace pdd
