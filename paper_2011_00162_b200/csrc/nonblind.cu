// Nonblind OD²P driver: NonblindSolver (proj/src/solver.cpp) on the GPU.
//
// Per iteration (the paper's Steps 1-4, solver.cpp:118-205), one CUDA graph
// node chain per rank:
//   gate -> frame SWEEP (z/Gamma step + back-projection, RF partials of u^n)
//        -> segsum/[all-reduce] -> rf_finalize (records RF of the previous
//           iterate and applies the R-factor stop rule with Gamma ping-pong
//           so a stop rolls back for free)
//        -> [join] gather (adjoint overlap-add + u-update + Lambda-update + RE)
//   branch forked at the gate, concurrent with the frame pass:
//           pack s = u + Lambda -> [NCCL send/recv per cut pair] -> v-step
//        -> segsum/[all-reduce] -> re_finalize (RE stop rule, max_iters)
// Two iterations (Gamma parities) per graph.  The R-factor of iterate n is
// produced by the frame pass of iteration n+1 (its forward transform is the
// reference's cached `au`), and by one trailing frame pass at the end.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <chrono>

#include "common.cuh"

namespace pdd {

void host_stage_reserve() { HostStage::get().reserve(); }


void NonblindConfig::validate() const {  // solver.cpp:24-31
  if (!(epsilon > 0.0 && epsilon < 1.0)) throw InvalidArgument("stagm: epsilon must lie in (0,1)");
  if (eta <= 0.0 || r <= 0.0) throw InvalidArgument("NonblindConfig: eta, r must be > 0");
  if (max_iters < 1) throw InvalidArgument("NonblindConfig: max_iters >= 1");
  if (tol_rf <= 0.0 || tol_re <= 0.0) throw InvalidArgument("NonblindConfig: tolerances must be > 0");
  if (threads < 0) throw InvalidArgument("NonblindConfig: threads >= 0");
}

namespace {

template <typename T>
class Nonblind final : public NonblindGpu {
 public:
  Nonblind(const Plan& plan, const DataSpec& data, const double* probe, const NonblindConfig& cfg,
           const double* pin_ones, int device, Comm* comm)
      : plan_(plan), cfg_(cfg), pool_(device) {
    AllocStream alloc_scope(R.st());  // every buffer is stream-ordered on the solver stream
    cfg_.validate();
    plan.g.validate();
    R.build(plan, data, pin_ones, device, comm, cfg.max_iters, "NonblindSolver", piece_length(plan, device));
    if (R.l1 <= 0.0) throw InvalidArgument("NonblindSolver: all-zero measurements, R-factor undefined");
    const int64_t SS = R.SS();
    cudaStream_t s = R.st();
    probe_ = upload(to_cx<T>(probe, SS), s);
    probe64_ = upload(to_cx<double>(probe, SS), s);
    const int64_t nf = R.L.nfr * SS;
    gamma_[0].alloc(sizeof(cx<T>) * std::max<int64_t>(nf, 1));
    gamma_[1].alloc(sizeof(cx<T>) * std::max<int64_t>(nf, 1));
    bp_.alloc(sizeof(cx<T>) * std::max<int64_t>(std::max(nf, R.L.part_elems), 1));  // partials; also A u scratch
    for (int p = 0; p < 2; ++p) {  // iterate ping-pong (state of iteration n in [n & 1])
      u_[p].alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.img_elems, 1));
      v_[p].alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.v_elems, 1));
      lam_[p].alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.lam_elems, 1));
    }
    s_.alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.s_elems, 1));
    SetupTimer tm;
    build_denominators();
    tm.mark("denominators");
    layout_ = R.state_layout(plan);
    init_state();
    tm.mark("init_state");
  }

  const StateLayout& layout() const override { return layout_; }

  // S = 128 float32: the streamed sweep accumulates back-projections over
  // pieces of frames in tensor memory.  The length depends on the plan and
  // the device only -- never on the GPU count, so iterates stay identical for
  // every G: at least 6 pieces per SM when each GPU holds a single subdomain
  // (the smallest per-GPU share; the static piece schedule then stays within
  // a few percent of balance), at most Layout::kPieceLen frames; pairs for
  // subdomains of 2 to 6 frames per SM.
  // PDD_PIECE_LEN overrides (1: one piece per frame, for A/B runs).
  static int piece_length(const Plan& plan, int device) {
    if (sizeof(T) != 4 || plan.g.s != 128) return 1;
    if (const char* e = std::getenv("PDD_PIECE_LEN")) return std::max(1, std::atoi(e));
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || sms <= 0) return 1;
    int64_t jmin = INT64_MAX;
    for (const auto& fr : plan.frames_of) jmin = std::min<int64_t>(jmin, static_cast<int64_t>(fr.size()));
    const int64_t bal = jmin / (6 * int64_t(sms));
    if (bal >= 1) return static_cast<int>(std::min<int64_t>(Layout::kPieceLen, bal));
    // small subdomains (config 2: 450 frames): pairs of frames still fill every
    // SM when a GPU holds one subdomain (>= 2 frames per SM either way), and
    // the update pass reads 10 instead of 16 partial values per pixel
    return jmin >= 2 * int64_t(sms) ? 2 : 1;
  }

  // solver.cpp:53-75: denom = eta * illumination_density + r per covering pair.
  void build_denominators() {
    cudaStream_t s = R.st();
    DevMem dens(sizeof(double) * std::max<int64_t>(R.L.img_elems, 1));
    GatherArgs<double> g;
    {
      auto gt = R.gather_args(kGatherDensity);
      g.mode = kGatherDensity;
      g.ntiles = gt.ntiles;
      g.tile_h = gt.tile_h;
      g.tile_w = gt.tile_w;
      g.sub_pbeg = gt.sub_pbeg;
      g.ps = gt.ps;
      g.tiles = gt.tiles;
      g.tile_frames = gt.tile_frames;
      g.fr_r = gt.fr_r;
      g.fr_c = gt.fr_c;
      g.fr_sub = gt.fr_sub;
      g.S = gt.S;
      g.sub_off = gt.sub_off;
      g.sub_h = gt.sub_h;
      g.sub_w = gt.sub_w;
    }
    g.probe = probe64_.as<cx<double>>();
    g.dens_out = dens.as<double>();
    PDD_CUDA(launch_gather<double>(g, s));
    denom_.alloc(sizeof(T) * std::max<int64_t>(R.L.img_elems, 1));
    DevMem bad(sizeof(unsigned long long) * std::max(R.L.nls(), 1));
    PDD_CUDA(cudaMemsetAsync(bad.get(), 0, bad.bytes(), s));
    for (int ld = 0; ld < R.L.nls(); ++ld) {
      const int nps = R.L.sub_pbeg[ld + 1] - R.L.sub_pbeg[ld];
      PDD_CUDA(launch_denom_sub<T>(dens.as<double>() + R.L.sub_img_off[ld], R.pins_of(ld),
                                   R.psides.template as<PairSide>() + R.L.sub_pbeg[ld], nps, R.L.sub_h[ld], R.L.sub_w[ld],
                                   static_cast<T>(cfg_.eta), static_cast<T>(cfg_.r),
                                   denom_.as<T>() + R.L.sub_img_off[ld], bad.as<unsigned long long>() + ld, s));
    }
    std::vector<unsigned long long> nbad(std::max(R.L.nls(), 1));
    PDD_CUDA(cudaMemcpyAsync(nbad.data(), bad.get(), bad.bytes(), cudaMemcpyDeviceToHost, s));
    PDD_CUDA(cudaStreamSynchronize(s));
    for (int ld = 0; ld < R.L.nls(); ++ld)
      if (nbad[ld])
        throw RuntimeError("NonblindSolver: illumination density vanishes inside subdomain " +
                           std::to_string(R.L.local_subs[ld]) +
                           "; A_d*A_d is singular (probe/scan leave interior pixels dark)");
  }

  void init_state() override {  // solver.cpp:96-116
    cudaStream_t s = R.st();
    PDD_CUDA(launch_fill<T>(U(0), R.L.img_elems, cx<T>{T(1), T(0)}, s));
    PDD_CUDA(cudaMemsetAsync(gamma_[0].get(), 0, gamma_[0].bytes(), s));
    PDD_CUDA(cudaMemsetAsync(lam_[0].get(), 0, lam_[0].bytes(), s));
    R.consensus(U(0), LAM(0), s_.as<cx<T>>(), V(0), nullptr);
    iter_ = 0;
    z_valid_ = false;
    if (z_.bytes()) {  // z^0 = A u^0
      forward_into(z_.as<cx<T>>());
      z_valid_ = true;
    }
    PDD_CUDA(cudaStreamSynchronize(s));
  }

  cx<T>* U(int64_t p) const { return u_[p & 1].template as<cx<T>>(); }
  cx<T>* V(int64_t p) const { return v_[p & 1].template as<cx<T>>(); }
  cx<T>* LAM(int64_t p) const { return lam_[p & 1].template as<cx<T>>(); }

  void forward_into(cx<T>* out, double* rf_part = nullptr) {
    FrameArgs<T> a = R.frame_args();
    a.probe = probe_.as<cx<T>>();
    a.img = U(iter_);
    a.frames_out = out;
    a.rf_part = rf_part;
    PDD_CUDA(launch_frame<T>(kFwd, R.S, a, R.st()));
  }

  // One iteration's kernels.  parity: Gamma_in = gamma_[parity].  ev (eager
  // profiling only): events recorded around the frame and gather kernels.
  void enqueue_iteration(int parity, bool store_z, cudaEvent_t* ev = nullptr) {
    cudaStream_t s = R.st();
    // (the pass switches were set by reset_ctl or by the previous iteration's RE finalize step)
    // v^{n+1} from u^n, Lambda^n (solver.cpp:141-151) into the outgoing
    // parity, on a branch concurrent with the frame pass
    R.fork_consensus(U(parity), LAM(parity), s_.as<cx<T>>(), V(1 - parity));
    if (ev) PDD_CUDA(cudaEventRecord(ev[0], s));
    FrameArgs<T> a = R.frame_args();
    a.probe = probe_.as<cx<T>>();
    a.img = U(parity);
    a.gamma_in = gamma_[parity].as<cx<T>>();
    a.gamma_out = gamma_[1 - parity].as<cx<T>>();
    a.z_out = store_z ? z_.as<cx<T>>() : nullptr;
    a.bp_out = bp_.as<cx<T>>();
    a.rf_part = R.rf_part.template as<double>();
    a.stop_flag = R.skipA();
    a.lam = static_cast<T>(cfg_.eta);
    a.eps = static_cast<T>(cfg_.epsilon);
    a.fast_prox = cfg_.eta <= (1.0 - cfg_.epsilon) / cfg_.epsilon;
    R.set_pieces(a);
    PDD_CUDA(launch_frame<T>(kSweep, R.S, a, s));
    if (ev) PDD_CUDA(cudaEventRecord(ev[1], s));
    R.reduce_rf_finalize();
    R.join_consensus();
    GatherArgs<T> g = R.gather_args(kGatherNonblind);
    R.set_pieces(g);
    g.bp = bp_.as<cx<T>>();
    g.u_in = U(parity);
    g.u = U(1 - parity);
    g.denom = denom_.as<T>();
    g.v = V(1 - parity);
    g.lam_in = LAM(parity);
    g.lam = LAM(1 - parity);
    g.eta = static_cast<T>(cfg_.eta);
    g.r = static_cast<T>(cfg_.r);
    g.re_part = R.re_part.template as<double>();
    g.stop_flag = R.skipB();
    if (ev) PDD_CUDA(cudaEventRecord(ev[2], s));
    PDD_CUDA(launch_gather<T>(g, s));
    if (ev) PDD_CUDA(cudaEventRecord(ev[3], s));
    R.reduce_re_finalize();
  }

  // Frame pass only: records the R-factor of the current iterate.
  void enqueue_tail(int parity) {
    cudaStream_t s = R.st();
    PDD_CUDA(launch_gate(R.ctlp(), s));
    FrameArgs<T> a = R.frame_args();
    a.probe = probe_.as<cx<T>>();
    a.img = U(parity);
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
      tail_[p].capture(R.st(), [this, p] { enqueue_tail(p); }, eager);
      one_[p].capture(R.st(), [this, p] { enqueue_iteration(p, false); }, eager);
    }
  }

  void ensure_z() {
    if (!z_.bytes()) z_.alloc(sizeof(cx<T>) * std::max<int64_t>(R.L.nfr * R.SS(), 1));
  }

  void step(bool store_z) override {
    if (store_z) ensure_z();
    R.reset_ctl(static_cast<int>(iter_), static_cast<int>(iter_) + 1, 2, cfg_.tol_rf, cfg_.tol_re);
    enqueue_iteration(static_cast<int>(iter_ & 1), store_z);
    PDD_CUDA(cudaStreamSynchronize(R.st()));
    ++iter_;
    z_valid_ = store_z;
  }

  // Launch iteration-pair graphs until the device reports a stop; poll every
  // kPoll launches.  Returns per-launch milliseconds.
  // on_poll(ctl, per-launch ms so far) at every poll (the stream is idle then).
  std::vector<double> drive(int max_total, bool poll, bool tail = true,
                            const std::function<void(const RunCtl&, const std::vector<double>&)>& on_poll = {}) {
    ensure_graphs();
    constexpr int kPoll = 8;
    cudaStream_t s = R.st();
    std::vector<cudaEvent_t> ev;
    std::vector<double> ms;
    int launched = 0;
    int parity = static_cast<int>(iter_ & 1);
    cudaEvent_t e0;
    PDD_CUDA(cudaEventCreate(&e0));
    PDD_CUDA(cudaEventRecord(e0, s));
    ev.push_back(e0);
    while (launched < max_total) {
      const int batch = std::min(kPoll, (max_total - launched + 1) / 2);
      for (int b = 0; b < batch; ++b) {
        if (!tail && launched + 2 * b + 1 == max_total) {
          // odd count without the trailing R-factor pass: a one-iteration graph
          // (the second half of a pair would run the final iterate's frame
          // pass, i.e. the R-factor pass this call leaves out)
          one_[parity].launch(s);
        } else {
          full_[parity].launch(s);  // parity is preserved across a 2-iteration graph
        }
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
    for (size_t i = 1; i < ev.size(); ++i) {
      float t = 0.f;
      PDD_CUDA(cudaEventElapsedTime(&t, ev[i - 1], ev[i]));
      ms.push_back(t);
    }
    for (auto e : ev) cudaEventDestroy(e);
    const RunCtl c = R.read_ctl();
    iter_ = c.iter;
    if (tail) {  // R-factor of the final iterate (its frame pass)
      tail_[iter_ & 1].launch(s);
      PDD_CUDA(cudaStreamSynchronize(s));
    }
    return ms;
  }

  // metrics.cpp:73-101 for the current device state (u, z, Gamma, v, Lambda)
  // with au = A u recomputed on the device.  Frame terms per frame and
  // overlap terms per (pair, side) are fp64 partials with a single owner each;
  // they are all-reduced exactly and summed on the host in the reference's
  // order (subdomains, then pairs and sides), so the value is GPU-count
  // invariant.
  double lagrangian() override {
    if (!z_valid_)
      throw InvalidArgument("augmented_lagrangian: z of the current iterate is not stored (step with store_z)");
    cudaStream_t s = R.st();
    const int np = static_cast<int>(R.L.lpairs.size());
    if (!lag_fr_.bytes()) {
      lag_fr_.alloc(sizeof(double) * std::max<int64_t>(R.L.nfr, 1));
      lag_pr_.alloc(sizeof(double) * 2 * std::max(np, 1));
      lag_glob_.alloc(sizeof(double) * (R.D + 2 * std::max<size_t>(plan_.overlaps.size(), 1)));
    }
    forward_into(bp_.as<cx<T>>());
    PDD_CUDA(launch_lagrangian_frames<T>(bp_.as<cx<T>>(), z_.as<cx<T>>(), gamma_[iter_ & 1].as<cx<T>>(),
                                         R.amp.template as<T>(), R.L.nfr, R.SS(), cfg_.epsilon, cfg_.eta,
                                         lag_fr_.as<double>(), s));
    PDD_CUDA(launch_lagrangian_pairs<T>(R.pgeom.template as<PairGeom>(), np, U(iter_), V(iter_), LAM(iter_), cfg_.r,
                                        lag_pr_.as<double>(), s));
    const size_t P = plan_.overlaps.size();
    double* glob = lag_glob_.as<double>();  // [D] frame terms, then [P][2] overlap terms
    PDD_CUDA(cudaMemsetAsync(glob, 0, sizeof(double) * (R.D + 2 * P), s));
    PDD_CUDA(launch_segsum(lag_fr_.as<double>(), 1, 0, R.sub_fr_beg.template as<int64_t>(), R.L.nls(),
                           R.local_map.template as<int>(), glob, nullptr, s));
    std::vector<double> pr(2 * static_cast<size_t>(np));
    if (np) PDD_CUDA(cudaMemcpyAsync(pr.data(), lag_pr_.get(), sizeof(double) * pr.size(), cudaMemcpyDeviceToHost, s));
    PDD_CUDA(cudaStreamSynchronize(s));
    std::vector<double> gp(2 * P, 0.0);
    for (int lp = 0; lp < np; ++lp)
      for (int side = 0; side < 2; ++side)
        if (R.L.pgeom[lp].u_off[side] >= 0) gp[2 * R.L.lpairs[lp] + side] = pr[2 * lp + side];
    if (P) PDD_CUDA(cudaMemcpyAsync(glob + R.D, gp.data(), sizeof(double) * 2 * P, cudaMemcpyHostToDevice, s));
    if (R.comm) R.comm->allreduce_sum_f64(glob, R.D + 2 * P, s);
    std::vector<double> h(R.D + 2 * P);
    PDD_CUDA(cudaMemcpyAsync(h.data(), glob, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
    PDD_CUDA(cudaStreamSynchronize(s));
    double total = 0.0;
    for (double x : h) total += x;
    return total;
  }

  // run() with record_lagrangian: eager iterations, z kept, L recorded after
  // each completed iteration (the reference's run loop, solver.cpp:258-260).
  RunRecords run_recording(const RecordFn& cb) {
    using clk = std::chrono::steady_clock;
    // records of iteration k complete after iteration k+1 (lagged R-factor)
    auto deliver = [&](int64_t upto, const std::vector<double>& lag, const std::vector<double>& tms) {
      if (!cb || upto < 1) return;
      std::vector<double> rec(2 * static_cast<size_t>(upto));
      PDD_CUDA(cudaMemcpyAsync(rec.data(), R.rec.get(), sizeof(double) * rec.size(), cudaMemcpyDeviceToHost, R.st()));
      PDD_CUDA(cudaStreamSynchronize(R.st()));
      for (int64_t n = delivered_ + 1; n <= upto; ++n)
        cb(n, rec[2 * (n - 1)], rec[2 * (n - 1) + 1], n - 1 < static_cast<int64_t>(tms.size()) ? tms[n - 1] : 0.0,
           n - 1 < static_cast<int64_t>(lag.size()) ? lag[n - 1] : NAN);
      delivered_ = std::max(delivered_, upto);
    };
    delivered_ = 0;
    ensure_z();
    init_state();
    R.reset_ctl(0, cfg_.max_iters, cfg_.stop_rule, cfg_.tol_rf, cfg_.tol_re);
    std::vector<double> lag, tms;
    for (;;) {
      const auto t0 = clk::now();
      enqueue_iteration(static_cast<int>(iter_ & 1), true);
      PDD_CUDA(cudaStreamSynchronize(R.st()));
      const RunCtl c = R.read_ctl();
      if (c.iter == iter_) break;  // stopped before completing another iteration
      iter_ = c.iter;
      z_valid_ = true;
      tms.push_back(std::chrono::duration<double, std::milli>(clk::now() - t0).count());
      lag.push_back(lagrangian());
      if (c.stop) break;
      deliver(c.iter - 1, lag, tms);
    }
    enqueue_tail(static_cast<int>(iter_ & 1));
    PDD_CUDA(cudaStreamSynchronize(R.st()));
    const RunCtl c = R.read_ctl();
    RunRecords out;
    out.iterations = c.stop ? c.stop : c.iter;
    out.diverged_at = c.diverged;
    std::vector<double> rec(2 * static_cast<size_t>(out.iterations));
    if (out.iterations)
      PDD_CUDA(cudaMemcpyAsync(rec.data(), R.rec.get(), sizeof(double) * rec.size(), cudaMemcpyDeviceToHost, R.st()));
      PDD_CUDA(cudaStreamSynchronize(R.st()));
    for (int64_t n = 0; n < out.iterations; ++n) {
      out.rf.push_back(rec[2 * n]);
      out.re.push_back(rec[2 * n + 1]);
      out.t_ms.push_back(n < static_cast<int64_t>(tms.size()) ? tms[n] : 0.0);
      out.lag.push_back(n < static_cast<int64_t>(lag.size()) ? lag[n] : NAN);
    }
    deliver(out.iterations, lag, tms);
    iter_ = out.iterations;
    last_lag_ = out.lag;
    return out;
  }

  RunRecords run(const RecordFn& on_record) override {  // solver.cpp:216-267
    if (cfg_.record_lagrangian) return run_recording(on_record);
    SetupTimer tm;
    init_state();
    R.reset_ctl(0, cfg_.max_iters, cfg_.stop_rule, cfg_.tol_rf, cfg_.tol_re);
    tm.mark("run: init");
    RecordFeed feed{&on_record, 0, 0};
    const auto ms = drive(cfg_.max_iters, true, true, [&](const RunCtl& c, const std::vector<double>& ms_now) {
      // rf of iterate n is recorded by iteration n + 1's frame pass
      feed.upto(R.rec.template as<double>(), R.rec_cap, R.st(), c.stop ? c.stop : c.iter - 1, ms_now);
    });
    tm.mark("run: iterations");
    const RunCtl c = R.read_ctl();
    RunRecords out;
    out.iterations = c.stop ? c.stop : c.iter;
    out.diverged_at = c.diverged;
    std::vector<double> rec(2 * static_cast<size_t>(out.iterations));
    if (out.iterations)
      PDD_CUDA(cudaMemcpyAsync(rec.data(), R.rec.get(), sizeof(double) * rec.size(), cudaMemcpyDeviceToHost, R.st()));
      PDD_CUDA(cudaStreamSynchronize(R.st()));
    for (int64_t n = 0; n < out.iterations; ++n) {
      out.rf.push_back(rec[2 * n]);
      out.re.push_back(rec[2 * n + 1]);
      out.t_ms.push_back(ms.empty() ? 0.0 : ms[std::min<size_t>(n / 2, ms.size() - 1)] / 2.0);
    }
    feed.upto(R.rec.template as<double>(), R.rec_cap, R.st(), out.iterations, ms);
    iter_ = out.iterations;
    z_valid_ = false;
    last_lag_.clear();
    return out;
  }

  std::vector<double> lagrangian_history() const override { return last_lag_; }

  void iterate(int n) override {
    if (n <= 0) return;
    R.reset_ctl(static_cast<int>(iter_), static_cast<int>(iter_) + n, 2, cfg_.tol_rf, cfg_.tol_re);
    drive(n, false);
    z_valid_ = false;
  }

  double iterate_timed(int n) override {
    if (n <= 0) return 0.0;
    R.reset_ctl(static_cast<int>(iter_), static_cast<int>(iter_) + n, 2, cfg_.tol_rf, cfg_.tol_re);
    ensure_graphs();
    cudaEvent_t e0, e1;
    PDD_CUDA(cudaEventCreate(&e0));
    PDD_CUDA(cudaEventCreate(&e1));
    PDD_CUDA(cudaEventRecord(e0, R.st()));
    drive(n, false, false);  // exactly n iterations (no trailing R-factor pass)
    PDD_CUDA(cudaEventRecord(e1, R.st()));
    PDD_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    PDD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    z_valid_ = false;
    return ms;
  }

  void profile(int n, double* out) override {
    cudaEvent_t ev[4];
    cudaEvent_t e_start, e_end;
    for (auto& e : ev) PDD_CUDA(cudaEventCreate(&e));
    PDD_CUDA(cudaEventCreate(&e_start));
    PDD_CUDA(cudaEventCreate(&e_end));
    double fr = 0.0, ga = 0.0;
    R.reset_ctl(static_cast<int>(iter_), static_cast<int>(iter_) + n, 2, cfg_.tol_rf, cfg_.tol_re);
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

  double last_rf() override {
    const RunCtl c = R.read_ctl();
    if (c.iter < 1) return NAN;
    double rf = NAN;
    PDD_CUDA(cudaMemcpyAsync(&rf, R.rec.template as<double>() + 2 * ((c.iter - 1) % R.rec_cap), sizeof(double),
                             cudaMemcpyDeviceToHost, R.st()));
    PDD_CUDA(cudaStreamSynchronize(R.st()));
    return rf;
  }

  void get_state(double* u, double* z, double* gamma, double* v, double* lam, int64_t* iteration) override {
    cudaStream_t s = R.st();
    const int64_t nf = R.L.nfr * R.SS();
    if (u) download_c128<T>(U(iter_), R.L.img_elems, u, s);
    if (gamma) download_c128<T>(gamma_[iter_ & 1].get(), nf, gamma, s);
    if (z) {
      if (!z_valid_) {
        ensure_z();
        std::fill(z, z + 2 * nf, NAN);
      } else {
        download_c128<T>(z_.get(), nf, z, s);
      }
    }
    if (v) download_c128<T>(V(iter_), R.L.v_elems, v, s);
    if (lam) download_c128<T>(LAM(iter_), R.L.lam_elems, lam, s);
    if (iteration) *iteration = iter_;
  }

  void set_state(const double* u, const double* z, const double* gamma, const double* v, const double* lam,
                 int64_t iteration) override {
    cudaStream_t s = R.st();
    const int64_t nf = R.L.nfr * R.SS();
    iter_ = iteration;
    if (u) upload_cx<T>(U(iter_), u, R.L.img_elems, s);
    if (gamma) upload_cx<T>(gamma_[iter_ & 1].get(), gamma, nf, s);
    if (z) {
      ensure_z();
      upload_cx<T>(z_.get(), z, nf, s);
      z_valid_ = true;
    }
    if (v) upload_cx<T>(V(iter_), v, R.L.v_elems, s);
    if (lam) upload_cx<T>(LAM(iter_), lam, R.L.lam_elems, s);
  }

  void forward_frames(double* au) override {
    forward_into(bp_.as<cx<T>>());
    download_c128<T>(bp_.get(), R.L.nfr * R.SS(), au, R.st());
  }

  void merged(double* out) override {  // bp_ is per-iteration scratch
    R.merge_to_host(plan_, U(iter_), out, bp_.get(), bp_.bytes());
  }
  void sync() override { R.stream.sync(); }
  void* stream() const override { return R.st(); }
  // pack, vstep, sweep, R-factor sums + finalize (one launch when fused, else two), update pass,
  // RE sums + finalize (one launch when fused, else three)
  int64_t kernel_launches_per_iteration() const override { return R.fused_finalize() ? 6 : 9; }

 private:
  Plan plan_;
  NonblindConfig cfg_;
  PoolUser pool_;  // before every DevMem: the pool outlives them
  RankData<T> R;
  StateLayout layout_;
  DevMem probe_, probe64_, gamma_[2], bp_, u_[2], v_[2], lam_[2], s_, denom_, z_;
  DevMem lag_fr_, lag_pr_, lag_glob_;
  std::vector<double> last_lag_;
  Graph full_[2], tail_[2], one_[2];
  int64_t iter_ = 0;
  int64_t delivered_ = 0;  // run_recording: records handed to the callback
  bool z_valid_ = false;
};

}  // namespace

std::unique_ptr<NonblindGpu> make_nonblind(const Plan& plan, const DataSpec& data, const double* probe,
                                           const NonblindConfig& cfg, const double* pin_ones, int dtype,
                                           int device, Comm* comm) {
  DeviceGuard guard(device);
  if (dtype == 2) return std::make_unique<Nonblind<double>>(plan, data, probe, cfg, pin_ones, device, comm);
  return std::make_unique<Nonblind<float>>(plan, data, probe, cfg, pin_ones, device, comm);
}

}  // namespace pdd
