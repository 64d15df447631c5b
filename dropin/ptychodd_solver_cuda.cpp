// Drop-in definitions of the reference's solver API over the B200 C-ABI.
//
// Compiled against the reference's own headers (proj/include/ptychodd/
// solver.hpp, blind.hpp), this file defines every member of
// ptychodd::NonblindSolver and ptychodd::BlindSolver, NonblindConfig::validate,
// BlindConfig::validate and the blind free functions disk_support_mask /
// estimate_support_mask -- i.e. it replaces proj/src/solver.cpp and
// proj/src/blind.cpp.  Everything numeric runs in libptychodd_cuda.so
// (include/ptychodd_cuda.h); what stays here is the host bookkeeping the
// reference constructors do (validation, frame partition, pins) and the
// conversions between the reference's value types and the C-ABI's packed
// arrays.  Linking the reference's unit tests (test_solver.cpp,
// test_blind.cpp) against this file instead of solver.cpp/blind.cpp is the
// drop-in proof ("Callers"); dropin/build_dropin.sh.
//
// The solver objects stay host-only (the reference classes have no slot for a
// device handle): each entry point opens a device handle, works, and closes
// it.  The handle spans min(threads or D, D, visible GPUs) devices
// (devices_for); run() streams on_iteration records while the device loop
// runs.  run() is one handle for the whole solve; step() round-trips the state
// (the correctness path, as in the reference's API).  Precision: float64 by
// default (the reference's), PTYCHODD_CUDA_DTYPE=f32 selects complex64.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <exception>
#include <functional>
#include <memory>
#include <string>

#include "ptychodd/blind.hpp"
#include "ptychodd/solver.hpp"
#include "ptychodd/stagm.hpp"
#include "ptychodd_cuda.hpp"

namespace ptychodd {
namespace {

using Clock = std::chrono::steady_clock;

int dtype() {
  const char* e = std::getenv("PTYCHODD_CUDA_DTYPE");
  return (e && std::string(e) == "f32") ? PDD_F32 : PDD_F64;
}
int device() {
  const char* e = std::getenv("PTYCHODD_CUDA_DEVICE");
  return e ? std::atoi(e) : 0;
}

// The reference's worker count (NonblindConfig::threads / BlindConfig::threads,
// 0 = one worker per subdomain, solver.cpp:122) mapped onto GPUs: G =
// min(threads or D, D, visible devices) ranks on consecutive devices from
// PTYCHODD_CUDA_DEVICE.  PTYCHODD_CUDA_DEVICES="0,0,..." lists them explicitly
// (a repeated device runs several ranks on one GPU through the host
// transport).  Results do not depend on G (bit-identical iterates).
std::vector<int32_t> devices_for(int threads, int D) {
  std::vector<int32_t> out;
  if (const char* e = std::getenv("PTYCHODD_CUDA_DEVICES")) {
    std::string l(e);
    size_t a = 0;
    while (a < l.size()) {
      const size_t b = l.find(',', a);
      out.push_back(std::atoi(l.substr(a, b == std::string::npos ? std::string::npos : b - a).c_str()));
      if (b == std::string::npos) break;
      a = b + 1;
    }
    if (static_cast<int>(out.size()) > D) out.resize(static_cast<size_t>(D));
    if (!out.empty()) return out;
  }
  int32_t n = 0;
  if (pdd_device_count(&n) != PDD_OK || n < 1) n = 1;
  const int base = device();
  int G = threads > 0 ? threads : D;
  G = std::max(1, std::min({G, D, n - std::min(base, n - 1)}));
  for (int r = 0; r < G; ++r) out.push_back(base + r);
  return out;
}

// ConvergenceRecord::t_sub_ms (solver.cpp:243-249) on the device: a rank runs
// all of its subdomains in one fused launch per kernel, so subdomain d is
// charged its rank's measured iteration time in proportion to its frame count
// (the frame kernel is ~90 % of an iteration and its cost is per frame),
// share[d] = J_d / sum of J over the subdomains of rank(d), rank(d) =
// floor(d G / D).  t_virtual_ms = max_d t_sub_ms[d] then models one GPU per
// subdomain exactly as the reference models one worker per subdomain;
// t_actual_ms stays the measured time of the iteration.
std::vector<double> frame_shares(const DecompositionPlan& plan, int G) {
  const int D = plan.D;
  G = std::max(1, std::min(G, D));
  std::vector<double> per_rank(static_cast<size_t>(G), 0.0), share(static_cast<size_t>(D), 1.0);
  auto rank_of = [&](int d) { return static_cast<int>((static_cast<int64_t>(d) * G) / D); };
  std::vector<double> jd(static_cast<size_t>(D), 0.0);
  for (int a : plan.frame_assignment)
    if (a >= 0 && a < D) jd[static_cast<size_t>(a)] += 1.0;
  for (int d = 0; d < D; ++d) per_rank[static_cast<size_t>(rank_of(d))] += jd[static_cast<size_t>(d)];
  for (int d = 0; d < D; ++d) {
    const double tot = per_rank[static_cast<size_t>(rank_of(d))];
    share[static_cast<size_t>(d)] = tot > 0.0 ? jd[static_cast<size_t>(d)] / tot : 1.0;
  }
  return share;
}
void fill_times(ConvergenceRecord& r, const std::vector<double>& share, double t_ms) {
  r.t_sub_ms.resize(share.size());
  for (size_t d = 0; d < share.size(); ++d) r.t_sub_ms[d] = t_ms * share[d];
  r.t_virtual_ms = share.empty() ? t_ms : *std::max_element(r.t_sub_ms.begin(), r.t_sub_ms.end());
  r.t_actual_ms = t_ms;
}

// run()'s per-iteration callback (solver.hpp:88) through pdd_*_run_cb: the
// C-ABI streams records while the device loop runs; an exception thrown by
// the caller's callback is held and rethrown once the run returns.
struct RecordTrampoline {
  const std::function<void(const ConvergenceRecord&)>* cb;
  std::vector<double> share;
  std::exception_ptr err;
  static void call(int64_t it, double rf, double re, double t_ms, double lag, void* user) {
    auto* self = static_cast<RecordTrampoline*>(user);
    if (self->err || !self->cb || !*self->cb) return;
    ConvergenceRecord r;
    r.iteration = it;
    r.rf = rf;
    r.re = re;
    if (!std::isnan(lag)) r.lagrangian = lag;
    fill_times(r, self->share, t_ms);
    try {
      (*self->cb)(r);
    } catch (...) {
      self->err = std::current_exception();
    }
  }
};

// C-ABI status -> the reference's exception types (DivergenceError included).
void check(int rc, int64_t iteration = 0) {
  if (rc == PDD_DIVERGENCE) throw DivergenceError(iteration);
  pdd_cuda::check(rc, iteration);
}

double* dp(std::vector<cdouble>& v) { return reinterpret_cast<double*>(v.data()); }
const double* dp(const std::vector<cdouble>& v) { return reinterpret_cast<const double*>(v.data()); }

struct PlanHandle {
  pdd_plan* h = nullptr;
  ~PlanHandle() { pdd_plan_destroy(h); }
};

// Any DecompositionPlan, exactly (ddplan.hpp:12-35) -> pdd_plan_from_arrays.
std::unique_ptr<PlanHandle> cuda_plan(const DecompositionPlan& plan) {
  const ScanGeometry& g = plan.geometry;
  std::vector<int64_t> pos;
  for (const auto& [r, c] : g.positions) {
    pos.push_back(r);
    pos.push_back(c);
  }
  std::vector<int32_t> assign(plan.frame_assignment.begin(), plan.frame_assignment.end());
  std::vector<int64_t> subs;
  for (const Region& s : plan.subdomains) subs.insert(subs.end(), {s.row_start, s.row_end, s.col_start, s.col_end});
  std::vector<int32_t> pairs;
  std::vector<int64_t> regions;
  for (const auto& p : plan.overlaps) {
    pairs.insert(pairs.end(), {p.d1, p.d2});
    regions.insert(regions.end(), {p.region.row_start, p.region.row_end, p.region.col_start, p.region.col_end});
  }
  auto out = std::make_unique<PlanHandle>();
  check(pdd_plan_from_arrays(g.frame_side, g.step, g.image_height, g.image_width, g.frame_count(), pos.data(),
                             plan.D, assign.data(), subs.data(), static_cast<int32_t>(plan.overlaps.size()),
                             pairs.data(), regions.data(), &out->h));
  return out;
}

// Partitioned frames back to one [J][s][s] stack in global scan order.
std::vector<double> global_frames(const std::vector<FrameStack>& parts, const DecompositionPlan& plan) {
  const int64_t s = plan.geometry.frame_side, ss = s * s;
  std::vector<double> f(static_cast<size_t>(plan.geometry.frame_count() * ss));
  for (int d = 0; d < plan.D; ++d)
    for (size_t k = 0; k < plan.frames_of[d].size(); ++k)
      std::copy(parts[d].frames[k].data().begin(), parts[d].frames[k].data().end(),
                f.begin() + plan.frames_of[d][k] * ss);
  return f;
}

// Subdomain-local pins (coverage == 0 or caller vacuum mask, solver.cpp:37-48)
// and their global image (the C-ABI's pin_ones argument).
std::vector<std::vector<uint8_t>> local_pins(const DecompositionPlan& plan, const RealField2D* pin_ones,
                                             const char* who) {
  RealField2D coverage = scan_coverage(plan.geometry);
  if (pin_ones && !(pin_ones->height() == coverage.height() && pin_ones->width() == coverage.width()))
    throw std::invalid_argument(std::string(who) + ": pin mask shape mismatch");
  std::vector<std::vector<uint8_t>> out;
  for (int d = 0; d < plan.D; ++d) {
    const Region& sub = plan.subdomains[d];
    std::vector<uint8_t> pin(static_cast<size_t>(sub.area()), 0);
    for (int64_t r = 0; r < sub.height(); ++r)
      for (int64_t c = 0; c < sub.width(); ++c) {
        const int64_t gr = sub.row_start + r, gc = sub.col_start + c;
        pin[r * sub.width() + c] = coverage.at(gr, gc) == 0.0 || (pin_ones && pin_ones->at(gr, gc) > 0.5);
      }
    out.push_back(std::move(pin));
  }
  return out;
}
std::vector<double> global_pins(const DecompositionPlan& plan, const std::vector<std::vector<uint8_t>>& pins) {
  const ScanGeometry& g = plan.geometry;
  std::vector<double> out(static_cast<size_t>(g.image_height * g.image_width), 0.0);
  for (int d = 0; d < plan.D; ++d) {
    const Region& sub = plan.subdomains[d];
    for (int64_t r = 0; r < sub.height(); ++r)
      for (int64_t c = 0; c < sub.width(); ++c)
        if (pins[d][r * sub.width() + c]) out[(sub.row_start + r) * g.image_width + sub.col_start + c] = 1.0;
  }
  return out;
}

std::vector<std::vector<RealField2D>> sqrt_frames(const std::vector<FrameStack>& parts, double* l1) {
  std::vector<std::vector<RealField2D>> out;
  *l1 = 0.0;
  for (const auto& st : parts) {
    std::vector<RealField2D> sf;
    for (const auto& f : st.frames) {
      RealField2D s(f.height(), f.width());
      for (int64_t i = 0; i < f.size(); ++i) {
        s[i] = std::sqrt(f[i]);
        *l1 += s[i];
      }
      sf.push_back(std::move(s));
    }
    out.push_back(std::move(sf));
  }
  return out;
}

// Packed state arrays <-> the reference's SolverState members.
struct Packed {
  std::vector<cdouble> u, z, gamma, v, lam;
};

Packed pack(const DecompositionPlan& plan, const std::vector<ComplexField2D>& u,
            const std::vector<std::vector<ComplexField2D>>& z, const std::vector<std::vector<ComplexField2D>>& gamma,
            const std::vector<ComplexField2D>& v, const std::vector<std::array<ComplexField2D, 2>>& lam) {
  Packed p;
  for (const auto& x : u) p.u.insert(p.u.end(), x.data().begin(), x.data().end());
  for (const auto& fr : z)
    for (const auto& x : fr) p.z.insert(p.z.end(), x.data().begin(), x.data().end());
  for (const auto& fr : gamma)
    for (const auto& x : fr) p.gamma.insert(p.gamma.end(), x.data().begin(), x.data().end());
  for (const auto& x : v) p.v.insert(p.v.end(), x.data().begin(), x.data().end());
  for (const auto& pr : lam)
    for (const auto& x : pr) p.lam.insert(p.lam.end(), x.data().begin(), x.data().end());
  (void)plan;
  return p;
}

Packed sized(const DecompositionPlan& plan) {
  Packed p;
  const int64_t ss = plan.geometry.frame_side * plan.geometry.frame_side;
  int64_t img = 0, ov = 0;
  for (const Region& s : plan.subdomains) img += s.area();
  for (const auto& pr : plan.overlaps) ov += pr.region.area();
  p.u.resize(static_cast<size_t>(img));
  p.z.resize(static_cast<size_t>(plan.geometry.frame_count() * ss));
  p.gamma.resize(p.z.size());
  p.v.resize(static_cast<size_t>(ov));
  p.lam.resize(static_cast<size_t>(2 * ov));
  return p;
}

void unpack(const DecompositionPlan& plan, const Packed& p, std::vector<ComplexField2D>& u,
            std::vector<std::vector<ComplexField2D>>& z, std::vector<std::vector<ComplexField2D>>& gamma,
            std::vector<ComplexField2D>& v, std::vector<std::array<ComplexField2D, 2>>& lam) {
  const int64_t s = plan.geometry.frame_side, ss = s * s;
  u.clear();
  z.clear();
  gamma.clear();
  v.clear();
  lam.clear();
  size_t o = 0, fo = 0;
  for (int d = 0; d < plan.D; ++d) {
    const Region& sub = plan.subdomains[d];
    u.emplace_back(sub.height(), sub.width(),
                   std::vector<cdouble>(p.u.begin() + o, p.u.begin() + o + sub.area()));
    o += static_cast<size_t>(sub.area());
    std::vector<ComplexField2D> zd, gd;
    for (size_t k = 0; k < plan.frames_of[d].size(); ++k, fo += ss) {
      zd.emplace_back(s, s, std::vector<cdouble>(p.z.begin() + fo, p.z.begin() + fo + ss));
      gd.emplace_back(s, s, std::vector<cdouble>(p.gamma.begin() + fo, p.gamma.begin() + fo + ss));
    }
    z.push_back(std::move(zd));
    gamma.push_back(std::move(gd));
  }
  size_t vo = 0, lo = 0;
  for (const auto& pr : plan.overlaps) {
    const int64_t h = pr.region.height(), w = pr.region.width(), n = h * w;
    v.emplace_back(h, w, std::vector<cdouble>(p.v.begin() + vo, p.v.begin() + vo + n));
    vo += n;
    std::array<ComplexField2D, 2> l;
    for (int side = 0; side < 2; ++side, lo += n)
      l[side] = ComplexField2D(h, w, std::vector<cdouble>(p.lam.begin() + lo, p.lam.begin() + lo + n));
    lam.push_back(std::move(l));
  }
}

pdd_nonblind_config c_config(const NonblindConfig& c) {
  return pdd_nonblind_config{c.epsilon,
                             c.eta,
                             c.r,
                             c.tol_rf,
                             c.tol_re,
                             c.max_iters,
                             c.stop_rule == StopRule::RFactor ? PDD_STOP_RFACTOR : PDD_STOP_RELATIVE_ERROR,
                             c.record_lagrangian ? 1 : 0,
                             c.threads};
}
pdd_blind_config c_config(const BlindConfig& c) {
  return pdd_blind_config{c.epsilon, c.eta, c.r, c.mu, c.gamma, c.support_energy, c.tol_rf, c.tol_re, c.max_iters,
                          c.stop_rule == StopRule::RFactor ? PDD_STOP_RFACTOR : PDD_STOP_RELATIVE_ERROR, c.threads};
}

// One device nonblind solver for the lifetime of a call.
struct NbHandle {
  pdd_nonblind* h = nullptr;
  std::unique_ptr<PlanHandle> plan;
  NbHandle(const DecompositionPlan& p, const std::vector<FrameStack>& frames, const ComplexField2D& probe,
           const NonblindConfig& cfg, const std::vector<std::vector<uint8_t>>& pins)
      : plan(cuda_plan(p)) {
    const auto f = global_frames(frames, p);
    const auto pin = global_pins(p, pins);
    const auto c = c_config(cfg);
    const auto devs = devices_for(cfg.threads, p.D);
    if (devs.size() == 1)
      check(pdd_nonblind_create(plan->h, f.data(), PDD_DATA_INTENSITY_F64, 0, dp(probe.data()), &c, pin.data(),
                                dtype(), devs[0], &h));
    else
      check(pdd_nonblind_create_multi(plan->h, f.data(), PDD_DATA_INTENSITY_F64, 0, dp(probe.data()), &c, pin.data(),
                                      dtype(), devs.data(), static_cast<int32_t>(devs.size()), &h));
  }
  ~NbHandle() { pdd_nonblind_destroy(h); }
};

struct BlHandle {
  pdd_blind* h = nullptr;
  std::unique_ptr<PlanHandle> plan;
  BlHandle(const DecompositionPlan& p, const std::vector<FrameStack>& frames, const BlindConfig& cfg,
           const std::vector<std::vector<uint8_t>>& pins) : plan(cuda_plan(p)) {
    const auto f = global_frames(frames, p);
    const auto pin = global_pins(p, pins);
    const auto c = c_config(cfg);
    const double* mask = cfg.support_mask.size() > 0 ? cfg.support_mask.data().data() : nullptr;
    const auto devs = devices_for(cfg.threads, p.D);
    if (devs.size() == 1)
      check(pdd_blind_create(plan->h, f.data(), PDD_DATA_INTENSITY_F64, 0, &c, mask, pin.data(), dtype(), devs[0],
                             &h));
    else
      check(pdd_blind_create_multi(plan->h, f.data(), PDD_DATA_INTENSITY_F64, 0, &c, mask, pin.data(), dtype(),
                                   devs.data(), static_cast<int32_t>(devs.size()), &h));
  }
  ~BlHandle() { pdd_blind_destroy(h); }
};

std::vector<ComplexField2D> split_images(const DecompositionPlan& plan, const std::vector<cdouble>& flat) {
  std::vector<ComplexField2D> out;
  size_t o = 0;
  for (const Region& s : plan.subdomains) {
    out.emplace_back(s.height(), s.width(), std::vector<cdouble>(flat.begin() + o, flat.begin() + o + s.area()));
    o += static_cast<size_t>(s.area());
  }
  return out;
}

std::vector<ConvergenceRecord> records_of(const std::vector<double>& rec, int64_t n, const std::vector<double>& share,
                                          const std::vector<double>& lag) {
  std::vector<ConvergenceRecord> out;
  for (int64_t k = 0; k < n; ++k) {
    ConvergenceRecord r;
    r.iteration = k + 1;
    r.rf = rec[3 * k];
    r.re = rec[3 * k + 1];
    if (k < static_cast<int64_t>(lag.size())) r.lagrangian = lag[k];
    fill_times(r, share, rec[3 * k + 2]);
    out.push_back(std::move(r));
  }
  return out;
}

}  // namespace

// ---------------------------------------------------------------- nonblind

void NonblindConfig::validate() const {  // solver.cpp:24-31
  stagm::check_epsilon(epsilon);
  if (eta <= 0.0 || r <= 0.0) throw std::invalid_argument("NonblindConfig: eta, r must be > 0");
  if (max_iters < 1) throw std::invalid_argument("NonblindConfig: max_iters >= 1");
  if (tol_rf <= 0.0 || tol_re <= 0.0) throw std::invalid_argument("NonblindConfig: tolerances must be > 0");
  if (threads < 0) throw std::invalid_argument("NonblindConfig: threads >= 0");
}

NonblindSolver::NonblindSolver(const DecompositionPlan& plan, const FrameStack& frames, const ComplexField2D& probe,
                               const NonblindConfig& config, const RealField2D* pin_ones)
    : plan_(plan), probe_(probe), config_(config) {
  config_.validate();
  frames.validate();
  frames_ = partition_frames(frames, plan_);
  pin_ = local_pins(plan_, pin_ones, "NonblindSolver");
  sqrt_f_ = sqrt_frames(frames_, &sqrt_f_l1_);
  // The device constructor performs the remaining checks (probe shape, the
  // singular-illumination runtime_error of solver.cpp:73-75).
  NbHandle probe_check(plan_, frames_, probe_, config_, pin_);
}

SolverState NonblindSolver::init_state() const {  // solver.cpp:96-116
  NbHandle g(plan_, frames_, probe_, config_, pin_);
  check(pdd_nonblind_init_state(g.h));
  Packed p = sized(plan_);
  check(pdd_nonblind_get_state(g.h, dp(p.u), dp(p.z), dp(p.gamma), dp(p.v), dp(p.lam), nullptr));
  SolverState s;
  unpack(plan_, p, s.u, s.z, s.gamma, s.v, s.lambda);
  s.iteration = 0;
  return s;
}

std::vector<double> NonblindSolver::step(SolverState& state,
                                         std::vector<std::vector<ComplexField2D>>& au) const {  // solver.cpp:118-205
  const auto t0 = Clock::now();
  NbHandle g(plan_, frames_, probe_, config_, pin_);
  Packed in = pack(plan_, state.u, state.z, state.gamma, state.v, state.lambda);
  check(pdd_nonblind_set_state(g.h, dp(in.u), dp(in.z), dp(in.gamma), dp(in.v), dp(in.lam), state.iteration));
  check(pdd_nonblind_step(g.h, 1));
  Packed p = sized(plan_);
  int64_t it = 0;
  check(pdd_nonblind_get_state(g.h, dp(p.u), dp(p.z), dp(p.gamma), dp(p.v), dp(p.lam), &it));
  unpack(plan_, p, state.u, state.z, state.gamma, state.v, state.lambda);
  state.iteration = it;
  std::vector<cdouble> a(p.z.size());
  check(pdd_nonblind_forward(g.h, dp(a)));
  const int64_t s = plan_.geometry.frame_side, ss = s * s;
  au.assign(static_cast<size_t>(plan_.D), {});
  size_t o = 0;
  for (int d = 0; d < plan_.D; ++d)
    for (size_t k = 0; k < plan_.frames_of[d].size(); ++k, o += ss)
      au[d].emplace_back(s, s, std::vector<cdouble>(a.begin() + o, a.begin() + o + ss));
  const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
  return std::vector<double>(static_cast<size_t>(plan_.D), ms);
}

double NonblindSolver::r_factor_of(const std::vector<std::vector<ComplexField2D>>& au) const {  // solver.cpp:207-214
  // host metric over the caller's host arrays (run() computes RF on the device)
  double num = 0.0;
  for (int d = 0; d < plan_.D; ++d)
    for (size_t j = 0; j < au[d].size(); ++j)
      for (int64_t i = 0; i < au[d][j].size(); ++i) num += std::fabs(std::abs(au[d][j][i]) - sqrt_f_[d][j][i]);
  return num / sqrt_f_l1_;
}

NonblindResult NonblindSolver::run(const std::function<void(const ConvergenceRecord&)>& on_iteration) const {
  NbHandle g(plan_, frames_, probe_, config_, pin_);
  std::vector<double> rec(3 * static_cast<size_t>(config_.max_iters));
  int64_t n = 0, div = 0;
  const std::vector<double> share = frame_shares(plan_, static_cast<int>(devices_for(config_.threads, plan_.D).size()));
  RecordTrampoline tr{&on_iteration, share, nullptr};
  check(pdd_nonblind_run_cb(g.h, on_iteration ? &RecordTrampoline::call : nullptr, &tr, &n, rec.data(), &div), div);
  if (tr.err) std::rethrow_exception(tr.err);
  std::vector<double> lag;
  if (config_.record_lagrangian) {
    int64_t nl = 0;
    lag.resize(static_cast<size_t>(std::max<int64_t>(n, 1)));
    check(pdd_nonblind_lagrangian_history(g.h, lag.data(), static_cast<int64_t>(lag.size()), &nl));
    lag.resize(static_cast<size_t>(std::min(nl, n)));
  }
  NonblindResult out;
  out.records = records_of(rec, n, share, lag);
  Packed p = sized(plan_);
  check(pdd_nonblind_get_state(g.h, dp(p.u), nullptr, nullptr, nullptr, nullptr, nullptr));
  out.sub_solutions = split_images(plan_, p.u);
  const ScanGeometry& geo = plan_.geometry;
  out.merged = ComplexField2D(geo.image_height, geo.image_width);
  check(pdd_nonblind_merged(g.h, dp(out.merged.data())));
  out.iterations = n;
  if (n) {
    out.final_rf = out.records.back().rf;
    out.final_re = out.records.back().re;
  }
  return out;
}

// ---------------------------------------------------------------- blind

RealField2D disk_support_mask(int64_t side, double radius) {
  RealField2D m(side, side, 0.0);
  check(pdd_disk_support_mask(side, radius, m.data().data()));
  return m;
}

RealField2D estimate_support_mask(const ComplexField2D& probe_guess, double energy_fraction) {
  const int64_t side = probe_guess.height();
  RealField2D m(side, side, 0.0);
  check(pdd_estimate_support_mask(dp(probe_guess.data()), side, energy_fraction, m.data().data()));
  return m;
}

void BlindConfig::validate(int64_t frame_side) const {  // blind.cpp:29-43
  stagm::check_epsilon(epsilon);
  if (eta <= 0.0 || r <= 0.0 || mu <= 0.0 || gamma <= 0.0)
    throw std::invalid_argument("BlindConfig: eta, r, mu, gamma must be > 0");
  if (max_iters < 1) throw std::invalid_argument("BlindConfig: max_iters >= 1");
  if (tol_rf <= 0.0 || tol_re <= 0.0) throw std::invalid_argument("BlindConfig: tolerances must be > 0");
  if (support_mask.size() > 0) {
    if (support_mask.height() != frame_side || support_mask.width() != frame_side)
      throw std::invalid_argument("BlindConfig: support mask must be frame-sized");
    for (double m : support_mask.data())
      if (m != 0.0 && m != 1.0) throw std::invalid_argument("BlindConfig: support mask entries must be 0 or 1");
  }
}

BlindSolver::BlindSolver(const DecompositionPlan& plan, const FrameStack& frames, const BlindConfig& config,
                         const RealField2D* pin_ones)
    : plan_(plan), config_(config) {
  config_.validate(plan.geometry.frame_side);
  frames.validate();
  frames_ = partition_frames(frames, plan_);
  pin_ = local_pins(plan_, pin_ones, "BlindSolver");
  sqrt_f_ = sqrt_frames(frames_, &sqrt_f_l1_);
  if (sqrt_f_l1_ <= 0.0) throw std::invalid_argument("BlindSolver: all-zero measurements");
  // w0 and the support mask as the device solver derives them (blind.cpp:123-156)
  BlHandle g(plan_, frames_, config_, pin_);
  const int64_t s = plan_.geometry.frame_side;
  mask_ = RealField2D(s, s, 0.0);
  w0_ = ComplexField2D(s, s);
  check(pdd_blind_get_probe(g.h, nullptr, nullptr, mask_.data().data(), dp(w0_.data())));
}

namespace {
struct BlindPacked {
  std::vector<cdouble> w, wc, delta;
  Packed rest;
};
BlindPacked blind_sized(const DecompositionPlan& plan) {
  BlindPacked b;
  const int64_t ss = plan.geometry.frame_side * plan.geometry.frame_side;
  b.w.resize(static_cast<size_t>(ss));
  b.wc.resize(static_cast<size_t>(plan.D * ss));
  b.delta.resize(b.wc.size());
  b.rest = sized(plan);
  return b;
}
void blind_unpack(const DecompositionPlan& plan, const BlindPacked& b, BlindState& st) {
  const int64_t s = plan.geometry.frame_side, ss = s * s;
  st.w = ComplexField2D(s, s, b.w);
  st.w_copies.clear();
  st.delta.clear();
  for (int d = 0; d < plan.D; ++d) {
    st.w_copies.emplace_back(s, s, std::vector<cdouble>(b.wc.begin() + d * ss, b.wc.begin() + (d + 1) * ss));
    st.delta.emplace_back(s, s, std::vector<cdouble>(b.delta.begin() + d * ss, b.delta.begin() + (d + 1) * ss));
  }
  unpack(plan, b.rest, st.u, st.z, st.gamma, st.v, st.lambda);
}
}  // namespace

BlindState BlindSolver::init_state() const {  // blind.cpp:169-192
  BlHandle g(plan_, frames_, config_, pin_);
  check(pdd_blind_init_state(g.h, nullptr));  // the device solver's own w0 (== w0_)
  BlindPacked b = blind_sized(plan_);
  check(pdd_blind_get_state(g.h, dp(b.w), dp(b.wc), dp(b.delta), dp(b.rest.u), dp(b.rest.z), dp(b.rest.gamma),
                            dp(b.rest.v), dp(b.rest.lam), nullptr));
  BlindState st;
  blind_unpack(plan_, b, st);
  st.iteration = 0;
  return st;
}

std::vector<double> BlindSolver::step(BlindState& state) const {  // blind.cpp:194-296
  const auto t0 = Clock::now();
  BlHandle g(plan_, frames_, config_, pin_);
  std::vector<cdouble> wc, delta;
  for (const auto& x : state.w_copies) wc.insert(wc.end(), x.data().begin(), x.data().end());
  for (const auto& x : state.delta) delta.insert(delta.end(), x.data().begin(), x.data().end());
  Packed in = pack(plan_, state.u, state.z, state.gamma, state.v, state.lambda);
  check(pdd_blind_set_state(g.h, dp(state.w.data()), dp(wc), dp(delta), dp(in.u), dp(in.z), dp(in.gamma), dp(in.v),
                            dp(in.lam), state.iteration));
  check(pdd_blind_step(g.h, 1));
  BlindPacked b = blind_sized(plan_);
  int64_t it = 0;
  check(pdd_blind_get_state(g.h, dp(b.w), dp(b.wc), dp(b.delta), dp(b.rest.u), dp(b.rest.z), dp(b.rest.gamma),
                            dp(b.rest.v), dp(b.rest.lam), &it));
  blind_unpack(plan_, b, state);
  state.iteration = it;
  const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
  return std::vector<double>(static_cast<size_t>(plan_.D), ms);
}

BlindResult BlindSolver::run(const std::function<void(const ConvergenceRecord&)>& on_iteration) const {
  BlHandle g(plan_, frames_, config_, pin_);
  check(pdd_blind_init_state(g.h, nullptr));  // the device solver's own w0 (== w0_)
  std::vector<double> rec(3 * static_cast<size_t>(config_.max_iters));
  int64_t n = 0, div = 0;
  const std::vector<double> share = frame_shares(plan_, static_cast<int>(devices_for(config_.threads, plan_.D).size()));
  RecordTrampoline tr{&on_iteration, share, nullptr};
  check(pdd_blind_run_cb(g.h, on_iteration ? &RecordTrampoline::call : nullptr, &tr, &n, rec.data(), &div), div);
  if (tr.err) std::rethrow_exception(tr.err);
  BlindResult out;
  out.records = records_of(rec, n, share, {});
  const int64_t s = plan_.geometry.frame_side;
  out.probe = ComplexField2D(s, s);
  out.probe_fourier = ComplexField2D(s, s);
  out.support_mask = RealField2D(s, s, 0.0);
  check(pdd_blind_get_probe(g.h, dp(out.probe.data()), dp(out.probe_fourier.data()), out.support_mask.data().data(),
                            nullptr));
  Packed p = sized(plan_);
  check(pdd_blind_get_state(g.h, nullptr, nullptr, nullptr, dp(p.u), nullptr, nullptr, nullptr, nullptr, nullptr));
  out.sub_solutions = split_images(plan_, p.u);
  const ScanGeometry& geo = plan_.geometry;
  out.merged = ComplexField2D(geo.image_height, geo.image_width);
  check(pdd_blind_merged(g.h, dp(out.merged.data())));
  out.iterations = n;
  if (n) {
    out.final_rf = out.records.back().rf;
    out.final_re = out.records.back().re;
  }
  return out;
}

}  // namespace ptychodd
