// ORACLE TEST INFRASTRUCTURE — not product code.
//
// extern "C" wrapper over the UNMODIFIED reference C++ API
// (/root/reference/proj/include/ptychodd/*.hpp), compiled together with the
// reference sources by oracle/build_ref.sh into oracle/_ref/libptychodd_ref.so.
// Python tests (ctypes) use it to pin the numpy restatement (oracle/od2p.py)
// and to generate golden fixtures; bench.py's reference arm uses it as the CPU
// baseline.  Nothing in the product path loads this library.
//
// Extensions that the reference API cannot express are
// built here from the reference's public types without touching its sources:
//   * plan_grid: a 2-D block plan built with the same rules as plan_stripes
//     (reference proj/src/ddplan.cpp:28-94): union-of-windows subdomains,
//     all pairwise intersections in d1<d2 order, local raster geometries.
//   * a blind driver with a caller-chosen initial probe: public init_state(),
//     overwrite w / w_copies / z, then the public step(); the loop restates
//     BlindSolver::run (proj/src/blind.cpp:298-358).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "ptychodd/blind.hpp"
#include "ptychodd/ddplan.hpp"
#include "ptychodd/fft.hpp"
#include "ptychodd/forward.hpp"
#ifdef REF_HAVE_IO
#include "ptychodd/io.hpp"
#endif
#include "ptychodd/metrics.hpp"
#include "ptychodd/simulate.hpp"
#include "ptychodd/solver.hpp"
#include "ptychodd/stagm.hpp"

using namespace ptychodd;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const DivergenceError& e) {
    return fail(e, 4);
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::out_of_range& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

ComplexField2D cfield(const double* p, int64_t h, int64_t w) {
  ComplexField2D f(h, w);
  std::memcpy(static_cast<void*>(f.data().data()), p, sizeof(double) * 2 * h * w);
  return f;
}
RealField2D rfield(const double* p, int64_t h, int64_t w) {
  RealField2D f(h, w);
  std::memcpy(f.data().data(), p, sizeof(double) * h * w);
  return f;
}
double* put(double* dst, const ComplexField2D& f) {
  std::memcpy(dst, f.data().data(), sizeof(double) * 2 * f.size());
  return dst + 2 * f.size();
}
double* put(double* dst, const RealField2D& f) {
  std::memcpy(dst, f.data().data(), sizeof(double) * f.size());
  return dst + f.size();
}

ScanGeometry geometry_from(int64_t H, int64_t W, int64_t s, int64_t step, const int64_t* pos,
                           int64_t J) {
  ScanGeometry g;
  g.frame_side = s;
  g.step = step;
  g.image_height = H;
  g.image_width = W;
  g.grid_rows = 1;
  g.grid_cols = J;
  for (int64_t j = 0; j < J; ++j) g.positions.emplace_back(pos[2 * j], pos[2 * j + 1]);
  return g;
}

std::vector<ComplexField2D> frames_from(const double* p, int64_t J, int64_t s) {
  std::vector<ComplexField2D> v;
  for (int64_t j = 0; j < J; ++j) v.push_back(cfield(p + 2 * s * s * j, s, s));
  return v;
}

// ---- 2-D block plan (extension; same rules as plan_stripes) ----------------
std::vector<int64_t> blocks(int64_t lines, int n) {
  std::vector<int64_t> b(static_cast<size_t>(n) + 1, 0);
  const int64_t base = lines / n, extra = lines % n;
  for (int i = 0; i < n; ++i) b[i + 1] = b[i] + base + (i < extra ? 1 : 0);
  return b;
}

DecompositionPlan plan_grid(const ScanGeometry& g, int Dr, int Dc) {
  g.validate();
  if (Dr < 1 || Dc < 1) throw std::invalid_argument("plan_grid: Dr, Dc must be >= 1");
  if (Dr > g.grid_rows || Dc > g.grid_cols)
    throw std::invalid_argument("plan_grid: block count exceeds the scan frame-line count");
  const auto rb = blocks(g.grid_rows, Dr), cb = blocks(g.grid_cols, Dc);
  DecompositionPlan plan;
  plan.D = Dr * Dc;
  plan.geometry = g;
  plan.frame_assignment.resize(static_cast<size_t>(g.frame_count()));
  plan.frames_of.resize(static_cast<size_t>(plan.D));
  for (int64_t j = 0; j < g.frame_count(); ++j) {
    const int64_t i = j / g.grid_cols, c = j % g.grid_cols;
    const int bi = static_cast<int>(std::upper_bound(rb.begin() + 1, rb.end(), i) - rb.begin() - 1);
    const int bj = static_cast<int>(std::upper_bound(cb.begin() + 1, cb.end(), c) - cb.begin() - 1);
    const int d = bi * Dc + bj;
    plan.frame_assignment[j] = d;
    plan.frames_of[d].push_back(j);
  }
  for (int d = 0; d < plan.D; ++d) {
    Region sub = g.window(plan.frames_of[d].front());
    for (int64_t j : plan.frames_of[d]) {
      Region w = g.window(j);
      sub.row_start = std::min(sub.row_start, w.row_start);
      sub.row_end = std::max(sub.row_end, w.row_end);
      sub.col_start = std::min(sub.col_start, w.col_start);
      sub.col_end = std::max(sub.col_end, w.col_end);
    }
    plan.subdomains.push_back(sub);
  }
  for (int d1 = 0; d1 < plan.D; ++d1)
    for (int d2 = d1 + 1; d2 < plan.D; ++d2)
      if (plan.subdomains[d1].intersects(plan.subdomains[d2]))
        plan.overlaps.push_back({d1, d2, plan.subdomains[d1].intersection(plan.subdomains[d2])});
  for (int d = 0; d < plan.D; ++d) {
    const Region& sub = plan.subdomains[d];
    const int bi = d / Dc, bj = d % Dc;
    ScanGeometry local;
    local.frame_side = g.frame_side;
    local.step = g.step;
    local.image_height = sub.height();
    local.image_width = sub.width();
    local.grid_rows = rb[bi + 1] - rb[bi];
    local.grid_cols = cb[bj + 1] - cb[bj];
    for (int64_t j : plan.frames_of[d]) {
      auto [r, c] = g.positions[j];
      local.positions.emplace_back(r - sub.row_start, c - sub.col_start);
    }
    local.validate();
    plan.local_geometries.push_back(std::move(local));
  }
  return plan;
}

}  // namespace

extern "C" {

// Plan spec shared by every solver entry point.
//   kind 0: plan_stripes(make_raster_scan(H,W,s,step), D, axis) (axis 0 Auto, 1 Columns, 2 Rows)
//   kind 1: plan_grid(..., Dr, Dc)
struct RefPlanSpec {
  int64_t H, W, s, step;
  int32_t kind, D, Dr, Dc, axis;
};

struct RefNonblindCfg {
  double epsilon, eta, r, tol_rf, tol_re;
  int32_t max_iters, stop_rule, record_lagrangian, threads;
};

struct RefBlindCfg {
  double epsilon, eta, r, mu, gamma, support_energy, tol_rf, tol_re;
  int32_t max_iters, stop_rule, threads, has_mask;
};

const char* ref_last_error() { return g_err.c_str(); }

static DecompositionPlan make_plan(const RefPlanSpec* ps) {
  ScanGeometry g = make_raster_scan(ps->H, ps->W, ps->s, ps->step);
  if (ps->kind == 1) return plan_grid(g, ps->Dr, ps->Dc);
  SplitAxis ax = ps->axis == 1 ? SplitAxis::Columns : ps->axis == 2 ? SplitAxis::Rows : SplitAxis::Auto;
  return plan_stripes(g, ps->D, ax);
}

// Plan introspection.  counts = {D, J, n_overlaps}; buffers sized by the caller
// after a first call with null buffers.
int ref_plan(const RefPlanSpec* ps, int64_t* counts, int64_t* positions, int32_t* assignment,
             int64_t* subdomains, int32_t* pairs, int64_t* regions, int64_t* local_grid) {
  return guard([&] {
    DecompositionPlan p = make_plan(ps);
    counts[0] = p.D;
    counts[1] = p.geometry.frame_count();
    counts[2] = static_cast<int64_t>(p.overlaps.size());
    if (!positions) return;
    for (int64_t j = 0; j < p.geometry.frame_count(); ++j) {
      positions[2 * j] = p.geometry.positions[j].first;
      positions[2 * j + 1] = p.geometry.positions[j].second;
      assignment[j] = p.frame_assignment[j];
    }
    for (int d = 0; d < p.D; ++d) {
      const Region& r = p.subdomains[d];
      int64_t* o = subdomains + 4 * d;
      o[0] = r.row_start; o[1] = r.row_end; o[2] = r.col_start; o[3] = r.col_end;
      local_grid[2 * d] = p.local_geometries[d].grid_rows;
      local_grid[2 * d + 1] = p.local_geometries[d].grid_cols;
    }
    for (size_t q = 0; q < p.overlaps.size(); ++q) {
      pairs[2 * q] = p.overlaps[q].d1;
      pairs[2 * q + 1] = p.overlaps[q].d2;
      const Region& r = p.overlaps[q].region;
      int64_t* o = regions + 4 * q;
      o[0] = r.row_start; o[1] = r.row_end; o[2] = r.col_start; o[3] = r.col_end;
    }
  });
}

int ref_fft2(double* data, int64_t h, int64_t w, int inverse) {
  return guard([&] {
    ComplexField2D f = cfield(data, h, w);
    if (inverse) ifft2_normalized_inplace(f); else fft2_normalized_inplace(f);
    put(data, f);
  });
}

int ref_forward(const double* probe, int64_t s, const double* image, int64_t H, int64_t W,
                const int64_t* pos, int64_t J, double* out) {
  return guard([&] {
    auto fr = forward(cfield(probe, s, s), cfield(image, H, W), geometry_from(H, W, s, 1, pos, J));
    for (const auto& f : fr) out = put(out, f);
  });
}

int ref_adjoint(const double* probe, int64_t s, const double* frames, const int64_t* pos, int64_t J,
                int64_t H, int64_t W, double* out) {
  return guard([&] {
    put(out, adjoint(cfield(probe, s, s), frames_from(frames, J, s), geometry_from(H, W, s, 1, pos, J)));
  });
}

int ref_illumination_density(const double* probe, int64_t s, const int64_t* pos, int64_t J,
                             int64_t H, int64_t W, double* out) {
  return guard([&] { put(out, illumination_density(cfield(probe, s, s), geometry_from(H, W, s, 1, pos, J))); });
}

int ref_probe_density(const double* image, int64_t H, int64_t W, const int64_t* pos, int64_t J,
                      int64_t s, double* out) {
  return guard([&] { put(out, probe_density(cfield(image, H, W), geometry_from(H, W, s, 1, pos, J))); });
}

int ref_adjoint_probe(const double* image, int64_t H, int64_t W, const double* frames,
                      const int64_t* pos, int64_t J, int64_t s, double* out) {
  return guard([&] {
    put(out, adjoint_probe(cfield(image, H, W), frames_from(frames, J, s), geometry_from(H, W, s, 1, pos, J)));
  });
}

int ref_pixel_prox(const double* y, const double* b, int64_t n, double lambda, double eps, double* out) {
  return guard([&] {
    for (int64_t i = 0; i < n; ++i) {
      cdouble z = stagm::pixel_prox(cdouble(y[2 * i], y[2 * i + 1]), b[i], lambda, eps);
      out[2 * i] = z.real();
      out[2 * i + 1] = z.imag();
    }
  });
}

int ref_pixel_value_gradient(const double* x, const double* b, int64_t n, double eps, double* val,
                             double* grad) {
  return guard([&] {
    for (int64_t i = 0; i < n; ++i) {
      const cdouble xi(x[2 * i], x[2 * i + 1]);
      val[i] = stagm::pixel_value(xi, b[i], eps);
      const cdouble g = stagm::pixel_gradient(xi, b[i], eps);
      grad[2 * i] = g.real();
      grad[2 * i + 1] = g.imag();
    }
  });
}

static FrameStack stack_from(const DecompositionPlan& plan, const double* f) {
  FrameStack fs;
  fs.geometry = plan.geometry;
  const int64_t s = plan.geometry.frame_side;
  for (int64_t j = 0; j < plan.geometry.frame_count(); ++j) fs.frames.push_back(rfield(f + s * s * j, s, s));
  return fs;
}

static NonblindConfig nb_cfg(const RefNonblindCfg* c) {
  NonblindConfig cfg;
  cfg.epsilon = c->epsilon;
  cfg.eta = c->eta;
  cfg.r = c->r;
  cfg.max_iters = c->max_iters;
  cfg.tol_rf = c->tol_rf;
  cfg.tol_re = c->tol_re;
  cfg.stop_rule = c->stop_rule ? StopRule::RelativeError : StopRule::RFactor;
  cfg.record_lagrangian = c->record_lagrangian != 0;
  cfg.threads = c->threads;
  return cfg;
}

// NonblindSolver::run.  Outputs: merged [H,W] c128, subs (concatenated local
// images), rec [max_iters x 4] = (rf, re, lagrangian, t_actual_ms), n_iter.
int ref_nonblind_run(const RefPlanSpec* ps, const double* intensities, const double* probe,
                     const double* pin, const RefNonblindCfg* c, double* merged, double* subs,
                     double* rec, int64_t* n_iter) {
  return guard([&] {
    DecompositionPlan plan = make_plan(ps);
    const int64_t s = ps->s;
    RealField2D pin_f;
    if (pin) pin_f = rfield(pin, ps->H, ps->W);
    NonblindSolver solver(plan, stack_from(plan, intensities), cfield(probe, s, s), nb_cfg(c),
                          pin ? &pin_f : nullptr);
    NonblindResult res = solver.run();
    put(merged, res.merged);
    for (const auto& u : res.sub_solutions) subs = put(subs, u);
    for (const auto& r : res.records) {
      rec[0] = r.rf;
      rec[1] = r.re;
      rec[2] = r.lagrangian ? *r.lagrangian : NAN;
      rec[3] = r.t_actual_ms;
      rec += 4;
    }
    *n_iter = res.iterations;
  });
}

// init_state + nsteps x step.  State outputs concatenated in plan order:
// u (local images), z / gamma / au (per subdomain, per local frame), v (per pair),
// lambda (per pair, side 0 then side 1).  rf[k] = r_factor_of(au) after step k.
int ref_nonblind_steps(const RefPlanSpec* ps, const double* intensities, const double* probe,
                       const double* pin, const RefNonblindCfg* c, int64_t nsteps, double* u_out,
                       double* z_out, double* g_out, double* au_out, double* v_out, double* l_out,
                       double* rf_out) {
  return guard([&] {
    DecompositionPlan plan = make_plan(ps);
    const int64_t s = ps->s;
    RealField2D pin_f;
    if (pin) pin_f = rfield(pin, ps->H, ps->W);
    NonblindSolver solver(plan, stack_from(plan, intensities), cfield(probe, s, s), nb_cfg(c),
                          pin ? &pin_f : nullptr);
    SolverState st = solver.init_state();
    std::vector<std::vector<ComplexField2D>> au;
    for (int d = 0; d < plan.D; ++d) au.push_back(st.z[d]);
    for (int64_t k = 0; k < nsteps; ++k) {
      solver.step(st, au);
      if (rf_out) rf_out[k] = solver.r_factor_of(au);
    }
    for (const auto& u : st.u) u_out = put(u_out, u);
    for (int d = 0; d < plan.D; ++d)
      for (size_t j = 0; j < st.z[d].size(); ++j) {
        z_out = put(z_out, st.z[d][j]);
        g_out = put(g_out, st.gamma[d][j]);
        au_out = put(au_out, au[d][j]);
      }
    for (const auto& v : st.v) v_out = put(v_out, v);
    for (const auto& l : st.lambda) {
      l_out = put(l_out, l[0]);
      l_out = put(l_out, l[1]);
    }
  });
}

static BlindConfig bl_cfg(const RefBlindCfg* c, const double* mask, int64_t s) {
  BlindConfig cfg;
  cfg.epsilon = c->epsilon;
  cfg.eta = c->eta;
  cfg.r = c->r;
  cfg.mu = c->mu;
  cfg.gamma = c->gamma;
  cfg.support_energy = c->support_energy;
  cfg.tol_rf = c->tol_rf;
  cfg.tol_re = c->tol_re;
  cfg.max_iters = c->max_iters;
  cfg.stop_rule = c->stop_rule ? StopRule::RelativeError : StopRule::RFactor;
  cfg.threads = c->threads;
  if (c->has_mask && mask) cfg.support_mask = rfield(mask, s, s);
  return cfg;
}

// Blind solve.  w0 == nullptr runs the stock BlindSolver::run; otherwise the
// public init_state()/step() are driven with w, w_copies and z replaced by the
// caller's initial probe (loop restated from proj/src/blind.cpp:298-358).
// Outputs: merged, subs, probe (w), probe_fourier, mask_out, w0_out (the
// solver's own amplitude-based initial probe), rec [iters x 4], n_iter.
int ref_blind_run(const RefPlanSpec* ps, const double* intensities, const double* pin,
                  const RefBlindCfg* c, const double* mask_in, const double* w0, double* merged,
                  double* subs, double* probe_out, double* probe_fourier, double* mask_out,
                  double* w0_out, double* rec, int64_t* n_iter) {
  return guard([&] {
    DecompositionPlan plan = make_plan(ps);
    const int64_t s = ps->s;
    RealField2D pin_f;
    if (pin) pin_f = rfield(pin, ps->H, ps->W);
    FrameStack frames = stack_from(plan, intensities);
    BlindConfig cfg = bl_cfg(c, mask_in, s);
    BlindSolver solver(plan, frames, cfg, pin ? &pin_f : nullptr);
    put(mask_out, solver.support_mask());
    BlindState st0 = solver.init_state();
    put(w0_out, st0.w);
    if (!w0) {
      BlindResult res = solver.run();
      put(merged, res.merged);
      for (const auto& u : res.sub_solutions) subs = put(subs, u);
      put(probe_out, res.probe);
      put(probe_fourier, res.probe_fourier);
      for (const auto& r : res.records) {
        rec[0] = r.rf; rec[1] = r.re; rec[2] = NAN; rec[3] = r.t_actual_ms;
        rec += 4;
      }
      *n_iter = res.iterations;
      return;
    }
    BlindState st = std::move(st0);
    const ComplexField2D w_init = cfield(w0, s, s);
    st.w = w_init;
    for (int d = 0; d < plan.D; ++d) {
      st.w_copies[d] = w_init;
      st.z[d] = forward(w_init, st.u[d], plan.local_geometries[d]);
    }
    const auto parts = solver.partitioned_frames();
    std::vector<ComplexField2D> u_prev = st.u;
    int64_t n = 1;
    for (; n <= cfg.max_iters; ++n) {
      const auto t0 = std::chrono::steady_clock::now();
      solver.step(st);
      double re = 0.0;
      for (int d = 0; d < plan.D; ++d) {
        double diff = 0.0, norm = 0.0;
        for (int64_t i = 0; i < st.u[d].size(); ++i) {
          diff += std::norm(st.u[d][i] - u_prev[d][i]);
          norm += std::norm(st.u[d][i]);
        }
        re = std::max(re, std::sqrt(diff) / std::sqrt(norm));
      }
      u_prev = st.u;
      const double rf = r_factor(st.u, parts, st.w);
      if (!std::isfinite(rf) || !std::isfinite(re)) throw DivergenceError(n);
      rec[0] = rf; rec[1] = re; rec[2] = NAN;
      rec[3] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      rec += 4;
      const bool stop = cfg.stop_rule == StopRule::RFactor ? rf <= cfg.tol_rf : re <= cfg.tol_re;
      if (stop) break;
    }
    *n_iter = std::min<int64_t>(n, cfg.max_iters);
    put(merged, merge(st.u, plan));
    for (const auto& u : st.u) subs = put(subs, u);
    // result.probe = project_support(state.w) (blind.cpp:440): FFT, mask, IFFT.
    ComplexField2D spec = fft2_normalized(st.w);
    for (int64_t i = 0; i < spec.size(); ++i)
      if (solver.support_mask()[i] == 0.0) spec[i] = {0.0, 0.0};
    put(probe_fourier, spec);
    put(probe_out, ifft2_normalized(spec));
  });
}

// Blind init_state + nsteps x step (stock initial probe unless w0 given).
// Outputs: w, w_copies (D), delta (D), u, z, gamma, v, lambda.
int ref_blind_steps(const RefPlanSpec* ps, const double* intensities, const double* pin,
                    const RefBlindCfg* c, const double* mask_in, const double* w0, int64_t nsteps,
                    double* w_out, double* wc_out, double* delta_out, double* u_out, double* z_out,
                    double* g_out, double* v_out, double* l_out) {
  return guard([&] {
    DecompositionPlan plan = make_plan(ps);
    const int64_t s = ps->s;
    RealField2D pin_f;
    if (pin) pin_f = rfield(pin, ps->H, ps->W);
    BlindSolver solver(plan, stack_from(plan, intensities), bl_cfg(c, mask_in, s), pin ? &pin_f : nullptr);
    BlindState st = solver.init_state();
    if (w0) {
      const ComplexField2D w_init = cfield(w0, s, s);
      st.w = w_init;
      for (int d = 0; d < plan.D; ++d) {
        st.w_copies[d] = w_init;
        st.z[d] = forward(w_init, st.u[d], plan.local_geometries[d]);
      }
    }
    for (int64_t k = 0; k < nsteps; ++k) solver.step(st);
    put(w_out, st.w);
    for (int d = 0; d < plan.D; ++d) {
      wc_out = put(wc_out, st.w_copies[d]);
      delta_out = put(delta_out, st.delta[d]);
      u_out = put(u_out, st.u[d]);
      for (size_t j = 0; j < st.z[d].size(); ++j) {
        z_out = put(z_out, st.z[d][j]);
        g_out = put(g_out, st.gamma[d][j]);
      }
    }
    for (const auto& v : st.v) v_out = put(v_out, v);
    for (const auto& l : st.lambda) {
      l_out = put(l_out, l[0]);
      l_out = put(l_out, l[1]);
    }
  });
}

// Reference data generation helpers used to build fixtures.
int ref_simulate_frames(const double* probe, int64_t s, const double* sample, int64_t H, int64_t W,
                        int64_t step, double* out) {
  return guard([&] {
    ScanGeometry g = make_raster_scan(H, W, s, step);
    FrameStack f = simulate_frames(cfield(probe, s, s), cfield(sample, H, W), g);
    for (const auto& fr : f.frames) out = put(out, fr);
  });
}

int ref_add_poisson_noise(const double* in, int64_t J, int64_t s, double scale, uint64_t seed,
                          double* out) {
  return guard([&] {
    FrameStack f;
    f.geometry.frame_side = s;
    f.geometry.step = 1;
    f.geometry.image_height = s;
    f.geometry.image_width = s + J - 1;
    f.geometry.grid_rows = 1;
    f.geometry.grid_cols = J;
    for (int64_t j = 0; j < J; ++j) {
      f.geometry.positions.emplace_back(0, j);
      f.frames.push_back(rfield(in + s * s * j, s, s));
    }
    auto [noisy, snr] = add_poisson_noise(f, NoiseSpec{scale, seed});
    (void)snr;
    for (const auto& fr : noisy.frames) out = put(out, fr);
  });
}

int ref_toy(int64_t size, int64_t probe_side, int64_t step, uint64_t seed, double* sample,
            double* probe, double* pin) {
  // make_toy of proj/tests/test_solver.cpp:22-32 through the public API.
  return guard([&] {
    ScanGeometry g = make_raster_scan(size, size, probe_side, step);
    const int64_t border = probe_side / 2;
    auto [mag, ph] = make_test_images(size, size, border, seed);
    put(sample, make_sample(mag, ph, &g));
    put(probe, make_zone_plate_probe(probe_side));
    put(pin, vacuum_border_mask(size, size, border));
  });
}

double ref_r_factor_subs(const RefPlanSpec* ps, const double* subs, const double* intensities,
                         const double* probe) {
  double out = NAN;
  guard([&] {
    DecompositionPlan plan = make_plan(ps);
    std::vector<ComplexField2D> u;
    for (int d = 0; d < plan.D; ++d) {
      const Region& r = plan.subdomains[d];
      u.push_back(cfield(subs, r.height(), r.width()));
      subs += 2 * r.area();
    }
    out = r_factor(u, partition_frames(stack_from(plan, intensities), plan), cfield(probe, ps->s, ps->s));
  });
  return out;
}

#ifdef REF_HAVE_IO
// ---- the reference's own I/O (io.cpp): PTYA files and dataset directories ----
// A dataset directory as cmd_simulate writes it (ptychodd_cli.cpp:155-169):
// frames.ptya, probe.ptya, optional pin.ptya / sample.ptya, meta.json with
// schema_version 1, kind "dataset", the geometry record and a noise record
// (null: noiseless).  Raster geometry from make_raster_scan(H, W, s, step).
int ref_write_dataset(const char* dir, int64_t H, int64_t W, int64_t s, int64_t step, const double* frames,
                      const double* probe, const double* pin, const double* sample, int noisy) {
  return guard([&] {
    const std::filesystem::path out(dir);
    std::filesystem::create_directories(out);
    const ScanGeometry g = make_raster_scan(H, W, s, step);
    std::vector<RealField2D> fr;
    for (int64_t j = 0; j < g.frame_count(); ++j) fr.push_back(rfield(frames + s * s * j, s, s));
    write_frames(out / "frames.ptya", fr);
    write_array(out / "probe.ptya", cfield(probe, s, s));
    if (pin) write_array(out / "pin.ptya", rfield(pin, H, W));
    if (sample) write_array(out / "sample.ptya", cfield(sample, H, W));
    nlohmann::json noise = nullptr;
    if (noisy) noise = {{"target_snr_db", 30.0}};
    nlohmann::json meta = {{"schema_version", 1}, {"kind", "dataset"}, {"geometry", geometry_to_json(g)},
                           {"seed", 1}, {"border", 0}, {"noise", noise}};
    write_json(out / "meta.json", meta);
  });
}

int ref_write_frames(const char* path, const double* frames, int64_t J, int64_t h, int64_t w) {
  return guard([&] {
    std::vector<RealField2D> fr;
    for (int64_t j = 0; j < J; ++j) fr.push_back(rfield(frames + h * w * j, h, w));
    write_frames(path, fr);
  });
}

int ref_write_complex(const char* path, const double* data, int64_t h, int64_t w) {
  return guard([&] { write_array(path, cfield(data, h, w)); });
}

int ref_write_real(const char* path, const double* data, int64_t h, int64_t w) {
  return guard([&] { write_array(path, rfield(data, h, w)); });
}

// read_complex_array / read_real_array / read_frames: dims first (out may be
// NULL), then the payload.  FormatError -> 6.
int ref_read_array(const char* path, int kind, int64_t* dims3, double* out) {
  try {
    if (kind == 2) {
      const ComplexField2D f = read_complex_array(path);
      dims3[0] = f.height();
      dims3[1] = f.width();
      dims3[2] = 1;
      if (out) put(out, f);
    } else if (kind == 1) {
      const RealField2D f = read_real_array(path);
      dims3[0] = f.height();
      dims3[1] = f.width();
      dims3[2] = 1;
      if (out) put(out, f);
    } else {
      const auto fr = read_frames(path);
      dims3[0] = static_cast<int64_t>(fr.size());
      dims3[1] = fr.empty() ? 0 : fr[0].height();
      dims3[2] = fr.empty() ? 0 : fr[0].width();
      if (out)
        for (const auto& f : fr) out = put(out, f);
    }
    return 0;
  } catch (const FormatError& e) {
    return fail(e, 6);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

#endif  // REF_HAVE_IO

}  // extern "C"
