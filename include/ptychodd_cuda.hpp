// ptychodd_cuda.hpp -- header-only C++ adapter over the C-ABI (ptychodd_cuda.h).
//
// Gives C++ callers of the reference API (proj/include/ptychodd/*.hpp) RAII
// objects with the reference's semantics: status codes are rethrown as the
// reference's exception types (std::invalid_argument, std::out_of_range,
// std::runtime_error, a DivergenceError carrying the iteration).  Buffers are
// std::vector<std::complex<double>> / std::vector<double>, the storage of the
// reference's ComplexField2D / RealField2D (field.hpp:48-130), so an adapter
// for the reference types is a data() pointer away.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ptychodd_cuda.h"

namespace pdd_cuda {

using cdouble = std::complex<double>;

struct DivergenceError : std::runtime_error {
  int64_t iteration;
  DivergenceError(int64_t it, const std::string& m) : std::runtime_error(m), iteration(it) {}
};

inline void check(int rc, int64_t iteration = 0) {
  if (rc == PDD_OK) return;
  const std::string msg = pdd_last_error();
  switch (rc) {
    case PDD_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PDD_OUT_OF_RANGE: throw std::out_of_range(msg);
    case PDD_DIVERGENCE: throw DivergenceError(iteration, msg);
    default: throw std::runtime_error(msg);
  }
}

inline const double* d(const std::vector<cdouble>& v) { return reinterpret_cast<const double*>(v.data()); }
inline double* d(std::vector<cdouble>& v) { return reinterpret_cast<double*>(v.data()); }

// make_raster_scan + plan_stripes / plan_grid (ddplan.hpp:40-41).
class Plan {
 public:
  static Plan stripes(int64_t H, int64_t W, int64_t s, int64_t step, int D, int axis = PDD_AXIS_AUTO) {
    Plan p;
    check(pdd_plan_stripes(H, W, s, step, D, axis, &p.h_));
    return p;
  }
  static Plan grid(int64_t H, int64_t W, int64_t s, int64_t step, int Dr, int Dc) {
    Plan p;
    check(pdd_plan_grid(H, W, s, step, Dr, Dc, &p.h_));
    return p;
  }
  Plan(Plan&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  Plan(const Plan&) = delete;
  ~Plan() { pdd_plan_destroy(h_); }
  const pdd_plan* get() const { return h_; }
  pdd_plan_info info() const {
    pdd_plan_info i{};
    check(pdd_plan_info_get(h_, &i));
    return i;
  }

 private:
  Plan() = default;
  pdd_plan* h_ = nullptr;
};

// forward / adjoint (forward.hpp:8-14) over a flat [J][s][s] stack.
inline std::vector<cdouble> forward(const std::vector<cdouble>& probe, int64_t s, const std::vector<cdouble>& image,
                                    int64_t H, int64_t W, const std::vector<int64_t>& pos, int dtype = PDD_F64) {
  const int64_t J = static_cast<int64_t>(pos.size() / 2);
  std::vector<cdouble> out(static_cast<size_t>(J * s * s));
  check(pdd_forward(d(probe), s, d(image), H, W, pos.data(), J, d(out), nullptr, dtype));
  return out;
}

inline std::vector<cdouble> adjoint(const std::vector<cdouble>& probe, int64_t s, const std::vector<cdouble>& frames,
                                    const std::vector<int64_t>& pos, int64_t H, int64_t W, int dtype = PDD_F64) {
  std::vector<cdouble> out(static_cast<size_t>(H * W));
  check(pdd_adjoint(d(probe), s, d(frames), pos.data(), static_cast<int64_t>(pos.size() / 2), H, W, d(out), dtype));
  return out;
}

struct Record {
  int64_t iteration;
  double rf, re, t_ms;
};

// NonblindSolver (solver.hpp:72-107): construct from intensities [J][s][s].
class NonblindSolver {
 public:
  NonblindSolver(const Plan& plan, const std::vector<double>& intensities, const std::vector<cdouble>& probe,
                 const pdd_nonblind_config& cfg, const std::vector<double>* pin_ones = nullptr,
                 int dtype = PDD_F32, int device = 0)
      : cfg_(cfg) {
    check(pdd_nonblind_create(plan.get(), intensities.data(), PDD_DATA_INTENSITY_F64, 0, d(probe), &cfg,
                              pin_ones ? pin_ones->data() : nullptr, dtype, device, &h_));
  }
  NonblindSolver(const NonblindSolver&) = delete;
  ~NonblindSolver() { pdd_nonblind_destroy(h_); }

  // run(): records of every iteration; the sub-solutions stay on the device
  // until sub_solutions() is called.
  std::vector<Record> run() {
    int64_t n = 0, div = 0;
    std::vector<double> rec(3 * static_cast<size_t>(cfg_.max_iters));
    check(pdd_nonblind_run(h_, &n, rec.data(), &div), div);
    std::vector<Record> out;
    for (int64_t k = 0; k < n; ++k) out.push_back({k + 1, rec[3 * k], rec[3 * k + 1], rec[3 * k + 2]});
    return out;
  }
  void step() { check(pdd_nonblind_step(h_, 1)); }
  void iterate(int n) { check(pdd_nonblind_iterate(h_, n)); }
  std::vector<cdouble> sub_solutions() {
    pdd_nonblind_layout l{};
    check(pdd_nonblind_layout_get(h_, &l));
    std::vector<cdouble> u(static_cast<size_t>(l.image_elems));
    check(pdd_nonblind_get_state(h_, d(u), nullptr, nullptr, nullptr, nullptr, nullptr));
    return u;
  }
  pdd_nonblind* get() { return h_; }

 private:
  pdd_nonblind_config cfg_;
  pdd_nonblind* h_ = nullptr;
};

inline std::vector<cdouble> merge(const Plan& plan, const std::vector<cdouble>& subs) {
  const pdd_plan_info i = plan.info();
  std::vector<cdouble> out(static_cast<size_t>(i.image_height * i.image_width));
  check(pdd_merge(plan.get(), d(subs), d(out)));
  return out;
}

}  // namespace pdd_cuda
