// extern "C" boundary (include/ptychodd_cuda.h): status codes instead of
// exceptions, thread-local error text, dtype dispatch.
#include "ptychodd_cuda.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "device.hpp"
#include "engine.hpp"
#include "layout.hpp"
#include "ops.hpp"
#include "plan.hpp"
#include "ptya.hpp"

struct pdd_plan {
  pdd::Plan plan;
};
struct pdd_nonblind {
  int device = 0;
  std::unique_ptr<pdd::Comm> comm;
  std::unique_ptr<pdd::NonblindGpu> s;
};
struct pdd_blind {
  int device = 0;
  std::unique_ptr<pdd::Comm> comm;
  std::unique_ptr<pdd::BlindGpu> s;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return PDD_OK;
  } catch (const pdd::Divergence& e) {
    g_err = e.what();
    return PDD_DIVERGENCE;
  } catch (const pdd::CudaError& e) {
    g_err = e.what();
    return PDD_CUDA_ERROR;
  } catch (const pdd::FormatError& e) {
    g_err = e.what();
    return PDD_FORMAT_ERROR;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return PDD_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return PDD_OUT_OF_RANGE;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("allocation failed: ") + e.what();
    return PDD_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PDD_RUNTIME_ERROR;
  } catch (...) {
    g_err = "unknown error";
    return PDD_RUNTIME_ERROR;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw pdd::InvalidArgument(std::string(what) + " must not be NULL");
}

bool is_f64(int32_t dtype) {
  if (dtype != PDD_F32 && dtype != PDD_F64) throw pdd::InvalidArgument("dtype must be PDD_F32 or PDD_F64");
  return dtype == PDD_F64;
}

class DeviceScope {
 public:
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev_);
    if (prev_ != dev) cudaSetDevice(dev);
  }
  ~DeviceScope() { cudaSetDevice(prev_); }

 private:
  int prev_ = 0;
};

pdd::NonblindConfig nb_cfg(const pdd_nonblind_config* c) {
  need(c, "config");
  pdd::NonblindConfig k;
  k.epsilon = c->epsilon;
  k.eta = c->eta;
  k.r = c->r;
  k.tol_rf = c->tol_rf;
  k.tol_re = c->tol_re;
  k.max_iters = c->max_iters;
  k.stop_rule = c->stop_rule;
  k.record_lagrangian = c->record_lagrangian;
  k.threads = c->threads;
  return k;
}

pdd::BlindConfig bl_cfg(const pdd_blind_config* c) {
  need(c, "config");
  pdd::BlindConfig k;
  k.epsilon = c->epsilon;
  k.eta = c->eta;
  k.r = c->r;
  k.mu = c->mu;
  k.gamma = c->gamma;
  k.support_energy = c->support_energy;
  k.tol_rf = c->tol_rf;
  k.tol_re = c->tol_re;
  k.max_iters = c->max_iters;
  k.stop_rule = c->stop_rule;
  k.threads = c->threads;
  return k;
}

void layout_out(const pdd::StateLayout& L, pdd_nonblind_layout* out) {
  out->n_local_sub = static_cast<int32_t>(L.local_subs.size());
  out->n_local_pairs = static_cast<int32_t>(L.local_pairs.size());
  out->frame_side = L.S;
  out->image_elems = 0;
  out->frame_elems = 0;
  out->v_elems = 0;
  for (size_t i = 0; i < L.local_subs.size(); ++i) {
    out->image_elems += L.sub_h[i] * L.sub_w[i];
    out->frame_elems += L.sub_frames[i] * L.S * L.S;
  }
  for (size_t i = 0; i < L.local_pairs.size(); ++i) out->v_elems += L.pair_h[i] * L.pair_w[i];
  out->lambda_elems = 2 * out->v_elems;
}

pdd::RecordFn record_fn(pdd_record_cb cb, void* user) {
  if (!cb) return {};
  return [cb, user](int64_t it, double rf, double re, double t, double lag) { cb(it, rf, re, t, lag, user); };
}

void records_out(const pdd::RunRecords& r, int64_t* iterations, double* records, int64_t* diverged_at) {
  if (iterations) *iterations = r.iterations;
  if (diverged_at) *diverged_at = r.diverged_at;
  if (records)
    for (int64_t n = 0; n < r.iterations; ++n) {
      records[3 * n] = r.rf[n];
      records[3 * n + 1] = r.re[n];
      records[3 * n + 2] = r.t_ms[n];
    }
  if (r.diverged_at) throw pdd::Divergence(r.diverged_at);
}

}  // namespace

extern "C" {

const char* pdd_last_error(void) { return g_err.c_str(); }
int pdd_version(void) { return 1; }

int pdd_device_count(int32_t* n) {
  return guard([&] {
    need(n, "n");
    int c = 0;
    const cudaError_t e = cudaGetDeviceCount(&c);
    *n = e == cudaSuccess ? c : 0;
  });
}

// ---- plans -----------------------------------------------------------------
int pdd_plan_stripes(int64_t H, int64_t W, int64_t s, int64_t step, int32_t D, int32_t axis, pdd_plan** out) {
  return guard([&] {
    need(out, "out");
    auto p = std::make_unique<pdd_plan>();
    p->plan = pdd::plan_stripes(pdd::make_raster_scan(H, W, s, step), D, axis);
    *out = p.release();
  });
}

int pdd_plan_grid(int64_t H, int64_t W, int64_t s, int64_t step, int32_t Dr, int32_t Dc, pdd_plan** out) {
  return guard([&] {
    need(out, "out");
    auto p = std::make_unique<pdd_plan>();
    p->plan = pdd::plan_grid(pdd::make_raster_scan(H, W, s, step), Dr, Dc);
    *out = p.release();
  });
}

int pdd_plan_from_arrays(int64_t s, int64_t step, int64_t H, int64_t W, int64_t J, const int64_t* positions, int32_t D,
                         const int32_t* assignment, const int64_t* subdomains, int32_t n_pairs, const int32_t* pairs,
                         const int64_t* regions, pdd_plan** out) {
  return guard([&] {
    need(out, "out");
    need(positions, "positions");
    need(assignment, "assignment");
    need(subdomains, "subdomains");
    if (n_pairs > 0) {
      need(pairs, "pairs");
      need(regions, "regions");
    }
    pdd::Geometry g;
    g.s = s;
    g.step = step;
    g.H = H;
    g.W = W;
    g.grid_rows = 1;
    g.grid_cols = J;
    g.pos.assign(positions, positions + 2 * J);
    for (int64_t j = 0; j < J; ++j)
      if (positions[2 * j] < 0 || positions[2 * j + 1] < 0 || positions[2 * j] + s > H || positions[2 * j + 1] + s > W)
        throw pdd::InvalidArgument("ScanGeometry: window outside image bounds");
    auto p = std::make_unique<pdd_plan>();
    p->plan = pdd::plan_from_arrays(g, D, assignment, subdomains, n_pairs, pairs, regions);
    *out = p.release();
  });
}

int pdd_plan_info_get(const pdd_plan* plan, pdd_plan_info* info) {
  return guard([&] {
    need(plan, "plan");
    need(info, "info");
    const auto& p = plan->plan;
    info->frame_side = p.g.s;
    info->step = p.g.step;
    info->image_height = p.g.H;
    info->image_width = p.g.W;
    info->grid_rows = p.g.grid_rows;
    info->grid_cols = p.g.grid_cols;
    info->n_frames = p.g.J();
    info->n_sub = p.D;
    info->n_pairs = static_cast<int32_t>(p.overlaps.size());
  });
}

int pdd_plan_arrays(const pdd_plan* plan, int64_t* positions, int32_t* assignment, int64_t* subdomains, int32_t* pairs,
                    int64_t* regions, int64_t* local_grid) {
  return guard([&] {
    need(plan, "plan");
    const auto& p = plan->plan;
    if (positions) std::memcpy(positions, p.g.pos.data(), sizeof(int64_t) * p.g.pos.size());
    if (assignment) std::memcpy(assignment, p.assign.data(), sizeof(int32_t) * p.assign.size());
    for (int d = 0; d < p.D; ++d) {
      if (subdomains) {
        const auto& r = p.subs[d];
        subdomains[4 * d] = r.r0;
        subdomains[4 * d + 1] = r.r1;
        subdomains[4 * d + 2] = r.c0;
        subdomains[4 * d + 3] = r.c1;
      }
      if (local_grid) {
        local_grid[2 * d] = p.local[d].grid_rows;
        local_grid[2 * d + 1] = p.local[d].grid_cols;
      }
    }
    for (size_t q = 0; q < p.overlaps.size(); ++q) {
      if (pairs) {
        pairs[2 * q] = p.overlaps[q].d1;
        pairs[2 * q + 1] = p.overlaps[q].d2;
      }
      if (regions) {
        const auto& r = p.overlaps[q].region;
        regions[4 * q] = r.r0;
        regions[4 * q + 1] = r.r1;
        regions[4 * q + 2] = r.c0;
        regions[4 * q + 3] = r.c1;
      }
    }
  });
}

int pdd_plan_destroy(pdd_plan* plan) {
  delete plan;
  return PDD_OK;
}

int pdd_rank_layout(const pdd_plan* plan, int32_t rank, int32_t world, int32_t* n_local_sub, int32_t* local_subs,
                    int32_t* n_local_pairs, int32_t* local_pairs, int32_t* n_exchange, int32_t* exchange) {
  return guard([&] {
    need(plan, "plan");
    if (world < 1 || rank < 0 || rank >= world) throw pdd::InvalidArgument("rank_layout: bad rank/world");
    const pdd::Layout L = pdd::Layout::build(plan->plan, rank, world);
    if (n_local_sub) *n_local_sub = L.nls();
    if (local_subs) std::copy(L.local_subs.begin(), L.local_subs.end(), local_subs);
    if (n_local_pairs) *n_local_pairs = static_cast<int32_t>(L.lpairs.size());
    if (local_pairs) std::copy(L.lpairs.begin(), L.lpairs.end(), local_pairs);
    if (n_exchange) *n_exchange = static_cast<int32_t>(L.exch.size());
    if (exchange)
      for (size_t i = 0; i < L.exch.size(); ++i) {
        exchange[3 * i] = L.exch[i].lp;
        exchange[3 * i + 1] = L.exch[i].peer;
        exchange[3 * i + 2] = L.exch[i].my_side;
      }
  });
}

int pdd_scan_coverage(const pdd_plan* plan, int32_t* out) {
  return guard([&] {
    need(plan, "plan");
    need(out, "out");
    const auto cov = pdd::scan_coverage(plan->plan.g);
    std::memcpy(out, cov.data(), sizeof(int32_t) * cov.size());
  });
}

// ---- operators -------------------------------------------------------------
int pdd_fft2(double* data, int64_t h, int64_t w, int32_t inverse, int32_t dtype) {
  return guard([&] {
    need(data, "data");
    if (is_f64(dtype)) pdd::op_fft2<double>(data, h, w, inverse != 0);
    else pdd::op_fft2<float>(data, h, w, inverse != 0);
  });
}

int pdd_forward(const double* probe, int64_t s, const double* image, int64_t H, int64_t W, const int64_t* positions,
                int64_t J, double* frames_out, double* intensity_out, int32_t dtype) {
  return guard([&] {
    need(probe, "probe");
    need(image, "image");
    need(positions, "positions");
    if (is_f64(dtype)) pdd::op_forward<double>(probe, s, image, H, W, positions, J, frames_out, intensity_out);
    else pdd::op_forward<float>(probe, s, image, H, W, positions, J, frames_out, intensity_out);
  });
}

int pdd_adjoint(const double* probe, int64_t s, const double* frames, const int64_t* positions, int64_t J, int64_t H,
                int64_t W, double* image_out, int32_t dtype) {
  return guard([&] {
    need(probe, "probe");
    need(frames, "frames");
    need(positions, "positions");
    need(image_out, "image_out");
    if (is_f64(dtype)) pdd::op_adjoint<double>(probe, s, frames, positions, J, H, W, image_out);
    else pdd::op_adjoint<float>(probe, s, frames, positions, J, H, W, image_out);
  });
}

int pdd_illumination_density(const double* probe, int64_t s, const int64_t* positions, int64_t J, int64_t H, int64_t W,
                             double* out, int32_t dtype) {
  return guard([&] {
    need(probe, "probe");
    need(positions, "positions");
    need(out, "out");
    if (is_f64(dtype)) pdd::op_illumination_density<double>(probe, s, positions, J, H, W, out);
    else pdd::op_illumination_density<float>(probe, s, positions, J, H, W, out);
  });
}

int pdd_probe_sums(const double* image, int64_t H, int64_t W, const double* frames, const int64_t* positions, int64_t J,
                   int64_t s, double* num_out, double* den_out, int32_t dtype) {
  return guard([&] {
    need(image, "image");
    need(positions, "positions");
    if (is_f64(dtype)) pdd::op_probe_sums<double>(image, H, W, frames, positions, J, s, num_out, den_out);
    else pdd::op_probe_sums<float>(image, H, W, frames, positions, J, s, num_out, den_out);
  });
}

int pdd_simulate_intensity_device(const double* probe, int64_t s, const double* image, int64_t H, int64_t W,
                                  const int64_t* positions, int64_t J, double* intensity_dev, int32_t dtype) {
  return guard([&] {
    need(probe, "probe");
    need(image, "image");
    need(positions, "positions");
    need(intensity_dev, "intensity_dev");
    if (is_f64(dtype)) pdd::op_simulate_device<double>(probe, s, image, H, W, positions, J, intensity_dev);
    else pdd::op_simulate_device<float>(probe, s, image, H, W, positions, J, intensity_dev);
  });
}

int pdd_intensity(const double* z, int64_t n, double* out, int32_t dtype) {
  return guard([&] {
    need(z, "z");
    need(out, "out");
    if (is_f64(dtype)) pdd::op_intensity<double>(z, n, out);
    else pdd::op_intensity<float>(z, n, out);
  });
}

int pdd_stagm_prox(const double* y, const double* b, int64_t n, double lambda, double epsilon, double* out,
                   int32_t dtype) {
  return guard([&] {
    need(y, "y");
    need(b, "b");
    need(out, "out");
    if (is_f64(dtype)) pdd::op_prox<double>(y, b, n, lambda, epsilon, out);
    else pdd::op_prox<float>(y, b, n, lambda, epsilon, out);
  });
}

int pdd_stagm_value_gradient(const double* x, const double* b, int64_t n, double epsilon, double* value,
                             double* gradient, int32_t dtype) {
  return guard([&] {
    need(x, "x");
    need(b, "b");
    if (is_f64(dtype)) pdd::op_value_gradient<double>(x, b, n, epsilon, value, gradient);
    else pdd::op_value_gradient<float>(x, b, n, epsilon, value, gradient);
  });
}

int pdd_r_factor(const pdd_plan* plan, const double* subs, const double* intensities, const double* probe, double* out,
                 int32_t dtype) {
  return guard([&] {
    need(plan, "plan");
    need(subs, "subs");
    need(intensities, "intensities");
    need(probe, "probe");
    need(out, "out");
    *out = is_f64(dtype) ? pdd::op_r_factor<double>(plan->plan, subs, intensities, probe)
                         : pdd::op_r_factor<float>(plan->plan, subs, intensities, probe);
  });
}

int pdd_relative_error(const double* current, const double* previous, int32_t D, const int64_t* sizes, double* out,
                       int32_t dtype) {
  return guard([&] {
    need(current, "current");
    need(previous, "previous");
    need(sizes, "sizes");
    need(out, "out");
    double worst = 0.0;
    int64_t off = 0;
    for (int d = 0; d < D; ++d) {  // metrics.cpp:29-46
      double diff = 0.0, norm = 0.0;
      if (is_f64(dtype)) pdd::op_diff_norm<double>(current + 2 * off, previous + 2 * off, sizes[d], &diff, &norm);
      else pdd::op_diff_norm<float>(current + 2 * off, previous + 2 * off, sizes[d], &diff, &norm);
      if (norm <= 0.0) throw pdd::InvalidArgument("relative_error: zero current norm");
      worst = std::max(worst, std::sqrt(diff / norm));
      off += sizes[d];
    }
    *out = worst;
  });
}

int pdd_merge(const pdd_plan* plan, const double* subs, double* out) {
  return guard([&] {  // ddplan.cpp:104-121 (exact host arithmetic, as the reference)
    need(plan, "plan");
    need(subs, "subs");
    need(out, "out");
    const auto& p = plan->plan;
    const int64_t H = p.g.H, W = p.g.W;
    std::vector<double> cnt(static_cast<size_t>(H * W), 0.0);
    std::fill(out, out + 2 * H * W, 0.0);
    int64_t off = 0;
    for (int d = 0; d < p.D; ++d) {
      const auto& r = p.subs[d];
      for (int64_t rr = 0; rr < r.h(); ++rr)
        for (int64_t cc = 0; cc < r.w(); ++cc) {
          const int64_t gi = (r.r0 + rr) * W + r.c0 + cc;
          const int64_t li = off + rr * r.w() + cc;
          out[2 * gi] += subs[2 * li];
          out[2 * gi + 1] += subs[2 * li + 1];
          cnt[gi] += 1.0;
        }
      off += r.area();
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
  });
}

// ---- nonblind --------------------------------------------------------------
int pdd_nccl_unique_id(void* out128) {
  return guard([&] {
    need(out128, "out");
    pdd::nccl_unique_id(out128);
  });
}

static int nonblind_create(const pdd_plan* plan, const void* data, int32_t kind, int32_t on_dev, const double* probe,
                           const pdd_nonblind_config* cfg, const double* pin, int32_t dtype, int32_t device,
                           int32_t rank, int32_t world, const void* nccl_id, pdd_nonblind** out) {
  return guard([&] {
    need(plan, "plan");
    need(data, "data");
    need(probe, "probe");
    need(out, "out");
    if (kind < 0 || kind > 3) throw pdd::InvalidArgument("data_kind out of range");
    if (kind == PDD_DATA_PTYA_FRAMES_F64 && on_dev) throw pdd::InvalidArgument("a PTYA path is host data");
    const bool f64 = is_f64(dtype);
    auto h = std::make_unique<pdd_nonblind>();
    h->device = device;
    DeviceScope ds(device);
    if (world > 1 || nccl_id) {  // world 1 with an id: single-rank NCCL communicator (plumbing test)
      need(nccl_id, "nccl_id");
      h->comm = pdd::is_host_hub_id(nccl_id) ? pdd::make_host_comm(nccl_id, rank, world)
                                             : pdd::make_nccl_comm(nccl_id, rank, world, device);
    }
    pdd::DataSpec spec{data, kind, on_dev != 0};
    h->s = pdd::make_nonblind(plan->plan, spec, probe, nb_cfg(cfg), pin, f64 ? 2 : 1, device, h->comm.get());
    *out = h.release();
  });
}

int pdd_nonblind_create(const pdd_plan* plan, const void* data, int32_t data_kind, int32_t data_on_device,
                        const double* probe, const pdd_nonblind_config* cfg, const double* pin_ones, int32_t dtype,
                        int32_t device, pdd_nonblind** out) {
  return nonblind_create(plan, data, data_kind, data_on_device, probe, cfg, pin_ones, dtype, device, 0, 1, nullptr,
                         out);
}

int pdd_nonblind_create_rank(const pdd_plan* plan, const void* data, int32_t data_kind, int32_t data_on_device,
                             const double* probe, const pdd_nonblind_config* cfg, const double* pin_ones,
                             int32_t dtype, int32_t device, int32_t rank, int32_t world, const void* nccl_id,
                             pdd_nonblind** out) {
  return nonblind_create(plan, data, data_kind, data_on_device, probe, cfg, pin_ones, dtype, device, rank, world,
                         nccl_id, out);
}

int pdd_nonblind_create_multi(const pdd_plan* plan, const void* data, int32_t kind, int32_t on_dev,
                              const double* probe, const pdd_nonblind_config* cfg, const double* pin, int32_t dtype,
                              const int32_t* devices, int32_t n_devices, pdd_nonblind** out) {
  return guard([&] {
    need(plan, "plan");
    need(data, "data");
    need(probe, "probe");
    need(devices, "devices");
    need(out, "out");
    if (kind < 0 || kind > 3) throw pdd::InvalidArgument("data_kind out of range");
    if (kind == PDD_DATA_PTYA_FRAMES_F64 && on_dev) throw pdd::InvalidArgument("a PTYA path is host data");
    if (n_devices < 1) throw pdd::InvalidArgument("n_devices >= 1");
    const bool f64 = is_f64(dtype);
    auto h = std::make_unique<pdd_nonblind>();
    h->device = devices[0];
    DeviceScope ds(devices[0]);
    pdd::DataSpec spec{data, kind, on_dev != 0};
    h->s = pdd::make_nonblind_multi(plan->plan, spec, probe, nb_cfg(cfg), pin, f64 ? 2 : 1,
                                    std::vector<int>(devices, devices + n_devices));
    *out = h.release();
  });
}

int pdd_ptya_header(const char* path, int32_t want_dtype, int32_t* ndim, int64_t* dims4, int64_t* payload_offset) {
  return guard([&] {
    need(path, "path");
    const pdd::PtyaHeader h = pdd::ptya_read_header(path, static_cast<uint16_t>(want_dtype));
    if (ndim) *ndim = static_cast<int32_t>(h.dims.size());
    if (dims4)
      for (size_t i = 0; i < 4; ++i) dims4[i] = i < h.dims.size() ? static_cast<int64_t>(h.dims[i]) : 0;
    if (payload_offset) *payload_offset = static_cast<int64_t>(h.payload_offset);
  });
}

int pdd_host_transport_id(void* out128) {
  return guard([&] {
    need(out128, "out");
    pdd::host_hub_id(out128);
  });
}

#define NB_CALL(h, body)                     \
  return guard([&] {                         \
    need(h, "handle");                       \
    DeviceScope ds_((h)->device);            \
    pdd::AllocStream as_(static_cast<cudaStream_t>((h)->s->stream())); \
    body;                                    \
  })

int pdd_nonblind_layout_get(const pdd_nonblind* h, pdd_nonblind_layout* out) {
  return guard([&] {
    need(h, "handle");
    need(out, "out");
    layout_out(h->s->layout(), out);
  });
}

int pdd_nonblind_layout_arrays(const pdd_nonblind* h, int32_t* local_subs, int64_t* sub_hw, int64_t* sub_frames,
                               int32_t* local_pairs, int64_t* pair_hw) {
  return guard([&] {
    need(h, "handle");
    const auto& L = h->s->layout();
    for (size_t i = 0; i < L.local_subs.size(); ++i) {
      if (local_subs) local_subs[i] = L.local_subs[i];
      if (sub_hw) {
        sub_hw[2 * i] = L.sub_h[i];
        sub_hw[2 * i + 1] = L.sub_w[i];
      }
      if (sub_frames) sub_frames[i] = L.sub_frames[i];
    }
    for (size_t i = 0; i < L.local_pairs.size(); ++i) {
      if (local_pairs) local_pairs[i] = L.local_pairs[i];
      if (pair_hw) {
        pair_hw[2 * i] = L.pair_h[i];
        pair_hw[2 * i + 1] = L.pair_w[i];
      }
    }
  });
}

int pdd_nonblind_init_state(pdd_nonblind* h) { NB_CALL(h, h->s->init_state()); }
int pdd_nonblind_step(pdd_nonblind* h, int32_t store_z) { NB_CALL(h, h->s->step(store_z != 0)); }
int pdd_nonblind_run(pdd_nonblind* h, int64_t* iterations, double* records, int64_t* diverged_at) {
  NB_CALL(h, records_out(h->s->run(), iterations, records, diverged_at));
}
int pdd_nonblind_run_cb(pdd_nonblind* h, pdd_record_cb cb, void* user, int64_t* iterations, double* records,
                        int64_t* diverged_at) {
  NB_CALL(h, records_out(h->s->run(record_fn(cb, user)), iterations, records, diverged_at));
}
int pdd_nonblind_iterate(pdd_nonblind* h, int32_t n) { NB_CALL(h, h->s->iterate(n)); }
int pdd_nonblind_iterate_timed(pdd_nonblind* h, int32_t n, double* ms) {
  NB_CALL(h, need(ms, "ms"); *ms = h->s->iterate_timed(n));
}
int pdd_nonblind_profile(pdd_nonblind* h, int32_t n, double* ms) {
  NB_CALL(h, need(ms, "ms"); if (n < 1) throw pdd::InvalidArgument("profile: n >= 1"); h->s->profile(n, ms));
}
int pdd_nonblind_last_rf(pdd_nonblind* h, double* rf) { NB_CALL(h, need(rf, "rf"); *rf = h->s->last_rf()); }
int pdd_nonblind_get_state(pdd_nonblind* h, double* u, double* z, double* gamma, double* v, double* lambda,
                           int64_t* iteration) {
  NB_CALL(h, h->s->get_state(u, z, gamma, v, lambda, iteration));
}
int pdd_nonblind_set_state(pdd_nonblind* h, const double* u, const double* z, const double* gamma, const double* v,
                           const double* lambda, int64_t iteration) {
  NB_CALL(h, h->s->set_state(u, z, gamma, v, lambda, iteration));
}
int pdd_nonblind_forward(pdd_nonblind* h, double* au) { NB_CALL(h, need(au, "au"); h->s->forward_frames(au)); }
int pdd_disk_support_mask(int64_t side, double radius, double* out) {
  return guard([&] {
    need(out, "out");
    if (side < 1) throw pdd::InvalidArgument("disk_support_mask: side >= 1");
    const auto m = pdd::disk_mask(side, radius);
    std::copy(m.begin(), m.end(), out);
  });
}
int pdd_estimate_support_mask(const double* probe_guess, int64_t side, double energy_fraction, double* out) {
  return guard([&] {
    need(probe_guess, "probe_guess");
    need(out, "out");
    if (side < 1) throw pdd::InvalidArgument("estimate_support_mask: side >= 1");
    const auto m = pdd::estimate_mask(std::vector<double>(probe_guess, probe_guess + 2 * side * side), side,
                                      energy_fraction);
    std::copy(m.begin(), m.end(), out);
  });
}
int pdd_nonblind_lagrangian(pdd_nonblind* h, double* out) {
  NB_CALL(h, need(out, "out"); *out = h->s->lagrangian());
}
int pdd_nonblind_lagrangian_history(pdd_nonblind* h, double* out, int64_t cap, int64_t* n) {
  NB_CALL(h, need(n, "n"); const auto v = h->s->lagrangian_history(); *n = static_cast<int64_t>(v.size());
          if (out) std::copy(v.begin(), v.begin() + std::min<int64_t>(cap, *n), out));
}
int pdd_nonblind_merged(pdd_nonblind* h, double* out) { NB_CALL(h, need(out, "out"); h->s->merged(out)); }
int pdd_nonblind_sync(pdd_nonblind* h) { NB_CALL(h, h->s->sync()); }
int pdd_nonblind_launches_per_iteration(const pdd_nonblind* h, int64_t* n) {
  return guard([&] {
    need(h, "handle");
    need(n, "n");
    *n = h->s->kernel_launches_per_iteration();
  });
}
int pdd_nonblind_destroy(pdd_nonblind* h) {
  if (!h) return PDD_OK;
  return guard([&] {
    DeviceScope ds(h->device);
    delete h;
  });
}

// ---- blind -----------------------------------------------------------------
static int blind_create(const pdd_plan* plan, const void* data, int32_t kind, int32_t on_dev,
                        const pdd_blind_config* cfg, const double* mask, const double* pin, int32_t dtype,
                        int32_t device, int32_t rank, int32_t world, const void* nccl_id, pdd_blind** out) {
  return guard([&] {
    need(plan, "plan");
    need(data, "data");
    need(out, "out");
    if (kind < 0 || kind > 3) throw pdd::InvalidArgument("data_kind out of range");
    if (kind == PDD_DATA_PTYA_FRAMES_F64 && on_dev) throw pdd::InvalidArgument("a PTYA path is host data");
    const bool f64 = is_f64(dtype);
    auto h = std::make_unique<pdd_blind>();
    h->device = device;
    DeviceScope ds(device);
    if (world > 1 || nccl_id) {
      need(nccl_id, "nccl_id");
      h->comm = pdd::is_host_hub_id(nccl_id) ? pdd::make_host_comm(nccl_id, rank, world)
                                             : pdd::make_nccl_comm(nccl_id, rank, world, device);
    }
    pdd::DataSpec spec{data, kind, on_dev != 0};
    h->s = pdd::make_blind(plan->plan, spec, bl_cfg(cfg), mask, pin, f64 ? 2 : 1, device, h->comm.get());
    *out = h.release();
  });
}

int pdd_blind_create_multi(const pdd_plan* plan, const void* data, int32_t kind, int32_t on_dev,
                           const pdd_blind_config* cfg, const double* mask, const double* pin, int32_t dtype,
                           const int32_t* devices, int32_t n_devices, pdd_blind** out) {
  return guard([&] {
    need(plan, "plan");
    need(data, "data");
    need(devices, "devices");
    need(out, "out");
    if (kind < 0 || kind > 3) throw pdd::InvalidArgument("data_kind out of range");
    if (kind == PDD_DATA_PTYA_FRAMES_F64 && on_dev) throw pdd::InvalidArgument("a PTYA path is host data");
    if (n_devices < 1) throw pdd::InvalidArgument("n_devices >= 1");
    const bool f64 = is_f64(dtype);
    auto h = std::make_unique<pdd_blind>();
    h->device = devices[0];
    DeviceScope ds(devices[0]);
    pdd::DataSpec spec{data, kind, on_dev != 0};
    h->s = pdd::make_blind_multi(plan->plan, spec, bl_cfg(cfg), mask, pin, f64 ? 2 : 1,
                                 std::vector<int>(devices, devices + n_devices));
    *out = h.release();
  });
}

int pdd_blind_create(const pdd_plan* plan, const void* data, int32_t data_kind, int32_t data_on_device,
                     const pdd_blind_config* cfg, const double* support_mask, const double* pin_ones, int32_t dtype,
                     int32_t device, pdd_blind** out) {
  return blind_create(plan, data, data_kind, data_on_device, cfg, support_mask, pin_ones, dtype, device, 0, 1, nullptr,
                      out);
}
int pdd_blind_create_rank(const pdd_plan* plan, const void* data, int32_t data_kind, int32_t data_on_device,
                          const pdd_blind_config* cfg, const double* support_mask, const double* pin_ones,
                          int32_t dtype, int32_t device, int32_t rank, int32_t world, const void* nccl_id,
                          pdd_blind** out) {
  return blind_create(plan, data, data_kind, data_on_device, cfg, support_mask, pin_ones, dtype, device, rank, world,
                      nccl_id, out);
}
int pdd_blind_layout_get(const pdd_blind* h, pdd_nonblind_layout* out) {
  return guard([&] {
    need(h, "handle");
    need(out, "out");
    layout_out(h->s->layout(), out);
  });
}
int pdd_blind_init_state(pdd_blind* h, const double* w0) { NB_CALL(h, h->s->init_state(w0)); }
int pdd_blind_step(pdd_blind* h, int32_t store_z) { NB_CALL(h, h->s->step(store_z != 0)); }
int pdd_blind_run(pdd_blind* h, int64_t* iterations, double* records, int64_t* diverged_at) {
  NB_CALL(h, records_out(h->s->run(), iterations, records, diverged_at));
}
int pdd_blind_run_cb(pdd_blind* h, pdd_record_cb cb, void* user, int64_t* iterations, double* records,
                     int64_t* diverged_at) {
  NB_CALL(h, records_out(h->s->run(record_fn(cb, user)), iterations, records, diverged_at));
}
int pdd_blind_iterate(pdd_blind* h, int32_t n) { NB_CALL(h, h->s->iterate(n)); }
int pdd_blind_iterate_timed(pdd_blind* h, int32_t n, double* ms) {
  NB_CALL(h, need(ms, "ms"); *ms = h->s->iterate_timed(n));
}
int pdd_blind_profile(pdd_blind* h, int32_t n, double* ms) {
  NB_CALL(h, need(ms, "ms"); if (n < 1) throw pdd::InvalidArgument("profile: n >= 1"); h->s->profile(n, ms));
}
int pdd_blind_get_state(pdd_blind* h, double* w, double* w_copies, double* delta, double* u, double* z, double* gamma,
                        double* v, double* lambda, int64_t* iteration) {
  NB_CALL(h, h->s->get_state(w, w_copies, delta, u, z, gamma, v, lambda, iteration));
}
int pdd_blind_set_state(pdd_blind* h, const double* w, const double* w_copies, const double* delta, const double* u,
                        const double* z, const double* gamma, const double* v, const double* lambda,
                        int64_t iteration) {
  NB_CALL(h, h->s->set_state(w, w_copies, delta, u, z, gamma, v, lambda, iteration));
}
int pdd_blind_get_probe(pdd_blind* h, double* probe, double* probe_fourier, double* mask, double* w0) {
  NB_CALL(h, h->s->get_probe(probe, probe_fourier, mask, w0));
}
int pdd_blind_merged(pdd_blind* h, double* out) { NB_CALL(h, need(out, "out"); h->s->merged(out)); }
int pdd_blind_sync(pdd_blind* h) { NB_CALL(h, h->s->sync()); }
int pdd_blind_launches_per_iteration(const pdd_blind* h, int64_t* n) {
  return guard([&] {
    need(h, "handle");
    need(n, "n");
    *n = h->s->kernel_launches_per_iteration();
  });
}
int pdd_blind_destroy(pdd_blind* h) {
  if (!h) return PDD_OK;
  return guard([&] {
    DeviceScope ds(h->device);
    delete h;
  });
}

// ---- pinned host memory ----------------------------------------------------
int pdd_host_alloc(void** p, int64_t bytes) {
  return guard([&] {
    need(p, "p");
    pdd::cuda_check(cudaMallocHost(p, static_cast<size_t>(bytes)), "cudaMallocHost");
  });
}
int pdd_release_cached_memory(void) {
  return guard([&] { pdd::release_cached_memory(); });
}
int pdd_host_stage_reserve(void) {
  return guard([&] { pdd::host_stage_reserve(); });
}
int pdd_host_free(void* p) {
  return guard([&] {
    if (p) pdd::cuda_check(cudaFreeHost(p), "cudaFreeHost");
  });
}

}  // extern "C"
