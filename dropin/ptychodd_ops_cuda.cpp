// Drop-in definitions of the reference's operator layer over the B200 C-ABI:
// fft.hpp (fft2_normalized[_inplace], ifft2_normalized[_inplace]),
// forward.hpp (forward, adjoint, illumination_density, probe_density,
// adjoint_probe, intensity) and stagm.hpp (check_epsilon, pixel_value,
// pixel_gradient, pixel_prox, value, gradient, prox, lipschitz_constant).
// Replaces proj/src/fft.cpp, forward.cpp and stagm.cpp at link time; the
// argument validation is the reference's (same conditions, same exception
// types), the arithmetic runs in libptychodd_cuda.so.  Precision: float64
// unless PTYCHODD_CUDA_DTYPE=f32.
#include <cstdlib>
#include <string>

#include "ptychodd/fft.hpp"
#include "ptychodd/forward.hpp"
#include "ptychodd/stagm.hpp"
#include "ptychodd_cuda.hpp"

namespace ptychodd {
namespace {

int dtype() {
  const char* e = std::getenv("PTYCHODD_CUDA_DTYPE");
  return (e && std::string(e) == "f32") ? PDD_F32 : PDD_F64;
}
void check(int rc) { pdd_cuda::check(rc); }
double* dp(std::vector<cdouble>& v) { return reinterpret_cast<double*>(v.data()); }
const double* dp(const std::vector<cdouble>& v) { return reinterpret_cast<const double*>(v.data()); }

// forward.cpp:8-24
void check_probe(const ComplexField2D& probe, const ScanGeometry& g) {
  if (probe.height() != g.frame_side || probe.width() != g.frame_side)
    throw std::invalid_argument("forward model: probe shape != frame_side^2");
}
void check_image(const ComplexField2D& image, const ScanGeometry& g) {
  if (image.height() != g.image_height || image.width() != g.image_width)
    throw std::invalid_argument("forward model: image shape != geometry image_shape");
}
void check_frames(const std::vector<ComplexField2D>& frames, const ScanGeometry& g) {
  if (static_cast<int64_t>(frames.size()) != g.frame_count())
    throw std::invalid_argument("forward model: frame count mismatch");
  for (const auto& f : frames)
    if (f.height() != g.frame_side || f.width() != g.frame_side)
      throw std::invalid_argument("forward model: frame shape mismatch");
}

std::vector<int64_t> positions(const ScanGeometry& g) {
  std::vector<int64_t> p;
  p.reserve(2 * g.positions.size());
  for (const auto& [r, c] : g.positions) {
    p.push_back(r);
    p.push_back(c);
  }
  return p;
}

std::vector<cdouble> packed(const std::vector<ComplexField2D>& frames) {
  std::vector<cdouble> out;
  for (const auto& f : frames) out.insert(out.end(), f.data().begin(), f.data().end());
  return out;
}
std::vector<double> packed(const FrameStack& f) {
  std::vector<double> out;
  for (const auto& x : f.frames) out.insert(out.end(), x.data().begin(), x.data().end());
  return out;
}
std::vector<ComplexField2D> unpacked(const std::vector<cdouble>& flat, const std::vector<ComplexField2D>& like) {
  std::vector<ComplexField2D> out;
  size_t o = 0;
  for (const auto& f : like) {
    out.emplace_back(f.height(), f.width(), std::vector<cdouble>(flat.begin() + o, flat.begin() + o + f.size()));
    o += static_cast<size_t>(f.size());
  }
  return out;
}

void same_shapes(const std::vector<ComplexField2D>& z, const FrameStack& f, const char* who) {
  if (z.size() != f.frames.size()) throw std::invalid_argument(std::string(who) + ": frame count mismatch");
  for (size_t j = 0; j < z.size(); ++j)
    if (!(z[j].height() == f.frames[j].height() && z[j].width() == f.frames[j].width()))
      throw std::invalid_argument(std::string(who) + ": frame shape mismatch");
}

}  // namespace

// ------------------------------------------------------------------ fft.hpp
void fft2_normalized_inplace(ComplexField2D& x) {
  if (x.size() == 0) return;
  check(pdd_fft2(dp(x.data()), x.height(), x.width(), 0, dtype()));
}
void ifft2_normalized_inplace(ComplexField2D& x) {
  if (x.size() == 0) return;
  check(pdd_fft2(dp(x.data()), x.height(), x.width(), 1, dtype()));
}
ComplexField2D fft2_normalized(const ComplexField2D& x) {
  ComplexField2D y = x;
  fft2_normalized_inplace(y);
  return y;
}
ComplexField2D ifft2_normalized(const ComplexField2D& x) {
  ComplexField2D y = x;
  ifft2_normalized_inplace(y);
  return y;
}

// -------------------------------------------------------------- forward.hpp
std::vector<ComplexField2D> forward(const ComplexField2D& probe, const ComplexField2D& image,
                                    const ScanGeometry& geometry) {
  check_probe(probe, geometry);
  check_image(image, geometry);
  const int64_t s = geometry.frame_side, J = geometry.frame_count();
  const auto pos = positions(geometry);
  std::vector<cdouble> out(static_cast<size_t>(J * s * s));
  if (J)
    check(pdd_forward(dp(probe.data()), s, dp(image.data()), geometry.image_height, geometry.image_width, pos.data(),
                      J, dp(out), nullptr, dtype()));
  std::vector<ComplexField2D> frames;
  frames.reserve(static_cast<size_t>(J));
  for (int64_t j = 0; j < J; ++j)
    frames.emplace_back(s, s, std::vector<cdouble>(out.begin() + j * s * s, out.begin() + (j + 1) * s * s));
  return frames;
}

ComplexField2D adjoint(const ComplexField2D& probe, const std::vector<ComplexField2D>& frames,
                       const ScanGeometry& geometry) {
  check_probe(probe, geometry);
  check_frames(frames, geometry);
  ComplexField2D out(geometry.image_height, geometry.image_width);
  const auto pos = positions(geometry);
  const auto f = packed(frames);
  if (!frames.empty())
    check(pdd_adjoint(dp(probe.data()), geometry.frame_side, dp(f), pos.data(), geometry.frame_count(),
                      geometry.image_height, geometry.image_width, dp(out.data()), dtype()));
  return out;
}

RealField2D illumination_density(const ComplexField2D& probe, const ScanGeometry& geometry) {
  check_probe(probe, geometry);
  RealField2D out(geometry.image_height, geometry.image_width, 0.0);
  const auto pos = positions(geometry);
  if (geometry.frame_count())
    check(pdd_illumination_density(dp(probe.data()), geometry.frame_side, pos.data(), geometry.frame_count(),
                                   geometry.image_height, geometry.image_width, out.data().data(), dtype()));
  return out;
}

RealField2D probe_density(const ComplexField2D& image, const ScanGeometry& geometry) {
  check_image(image, geometry);
  RealField2D out(geometry.frame_side, geometry.frame_side, 0.0);
  const auto pos = positions(geometry);
  if (geometry.frame_count())
    check(pdd_probe_sums(dp(image.data()), geometry.image_height, geometry.image_width, nullptr, pos.data(),
                         geometry.frame_count(), geometry.frame_side, nullptr, out.data().data(), dtype()));
  return out;
}

ComplexField2D adjoint_probe(const ComplexField2D& image, const std::vector<ComplexField2D>& frames,
                             const ScanGeometry& geometry) {
  check_image(image, geometry);
  check_frames(frames, geometry);
  ComplexField2D out(geometry.frame_side, geometry.frame_side);
  const auto pos = positions(geometry);
  const auto f = packed(frames);
  if (!frames.empty())
    check(pdd_probe_sums(dp(image.data()), geometry.image_height, geometry.image_width, dp(f), pos.data(),
                         geometry.frame_count(), geometry.frame_side, dp(out.data()), nullptr, dtype()));
  return out;
}

FrameStack intensity(const std::vector<ComplexField2D>& frames, const ScanGeometry& geometry) {
  check_frames(frames, geometry);
  FrameStack out;
  out.geometry = geometry;
  const auto f = packed(frames);
  std::vector<double> m(f.size());
  if (!f.empty()) check(pdd_intensity(dp(f), static_cast<int64_t>(f.size()), m.data(), dtype()));
  size_t o = 0;
  for (const auto& x : frames) {
    out.frames.emplace_back(x.height(), x.width(), std::vector<double>(m.begin() + o, m.begin() + o + x.size()));
    o += static_cast<size_t>(x.size());
  }
  return out;
}

// ---------------------------------------------------------------- stagm.hpp
namespace stagm {

void check_epsilon(double epsilon) {  // stagm.cpp:24-27
  if (!(epsilon > 0.0 && epsilon < 1.0)) throw std::invalid_argument("stagm: epsilon must lie in (0,1)");
}

double pixel_value(cdouble x, double b, double epsilon) {
  double v = 0.0;
  check(pdd_stagm_value_gradient(reinterpret_cast<const double*>(&x), &b, 1, epsilon, &v, nullptr, dtype()));
  return v;
}

cdouble pixel_gradient(cdouble x, double b, double epsilon) {
  cdouble g;
  check(pdd_stagm_value_gradient(reinterpret_cast<const double*>(&x), &b, 1, epsilon, nullptr,
                                 reinterpret_cast<double*>(&g), dtype()));
  return g;
}

cdouble pixel_prox(cdouble y, double b, double lambda, double epsilon) {
  cdouble z;
  check(pdd_stagm_prox(reinterpret_cast<const double*>(&y), &b, 1, lambda, epsilon, reinterpret_cast<double*>(&z),
                       dtype()));
  return z;
}

double value(const std::vector<ComplexField2D>& z, const FrameStack& f, double epsilon) {  // stagm.cpp:75-85
  check_epsilon(epsilon);
  same_shapes(z, f, "stagm::value");
  const auto x = packed(z);
  const auto b = packed(f);
  std::vector<double> v(b.size());
  if (!b.empty())
    check(pdd_stagm_value_gradient(dp(x), b.data(), static_cast<int64_t>(b.size()), epsilon, v.data(), nullptr,
                                   dtype()));
  double s = 0.0;
  for (double e : v) s += e;
  return s;
}

std::vector<ComplexField2D> gradient(const std::vector<ComplexField2D>& z, const FrameStack& f, double epsilon) {
  check_epsilon(epsilon);
  if (z.size() != f.frames.size()) throw std::invalid_argument("stagm::gradient: frame count mismatch");
  const auto x = packed(z);
  const auto b = packed(f);
  std::vector<cdouble> g(x.size());
  if (!b.empty())
    check(pdd_stagm_value_gradient(dp(x), b.data(), static_cast<int64_t>(b.size()), epsilon, nullptr, dp(g),
                                   dtype()));
  return unpacked(g, z);
}

std::vector<ComplexField2D> prox(const std::vector<ComplexField2D>& y, const FrameStack& f, double lambda,
                                 double epsilon) {  // stagm.cpp:102-117
  check_epsilon(epsilon);
  if (lambda <= 0.0) throw std::invalid_argument("stagm::prox: lambda must be positive");
  if (y.size() != f.frames.size()) throw std::invalid_argument("stagm::prox: frame count mismatch");
  const auto x = packed(y);
  const auto b = packed(f);
  std::vector<cdouble> out(x.size());
  if (!b.empty())
    check(pdd_stagm_prox(dp(x), b.data(), static_cast<int64_t>(b.size()), lambda, epsilon, dp(out), dtype()));
  return unpacked(out, y);
}

double lipschitz_constant(double epsilon) {  // stagm.cpp:119-122
  check_epsilon(epsilon);
  return 2.0 / epsilon - 1.0;
}

}  // namespace stagm
}  // namespace ptychodd
