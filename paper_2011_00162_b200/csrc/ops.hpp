// Stand-alone GPU operators behind the C-ABI (see ops.cu).
#pragma once

#include <cstdint>

#include "plan.hpp"

namespace pdd {

template <typename T>
void op_fft2(double* data, int64_t h, int64_t w, bool inverse);
template <typename T>
void op_forward(const double* probe, int64_t s, const double* image, int64_t H, int64_t W, const int64_t* pos,
                int64_t J, double* frames_out, double* intensity_out);
template <typename T>
void op_simulate_device(const double* probe, int64_t s, const double* image, int64_t H, int64_t W,
                        const int64_t* pos, int64_t J, double* intensity_dev);
template <typename T>
void op_adjoint(const double* probe, int64_t s, const double* frames, const int64_t* pos, int64_t J, int64_t H,
                int64_t W, double* out);
template <typename T>
void op_illumination_density(const double* probe, int64_t s, const int64_t* pos, int64_t J, int64_t H, int64_t W,
                             double* out);
// num = sum_j conj(image|w_j) o IFFT(frame_j) (adjoint_probe), den = sum_j |image|w_j|^2 (probe_density)
template <typename T>
void op_probe_sums(const double* image, int64_t H, int64_t W, const double* frames, const int64_t* pos, int64_t J,
                   int64_t s, double* num_out, double* den_out);
template <typename T>
void op_prox(const double* y, const double* b, int64_t n, double lambda, double eps, double* out);
template <typename T>
void op_value_gradient(const double* x, const double* b, int64_t n, double eps, double* val, double* grad);
template <typename T>
void op_intensity(const double* z, int64_t n, double* out);
template <typename T>
void op_diff_norm(const double* cur, const double* prev, int64_t n, double* diff, double* norm);
template <typename T>
double op_r_factor(const Plan& plan, const double* subs, const double* intensities, const double* probe);

}  // namespace pdd
