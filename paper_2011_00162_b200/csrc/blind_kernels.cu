// Probe-side kernels of the blind OD²BP iteration (blind.cpp:194-296).
//
// The probe copies W_d are s x s tiles shared by all frames of a subdomain, so
// their updates are reductions over frames:
//   adjoint_probe  sum_j conj(u|w_j) o q_j   (forward.cpp:80-93)
//   probe_density  sum_j |u|w_j|^2           (forward.cpp:68-78)
// computed deterministically as fixed frame chunks (each summed in ascending
// j) followed by an ordered sum of the chunks, never with atomics.
#include "blind_kernels.hpp"
#include "cx.cuh"

namespace pdd {

// partial[c][pix] over frames [chunk_f0[c], chunk_f1[c]).
// mode 0: num = sum conj(u) q, den = sum |u|^2 ; mode 1: num = sum q (no image)
template <typename T>
__global__ void probe_partials_kernel(const cx<T>* img, const int64_t* off, const int32_t* pitch, const cx<T>* q,
                                      const int32_t* chunk_f0, const int32_t* chunk_f1, int S, int mode,
                                      cx<T>* num_part, T* den_part, const int* skip) {
  if (skip && *skip) return;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  const int SS = S * S;
  if (pix >= SS) return;
  const int y = pix / S, x = pix % S;
  const int c = blockIdx.y;
  const int f0 = chunk_f0[c], f1 = chunk_f1[c];
  cx<T> num{T(0), T(0)};
  T den = T(0);
#pragma unroll 8  // eight frames' loads in flight; the adds keep their order
  for (int f = f0; f < f1; ++f) {
    const cx<T> qq = q[static_cast<int64_t>(f) * SS + pix];
    if (mode == 1) {
      num += qq;
    } else {
      const cx<T> u = img[off[f] + static_cast<int64_t>(y) * pitch[f] + x];
      num += mul_conj(qq, u);
      den += norm2(u);
    }
  }
  num_part[static_cast<int64_t>(c) * SS + pix] = num;
  if (den_part) den_part[static_cast<int64_t>(c) * SS + pix] = den;
}

template <typename T>
__global__ void chunk_reduce_kernel(const cx<T>* num_part, const T* den_part, const int32_t* seg_beg, int SS,
                                    cx<T>* num, T* den, const int* skip) {
  if (skip && *skip) return;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= SS) return;
  const int sg = blockIdx.y;
  cx<T> a{T(0), T(0)};
  T b = T(0);
  for (int c = seg_beg[sg]; c < seg_beg[sg + 1]; ++c) {
    a += num_part[static_cast<int64_t>(c) * SS + pix];
    if (den_part) b += den_part[static_cast<int64_t>(c) * SS + pix];
  }
  num[static_cast<int64_t>(sg) * SS + pix] = a;
  if (den) den[static_cast<int64_t>(sg) * SS + pix] = b;
}

// W_d = (eta num + mu (w - Delta_d)) / (eta den + mu);  Delta_d += W_d - w
// (blind.cpp:246-251, 276-277); also publishes Delta_d + W_d for the next
// consensus average into wd_all[d].
template <typename T>
__global__ void probe_update_kernel(const cx<T>* num, const T* den, const cx<T>* w, cx<T>* wc, cx<T>* delta,
                                    cx<T>* wd_all, const int* local_map, int SS, T eta, T mu, const int* skip) {
  if (skip && *skip) return;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= SS) return;
  const int ld = blockIdx.y;
  const int64_t i = static_cast<int64_t>(ld) * SS + pix;
  const cx<T> wv = w[pix];
  const cx<T> dl = delta[i];
  const cx<T> n = num[i] * eta + (wv - dl) * mu;
  const T d = eta * den[i] + mu;
  const cx<T> wn{n.x / d, n.y / d};
  const cx<T> dn = dl + (wn - wv);
  wc[i] = wn;
  delta[i] = dn;
  wd_all[static_cast<int64_t>(local_map[ld]) * SS + pix] = dn + wn;
}

// avg = (sum_{d<D} (Delta_d + W_d)) / D  (blind.cpp:200-206, sum in d order)
template <typename T>
__global__ void probe_avg_kernel(const cx<T>* wd_all, int D, int SS, cx<T>* avg, const int* skip) {
  if (skip && *skip) return;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= SS) return;
  cx<T> a{T(0), T(0)};
  for (int d = 0; d < D; ++d) a += wd_all[static_cast<int64_t>(d) * SS + pix];
  avg[pix] = cx<T>{a.x / static_cast<T>(D), a.y / static_cast<T>(D)};
}

template <typename T>
__global__ void apply_mask_kernel(cx<T>* spec, const T* mask, int SS, const int* skip) {
  if (skip && *skip) return;
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= SS) return;
  if (mask[pix] == T(0)) spec[pix] = cx<T>{T(0), T(0)};
}

// checkerboard-signed amplitudes as complex frames (blind.cpp:219-222)
template <typename T>
__global__ void checker_kernel(const T* amp, int64_t nfr, int S, cx<T>* out) {
  const int64_t n = nfr * S * S;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int pix = static_cast<int>(i % (S * S));
    const int k = pix / S, l = pix % S;
    out[i] = cx<T>{((k + l) % 2 == 0) ? amp[i] : -amp[i], T(0)};
  }
}

template <typename T>
__global__ void frame_flux_kernel(const T* amp, int64_t per, double* out) {
  __shared__ double sm[32];
  const T* p = amp + blockIdx.x * per;
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < per; i += blockDim.x) {
    const double a = static_cast<double>(p[i]);
    acc += a * a;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += sm[w];
    out[blockIdx.x] = s;
  }
}

template <typename T>
__global__ void scale_copy_kernel(const cx<T>* in, cx<T>* out, int64_t n, double scale, int copies, int64_t stride) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const cx<T> v{static_cast<T>(static_cast<double>(in[i].x) * scale),
                  static_cast<T>(static_cast<double>(in[i].y) * scale)};
    for (int c = 0; c < copies; ++c) out[c * stride + i] = v;
  }
}

namespace {
inline dim3 pix_grid(int SS, int y) { return dim3(static_cast<unsigned>((SS + 127) / 128), static_cast<unsigned>(y)); }
}  // namespace

template <typename T>
cudaError_t launch_probe_partials(const cx<T>* img, const int64_t* off, const int32_t* pitch, const cx<T>* q,
                                  const int32_t* chunk_f0, const int32_t* chunk_f1, int nchunks, int S, int mode,
                                  cx<T>* num_part, T* den_part, const int* skip, cudaStream_t st) {
  if (nchunks <= 0) return cudaSuccess;
  probe_partials_kernel<T><<<pix_grid(S * S, nchunks), 128, 0, st>>>(img, off, pitch, q, chunk_f0, chunk_f1, S, mode,
                                                                    num_part, den_part, skip);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_chunk_reduce(const cx<T>* num_part, const T* den_part, const int32_t* seg_beg, int nseg, int SS,
                                cx<T>* num, T* den, const int* skip, cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  chunk_reduce_kernel<T><<<pix_grid(SS, nseg), 128, 0, st>>>(num_part, den_part, seg_beg, SS, num, den, skip);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_probe_update(const cx<T>* num, const T* den, const cx<T>* w, cx<T>* wc, cx<T>* delta,
                                cx<T>* wd_all, const int* local_map, int nls, int SS, T eta, T mu, const int* skip,
                                cudaStream_t st) {
  if (nls <= 0) return cudaSuccess;
  probe_update_kernel<T><<<pix_grid(SS, nls), 128, 0, st>>>(num, den, w, wc, delta, wd_all, local_map, SS, eta, mu,
                                                            skip);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_probe_avg(const cx<T>* wd_all, int D, int SS, cx<T>* avg, const int* skip, cudaStream_t st) {
  probe_avg_kernel<T><<<pix_grid(SS, 1), 128, 0, st>>>(wd_all, D, SS, avg, skip);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_apply_mask(cx<T>* spec, const T* mask, int SS, const int* skip, cudaStream_t st) {
  apply_mask_kernel<T><<<pix_grid(SS, 1), 128, 0, st>>>(spec, mask, SS, skip);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_checker(const T* amp, int64_t nfr, int S, cx<T>* out, cudaStream_t st) {
  const int64_t n = nfr * S * S;
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  checker_kernel<T><<<grid, 256, 0, st>>>(amp, nfr, S, out);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_frame_flux(const T* amp, int64_t nfr, int64_t per, double* out, cudaStream_t st) {
  if (nfr <= 0) return cudaSuccess;
  frame_flux_kernel<T><<<static_cast<unsigned>(nfr), 256, 0, st>>>(amp, per, out);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_scale_copy(const cx<T>* in, cx<T>* out, int64_t n, double scale, int copies, int64_t stride,
                              cudaStream_t st) {
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 1024));
  scale_copy_kernel<T><<<grid, 256, 0, st>>>(in, out, n, scale, copies, stride);
  return cudaGetLastError();
}

#define PDD_BLIND_INST(T)                                                                                            \
  template cudaError_t launch_probe_partials<T>(const cx<T>*, const int64_t*, const int32_t*, const cx<T>*,         \
                                                const int32_t*, const int32_t*, int, int, int, cx<T>*, T*,          \
                                                const int*, cudaStream_t);                                           \
  template cudaError_t launch_chunk_reduce<T>(const cx<T>*, const T*, const int32_t*, int, int, cx<T>*, T*,         \
                                              const int*, cudaStream_t);                                             \
  template cudaError_t launch_probe_update<T>(const cx<T>*, const T*, const cx<T>*, cx<T>*, cx<T>*, cx<T>*,         \
                                              const int*, int, int, T, T, const int*, cudaStream_t);                 \
  template cudaError_t launch_probe_avg<T>(const cx<T>*, int, int, cx<T>*, const int*, cudaStream_t);               \
  template cudaError_t launch_apply_mask<T>(cx<T>*, const T*, int, const int*, cudaStream_t);                       \
  template cudaError_t launch_checker<T>(const T*, int64_t, int, cx<T>*, cudaStream_t);                             \
  template cudaError_t launch_frame_flux<T>(const T*, int64_t, int64_t, double*, cudaStream_t);                     \
  template cudaError_t launch_scale_copy<T>(const cx<T>*, cx<T>*, int64_t, double, int, int64_t, cudaStream_t);
PDD_BLIND_INST(float)
PDD_BLIND_INST(double)

}  // namespace pdd
