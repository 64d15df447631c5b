// Stand-alone operators of the reference's public headers, on the GPU:
//   fft2_normalized / ifft2_normalized      (fft.hpp:8-15, fft.cpp:39-62)
//   forward / adjoint / illumination_density / probe_density / adjoint_probe /
//   intensity                               (forward.hpp:8-27, forward.cpp)
//   stagm::pixel_prox / value / gradient    (stagm.hpp:16-37, stagm.cpp)
//   r_factor / relative_error               (metrics.hpp:9-14, metrics.cpp:11-46)
// Host buffers in, host buffers out (the reference's value semantics); the
// device work reuses the solver kernels so these ops are parity probes of the
// same code the solvers run.  Square power-of-two frames use the register FFT;
// any other shape goes through a direct-DFT kernel (the reference's FFT tests
// use 16x12 and 4x5, test_field_fft.cpp:75-112).
#include <cmath>

#include "common.cuh"
#include "ops.hpp"

namespace pdd {
namespace {

// ---- generic separable DFT (any h, w) ---------------------------------------
template <typename T>
__global__ void dft_lines_kernel(const cx<T>* in, cx<T>* out, int lines, int len, int64_t line_stride,
                                 int64_t elem_stride, const cx<T>* tw, T scale) {
  const int64_t total = static_cast<int64_t>(lines) * len;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int line = static_cast<int>(i / len), k = static_cast<int>(i % len);
    const cx<T>* src = in + line * line_stride;
    cx<T> acc{T(0), T(0)};
    for (int t = 0; t < len; ++t)
      acc += src[t * elem_stride] * tw[(static_cast<int64_t>(k) * t) % len];
    out[line * line_stride + k * elem_stride] = acc * scale;
  }
}

template <typename T>
void generic_fft2(double* data, int64_t h, int64_t w, bool inverse, cudaStream_t st) {
  const int64_t n = h * w;
  DevMem a = upload(to_cx<T>(data, n), st), b(sizeof(cx<T>) * n);
  auto table = [&](int64_t len) {
    std::vector<cx<T>> t(static_cast<size_t>(len));
    for (int64_t k = 0; k < len; ++k) {
      const double ang = (inverse ? 2.0 : -2.0) * M_PI * static_cast<double>(k) / static_cast<double>(len);
      t[k] = cx<T>{static_cast<T>(std::cos(ang)), static_cast<T>(std::sin(ang))};
    }
    return upload(t, st);
  };
  DevMem tr = table(w), tc = table(h);
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 4096));
  // rows: lines = h, len = w; then columns: lines = w, len = h
  dft_lines_kernel<T><<<grid, 256, 0, st>>>(a.as<cx<T>>(), b.as<cx<T>>(), static_cast<int>(h), static_cast<int>(w),
                                             w, 1, tr.as<cx<T>>(), T(1));
  PDD_CUDA(cudaGetLastError());
  const T scale = static_cast<T>(1.0 / std::sqrt(static_cast<double>(n)));
  dft_lines_kernel<T><<<grid, 256, 0, st>>>(b.as<cx<T>>(), a.as<cx<T>>(), static_cast<int>(w), static_cast<int>(h),
                                             1, w, tc.as<cx<T>>(), scale);
  PDD_CUDA(cudaGetLastError());
  from_cx(download_cx<T>(a.get(), n, st), data);
}

// ---- frame ops over an arbitrary set of windows ----------------------------
// A one-subdomain plan covering the image, so the solver's layout/tile code
// (ascending-j gather) serves the stand-alone operators unchanged.
Plan single_plan(int64_t s, int64_t H, int64_t W, const int64_t* pos, int64_t J) {
  Geometry g;
  g.s = s;
  g.step = 1;
  g.H = H;
  g.W = W;
  g.grid_rows = 1;
  g.grid_cols = J;
  g.pos.assign(pos, pos + 2 * J);
  if (s < 1) throw InvalidArgument("forward model: probe shape != frame_side^2");
  for (int64_t j = 0; j < J; ++j)
    if (pos[2 * j] < 0 || pos[2 * j + 1] < 0 || pos[2 * j] + s > H || pos[2 * j + 1] + s > W)
      throw OutOfRange("extract: region exceeds field bounds");
  const int32_t zero = 0;
  std::vector<int32_t> assign(static_cast<size_t>(J), zero);
  const int64_t sub[4] = {0, H, 0, W};
  return plan_from_arrays(g, 1, assign.data(), sub, 0, nullptr, nullptr);
}

template <typename T>
struct FrameOp {
  Plan plan;
  Layout L;
  Stream stream;
  AllocStream scope{stream.get()};  // temporaries of the op are ordered on its stream
  DevMem tw, fr_off, fr_pitch, fr_r, fr_c, fr_sub, tiles, tile_frames, sub_off, sub_h, sub_w, sub_pbeg, scratch;
  int S;
  FrameOp(int64_t s, int64_t H, int64_t W, const int64_t* pos, int64_t J)
      : plan(single_plan(s, H, W, pos, J)), L(Layout::build(plan, 0, 1)), S(static_cast<int>(s)) {
    if (!frame_supported<T>(S))
      throw InvalidArgument("forward model: frame side " + std::to_string(s) + " not supported by the CUDA path");
    cudaStream_t st = stream.get();
    tw = upload(twiddles<T>(S), st);
    fr_off = upload(L.fr_off, st);
    fr_pitch = upload(L.fr_pitch, st);
    fr_r = upload(L.fr_r, st);
    fr_c = upload(L.fr_c, st);
    fr_sub = upload(L.fr_sub, st);
    tiles = upload(L.tiles, st);
    tile_frames = upload(L.tile_frames, st);
    sub_off = upload(L.sub_img_off, st);
    sub_h = upload(L.sub_h, st);
    sub_w = upload(L.sub_w, st);
    std::vector<int32_t> pb(2, 0);
    sub_pbeg = upload(pb, st);
    if (const size_t b = stream_scratch_bytes<T>(S)) scratch.alloc(b, st);
  }
  FrameArgs<T> fargs() const {
    FrameArgs<T> a;
    a.nframes = static_cast<int>(L.nfr);
    a.tw = tw.as<cx<T>>();
    a.off = fr_off.as<int64_t>();
    a.pitch = fr_pitch.as<int32_t>();
    a.scale = static_cast<T>(1.0 / static_cast<double>(S));
    a.scratch = scratch.as<cx<T>>();
    return a;
  }
  template <typename U>
  GatherArgs<U> gargs(int mode) const {
    GatherArgs<U> g;
    g.mode = mode;
    g.ntiles = L.ntiles();
    g.tile_h = L.tile_h;
    g.tile_w = L.tile_w;
    g.tiles = tiles.as<int4>();
    g.tile_frames = tile_frames.as<int32_t>();
    g.fr_r = fr_r.as<int32_t>();
    g.fr_c = fr_c.as<int32_t>();
    g.fr_sub = fr_sub.as<int32_t>();
    g.S = S;
    g.sub_off = sub_off.as<int64_t>();
    g.sub_h = sub_h.as<int32_t>();
    g.sub_w = sub_w.as<int32_t>();
    g.sub_pbeg = sub_pbeg.as<int32_t>();
    return g;
  }
};

// Probe-shaped reductions over frames (forward.cpp:68-93), deterministic:
// frames split into fixed chunks, each chunk summed in ascending j, chunks
// then summed in order.
template <typename T>
__global__ void probe_sums_kernel(const cx<T>* img, const int64_t* off, const int32_t* pitch, const cx<T>* q,
                                  int nframes, int S, int chunk, cx<T>* num_part, T* den_part) {
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  const int SS = S * S;
  if (pix >= SS) return;
  const int y = pix / S, x = pix % S;
  const int f0 = blockIdx.y * chunk, f1 = min(nframes, f0 + chunk);
  cx<T> num{T(0), T(0)};
  T den = T(0);
  for (int f = f0; f < f1; ++f) {
    const cx<T> u = img[off[f] + static_cast<int64_t>(y) * pitch[f] + x];
    den += norm2(u);
    if (q) num += mul_conj(q[static_cast<int64_t>(f) * SS + pix], u);
  }
  if (num_part) num_part[static_cast<int64_t>(blockIdx.y) * SS + pix] = num;
  den_part[static_cast<int64_t>(blockIdx.y) * SS + pix] = den;
}

template <typename T>
__global__ void chunk_sum_kernel(const cx<T>* num_part, const T* den_part, int nchunks, int SS, cx<T>* num,
                                 T* den) {
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= SS) return;
  cx<T> a{T(0), T(0)};
  T b = T(0);
  for (int c = 0; c < nchunks; ++c) {
    if (num_part) a += num_part[static_cast<int64_t>(c) * SS + pix];
    b += den_part[static_cast<int64_t>(c) * SS + pix];
  }
  if (num) num[pix] = a;
  den[pix] = b;
}

template <typename T>
__global__ void prox_kernel(const double* y, const double* b, int64_t n, T lam, T eps, int fast, double* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const cx<T> yy{static_cast<T>(y[2 * i]), static_cast<T>(y[2 * i + 1])};
    const cx<T> z = stagm_prox(yy, static_cast<T>(sqrt(b[i])), lam, eps, fast != 0);
    out[2 * i] = static_cast<double>(z.x);
    out[2 * i + 1] = static_cast<double>(z.y);
  }
}

// stagm.cpp:29-43
template <typename T>
__global__ void value_grad_kernel(const double* xin, const double* b, int64_t n, T eps, double* val, double* grad) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const cx<T> x{static_cast<T>(xin[2 * i]), static_cast<T>(xin[2 * i + 1])};
    const T ax = sqrt(norm2(x));
    const T bb = static_cast<T>(b[i]);
    const T rb = sqrt(bb);
    T v;
    cx<T> g;
    if (ax < eps * rb) {
      v = T(0.5) * (T(1) - eps) * (bb - ax * ax / eps);
      g = x * (T(1) - T(1) / eps);
    } else {
      const T d = ax - rb;
      v = T(0.5) * d * d;
      g = ax == T(0) ? cx<T>{T(0), T(0)} : x * (T(1) - rb / ax);
    }
    if (val) val[i] = static_cast<double>(v);
    if (grad) {
      grad[2 * i] = static_cast<double>(g.x);
      grad[2 * i + 1] = static_cast<double>(g.y);
    }
  }
}

template <typename T>
__global__ void intensity_kernel(const double* z, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T a = static_cast<T>(z[2 * i]), b = static_cast<T>(z[2 * i + 1]);
    out[i] = static_cast<double>(a * a + b * b);
  }
}

template <typename T>
__global__ void rel_err_kernel(const double* cur, const double* prev, int64_t n, double* part) {
  __shared__ double sm[64];
  double diff = 0.0, nrm = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const T cr = static_cast<T>(cur[2 * i]), ci = static_cast<T>(cur[2 * i + 1]);
    const T dr = cr - static_cast<T>(prev[2 * i]), di = ci - static_cast<T>(prev[2 * i + 1]);
    diff += static_cast<double>(dr * dr + di * di);
    nrm += static_cast<double>(cr * cr + ci * ci);
  }
  for (int o = 16; o > 0; o >>= 1) {
    diff += __shfl_down_sync(0xffffffffu, diff, o);
    nrm += __shfl_down_sync(0xffffffffu, nrm, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sm[2 * (threadIdx.x >> 5)] = diff;
    sm[2 * (threadIdx.x >> 5) + 1] = nrm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      a += sm[2 * w];
      b += sm[2 * w + 1];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

template <typename T>
DevMem up_double_as_cx(const double* p, int64_t n, cudaStream_t st) {
  return upload(to_cx<T>(p, n), st);
}

template <typename T>
DevMem up_doubles(const double* p, int64_t n, cudaStream_t st) {
  DevMem m(sizeof(double) * std::max<int64_t>(n, 1));
  if (n) PDD_CUDA(cudaMemcpyAsync(m.get(), p, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  return m;
}

int grid_for(int64_t n) { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 4096)); }

}  // namespace

template <typename T>
void op_fft2(double* data, int64_t h, int64_t w, bool inverse) {
  if (h < 1 || w < 1) throw InvalidArgument("ComplexField2D: height, width must be >= 1");
  if (h != w || !frame_supported<T>(static_cast<int>(h))) {
    Stream s;
    AllocStream scope(s.get());
    generic_fft2<T>(data, h, w, inverse, s.get());
    return;
  }
  const int64_t pos[2] = {0, 0};
  FrameOp<T> op(h, h, w, pos, 1);
  cudaStream_t st = op.stream.get();
  std::vector<cx<T>> ones(static_cast<size_t>(h * w), cx<T>{T(1), T(0)});
  DevMem one = upload(ones, st), x = up_double_as_cx<T>(data, h * w, st), y(sizeof(cx<T>) * h * w);
  FrameArgs<T> a = op.fargs();
  a.probe = one.as<cx<T>>();
  if (!inverse) {
    a.img = x.as<cx<T>>();
    a.frames_out = y.as<cx<T>>();
    PDD_CUDA(launch_frame<T>(kFwd, op.S, a, st));
  } else {
    a.frames_in = x.as<cx<T>>();
    a.bp_out = y.as<cx<T>>();
    PDD_CUDA(launch_frame<T>(kAdj, op.S, a, st));
  }
  from_cx(download_cx<T>(y.get(), h * w, st), data);
}

template <typename T>
void op_forward(const double* probe, int64_t s, const double* image, int64_t H, int64_t W, const int64_t* pos,
                int64_t J, double* frames_out, double* intensity_out) {
  FrameOp<T> op(s, H, W, pos, J);
  cudaStream_t st = op.stream.get();
  DevMem p = up_double_as_cx<T>(probe, s * s, st), img = up_double_as_cx<T>(image, H * W, st);
  DevMem out(sizeof(cx<T>) * std::max<int64_t>(J * s * s, 1)), inten(sizeof(T) * std::max<int64_t>(J * s * s, 1));
  FrameArgs<T> a = op.fargs();
  a.probe = p.as<cx<T>>();
  a.img = img.as<cx<T>>();
  a.frames_out = frames_out ? out.as<cx<T>>() : nullptr;
  a.inten_out = intensity_out ? inten.as<T>() : nullptr;
  PDD_CUDA(launch_frame<T>(kFwd, op.S, a, st));
  if (frames_out) from_cx(download_cx<T>(out.get(), J * s * s, st), frames_out);
  if (intensity_out) {
    std::vector<T> h(static_cast<size_t>(J * s * s));
    PDD_CUDA(cudaMemcpyAsync(h.data(), inten.get(), sizeof(T) * h.size(), cudaMemcpyDeviceToHost, st));
    PDD_CUDA(cudaStreamSynchronize(st));
    for (size_t i = 0; i < h.size(); ++i) intensity_out[i] = static_cast<double>(h[i]);
  }
}

template <typename T>
__global__ void widen_kernel(const T* in, double* out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<double>(in[i]);
}

template <typename T>
void op_simulate_device(const double* probe, int64_t s, const double* image, int64_t H, int64_t W, const int64_t* pos,
                        int64_t J, double* intensity_dev) {
  FrameOp<T> op(s, H, W, pos, J);
  cudaStream_t st = op.stream.get();
  DevMem p = up_double_as_cx<T>(probe, s * s, st), img = up_double_as_cx<T>(image, H * W, st);
  FrameArgs<T> a = op.fargs();
  a.probe = p.as<cx<T>>();
  a.img = img.as<cx<T>>();
  if constexpr (sizeof(T) == sizeof(double)) {
    a.inten_out = reinterpret_cast<T*>(intensity_dev);
    PDD_CUDA(launch_frame<T>(kFwd, op.S, a, st));
  } else {
    DevMem tmp(sizeof(T) * std::max<int64_t>(J * s * s, 1));
    a.inten_out = tmp.as<T>();
    PDD_CUDA(launch_frame<T>(kFwd, op.S, a, st));
    widen_kernel<T><<<grid_for(J * s * s), 256, 0, st>>>(tmp.as<T>(), intensity_dev, J * s * s);
    PDD_CUDA(cudaGetLastError());
  }
  PDD_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void op_adjoint(const double* probe, int64_t s, const double* frames, const int64_t* pos, int64_t J, int64_t H,
                int64_t W, double* out) {
  FrameOp<T> op(s, H, W, pos, J);
  cudaStream_t st = op.stream.get();
  DevMem p = up_double_as_cx<T>(probe, s * s, st), fr = up_double_as_cx<T>(frames, J * s * s, st);
  DevMem bp(sizeof(cx<T>) * std::max<int64_t>(J * s * s, 1)), img(sizeof(cx<T>) * H * W);
  FrameArgs<T> a = op.fargs();
  a.probe = p.as<cx<T>>();
  a.frames_in = fr.as<cx<T>>();
  a.bp_out = bp.as<cx<T>>();
  PDD_CUDA(launch_frame<T>(kAdj, op.S, a, st));
  GatherArgs<T> g = op.template gargs<T>(kGatherAdjoint);
  g.bp = bp.as<cx<T>>();
  g.out = img.as<cx<T>>();
  PDD_CUDA(launch_gather<T>(g, st));
  from_cx(download_cx<T>(img.get(), H * W, st), out);
}

template <typename T>
void op_illumination_density(const double* probe, int64_t s, const int64_t* pos, int64_t J, int64_t H, int64_t W,
                             double* out) {
  FrameOp<T> op(s, H, W, pos, J);
  cudaStream_t st = op.stream.get();
  DevMem p = up_double_as_cx<T>(probe, s * s, st), dens(sizeof(double) * H * W);
  GatherArgs<T> g = op.template gargs<T>(kGatherDensity);
  g.probe = p.as<cx<T>>();
  g.dens_out = dens.as<double>();
  PDD_CUDA(launch_gather<T>(g, st));
  PDD_CUDA(cudaMemcpyAsync(out, dens.get(), sizeof(double) * H * W, cudaMemcpyDeviceToHost, st));
  PDD_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void op_probe_sums(const double* image, int64_t H, int64_t W, const double* frames, const int64_t* pos, int64_t J,
                   int64_t s, double* num_out, double* den_out) {
  FrameOp<T> op(s, H, W, pos, J);
  cudaStream_t st = op.stream.get();
  const int64_t SS = s * s;
  DevMem img = up_double_as_cx<T>(image, H * W, st);
  DevMem q;
  if (frames) {  // q_j = IFFT(frame_j)
    DevMem fr = up_double_as_cx<T>(frames, J * SS, st);
    std::vector<cx<T>> ones(static_cast<size_t>(SS), cx<T>{T(1), T(0)});
    DevMem one = upload(ones, st);
    q.alloc(sizeof(cx<T>) * std::max<int64_t>(J * SS, 1));
    FrameArgs<T> a = op.fargs();
    a.probe = one.as<cx<T>>();
    a.frames_in = fr.as<cx<T>>();
    a.bp_out = q.as<cx<T>>();
    PDD_CUDA(launch_frame<T>(kAdj, op.S, a, st));
    PDD_CUDA(cudaStreamSynchronize(st));
  }
  const int chunk = 64;
  const int nch = static_cast<int>(std::max<int64_t>(1, (J + chunk - 1) / chunk));
  DevMem np(sizeof(cx<T>) * nch * SS), dp(sizeof(T) * nch * SS), num(sizeof(cx<T>) * SS), den(sizeof(T) * SS);
  dim3 grid(static_cast<unsigned>((SS + 127) / 128), nch);
  probe_sums_kernel<T><<<grid, 128, 0, st>>>(img.as<cx<T>>(), op.fr_off.template as<int64_t>(),
                                             op.fr_pitch.template as<int32_t>(), frames ? q.as<cx<T>>() : nullptr,
                                             static_cast<int>(J), static_cast<int>(s), chunk,
                                             frames ? np.as<cx<T>>() : nullptr, dp.as<T>());
  PDD_CUDA(cudaGetLastError());
  chunk_sum_kernel<T><<<static_cast<unsigned>((SS + 127) / 128), 128, 0, st>>>(
      frames ? np.as<cx<T>>() : nullptr, dp.as<T>(), nch, static_cast<int>(SS), frames ? num.as<cx<T>>() : nullptr,
      den.as<T>());
  PDD_CUDA(cudaGetLastError());
  if (num_out && frames) from_cx(download_cx<T>(num.get(), SS, st), num_out);
  if (den_out) {
    std::vector<T> h(static_cast<size_t>(SS));
    PDD_CUDA(cudaMemcpyAsync(h.data(), den.get(), sizeof(T) * SS, cudaMemcpyDeviceToHost, st));
    PDD_CUDA(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < SS; ++i) den_out[i] = static_cast<double>(h[i]);
  }
}

template <typename T>
void op_prox(const double* y, const double* b, int64_t n, double lambda, double eps, double* out) {
  if (!(eps > 0.0 && eps < 1.0)) throw InvalidArgument("stagm: epsilon must lie in (0,1)");
  if (lambda <= 0.0) throw InvalidArgument("stagm::prox: lambda must be positive");
  Stream s;
  AllocStream scope(s.get());
  cudaStream_t st = s.get();
  DevMem dy = up_doubles<T>(y, 2 * n, st), db = up_doubles<T>(b, n, st), dz(sizeof(double) * 2 * std::max<int64_t>(n, 1));
  prox_kernel<T><<<grid_for(n), 256, 0, st>>>(dy.as<double>(), db.as<double>(), n, static_cast<T>(lambda),
                                              static_cast<T>(eps), 0, dz.as<double>());
  PDD_CUDA(cudaGetLastError());
  PDD_CUDA(cudaMemcpyAsync(out, dz.get(), sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
  PDD_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void op_value_gradient(const double* x, const double* b, int64_t n, double eps, double* val, double* grad) {
  if (!(eps > 0.0 && eps < 1.0)) throw InvalidArgument("stagm: epsilon must lie in (0,1)");
  Stream s;
  AllocStream scope(s.get());
  cudaStream_t st = s.get();
  DevMem dx = up_doubles<T>(x, 2 * n, st), db = up_doubles<T>(b, n, st);
  DevMem dv(sizeof(double) * std::max<int64_t>(n, 1)), dg(sizeof(double) * 2 * std::max<int64_t>(n, 1));
  value_grad_kernel<T><<<grid_for(n), 256, 0, st>>>(dx.as<double>(), db.as<double>(), n, static_cast<T>(eps),
                                                    dv.as<double>(), dg.as<double>());
  PDD_CUDA(cudaGetLastError());
  if (val) PDD_CUDA(cudaMemcpyAsync(val, dv.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  if (grad) PDD_CUDA(cudaMemcpyAsync(grad, dg.get(), sizeof(double) * 2 * n, cudaMemcpyDeviceToHost, st));
  PDD_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void op_intensity(const double* z, int64_t n, double* out) {
  Stream s;
  AllocStream scope(s.get());
  cudaStream_t st = s.get();
  DevMem dz = up_doubles<T>(z, 2 * n, st), di(sizeof(double) * std::max<int64_t>(n, 1));
  intensity_kernel<T><<<grid_for(n), 256, 0, st>>>(dz.as<double>(), n, di.as<double>());
  PDD_CUDA(cudaGetLastError());
  PDD_CUDA(cudaMemcpyAsync(out, di.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  PDD_CUDA(cudaStreamSynchronize(st));
}

template <typename T>
void op_diff_norm(const double* cur, const double* prev, int64_t n, double* diff, double* norm) {
  Stream s;
  AllocStream scope(s.get());
  cudaStream_t st = s.get();
  DevMem a = up_doubles<T>(cur, 2 * n, st), b = up_doubles<T>(prev, 2 * n, st);
  const int nb = static_cast<int>(std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 256));
  DevMem part(sizeof(double) * 2 * nb);
  rel_err_kernel<T><<<nb, 256, 0, st>>>(a.as<double>(), b.as<double>(), n, part.as<double>());
  PDD_CUDA(cudaGetLastError());
  std::vector<double> h(2 * nb);
  PDD_CUDA(cudaMemcpyAsync(h.data(), part.get(), sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, st));
  PDD_CUDA(cudaStreamSynchronize(st));
  *diff = 0.0;
  *norm = 0.0;
  for (int i = 0; i < nb; ++i) {
    *diff += h[2 * i];
    *norm += h[2 * i + 1];
  }
}

// r_factor (metrics.cpp:11-27): forward each subdomain image, compare with sqrt(f).
template <typename T>
double op_r_factor(const Plan& plan, const double* subs, const double* intensities, const double* probe) {
  RankData<T> R;
  AllocStream scope(R.st());
  DataSpec data{intensities, kIntensityF64, false};
  R.build(plan, data, nullptr, 0, nullptr, 1, "r_factor");
  if (R.l1 <= 0.0) throw InvalidArgument("r_factor: all-zero data, metric undefined");
  cudaStream_t st = R.st();
  DevMem p = up_double_as_cx<T>(probe, R.SS(), st), u = up_double_as_cx<T>(subs, R.L.img_elems, st);
  FrameArgs<T> a = R.frame_args();
  a.probe = p.as<cx<T>>();
  a.img = u.as<cx<T>>();
  a.rf_part = R.rf_part.template as<double>();
  PDD_CUDA(launch_frame<T>(kFwd, R.S, a, st));
  R.reduce_rf(false);
  std::vector<double> sub(R.D);
  PDD_CUDA(cudaMemcpyAsync(sub.data(), R.rf_sub(), sizeof(double) * R.D, cudaMemcpyDeviceToHost, st));
  PDD_CUDA(cudaStreamSynchronize(st));
  double num = 0.0;
  for (double x : sub) num += x;
  return num / R.l1;
}

#define PDD_INST(T)                                                                                                 \
  template void op_fft2<T>(double*, int64_t, int64_t, bool);                                                        \
  template void op_forward<T>(const double*, int64_t, const double*, int64_t, int64_t, const int64_t*, int64_t,    \
                              double*, double*);                                                                    \
  template void op_simulate_device<T>(const double*, int64_t, const double*, int64_t, int64_t, const int64_t*,      \
                                      int64_t, double*);                                                            \
  template void op_adjoint<T>(const double*, int64_t, const double*, const int64_t*, int64_t, int64_t, int64_t,    \
                              double*);                                                                             \
  template void op_illumination_density<T>(const double*, int64_t, const int64_t*, int64_t, int64_t, int64_t,      \
                                           double*);                                                                \
  template void op_probe_sums<T>(const double*, int64_t, int64_t, const double*, const int64_t*, int64_t, int64_t, \
                                 double*, double*);                                                                 \
  template void op_prox<T>(const double*, const double*, int64_t, double, double, double*);                         \
  template void op_value_gradient<T>(const double*, const double*, int64_t, double, double*, double*);              \
  template void op_intensity<T>(const double*, int64_t, double*);                                                   \
  template void op_diff_norm<T>(const double*, const double*, int64_t, double*, double*);                            \
  template double op_r_factor<T>(const Plan&, const double*, const double*, const double*);
PDD_INST(float)
PDD_INST(double)

}  // namespace pdd
