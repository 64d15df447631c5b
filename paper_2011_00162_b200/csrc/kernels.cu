// CUDA kernels of the OD²P iteration (sm_100a) and their launchers.
//
// frame_kernel (frame_kernel.cuh) carries the FFT-bound per-frame work; the
// kernels here are the HBM-bound image-side passes:
//   gather_kernel : deterministic overlap-add, i.e. the embed_add loop of
//                   adjoint (forward.cpp:43-54) in gather form -- every output
//                   pixel sums its covering frames in ascending frame index,
//                   the reference's accumulation order -- fused with the
//                   u-update, the Lambda-update and the RE partials of
//                   solver.cpp:154-193 (or blind.cpp:253-277).
//   pack / vstep  : the overlap consensus v = (s_1 + s_2)/2 with
//                   s_side = u_side|overlap + Lambda_side (solver.cpp:141-151);
//                   packing s separately is what makes the multi-GPU exchange a
//                   single send/recv of s per pair.
//   segsum        : fixed-shape reductions of per-frame / per-tile partials
//                   (bit-identical for any GPU count at fixed D).
#include <cuda_runtime.h>

#include <cmath>
#include <type_traits>

#include "frame_kernel.cuh"
#include "frame_stream.cuh"
#include "kernels.hpp"

namespace pdd {

// ---------------------------------------------------------------------------
// frame kernel dispatch
template <typename T, int S>
struct FrameCfg;
// float: whole rows in registers up to S = 32; two-level rows beyond.
template <> struct FrameCfg<float, 2> { static constexpr int R = 2, FPB = 64; };
template <> struct FrameCfg<float, 4> { static constexpr int R = 4, FPB = 32; };
template <> struct FrameCfg<float, 8> { static constexpr int R = 8, FPB = 16; };
template <> struct FrameCfg<float, 16> { static constexpr int R = 16, FPB = 8; };
template <> struct FrameCfg<float, 32> { static constexpr int R = 32, FPB = 4; };
template <> struct FrameCfg<float, 64> { static constexpr int R = 16, FPB = 1; };
template <> struct FrameCfg<float, 128> { static constexpr int R = 32, FPB = 1; };
template <> struct FrameCfg<double, 2> { static constexpr int R = 2, FPB = 64; };
template <> struct FrameCfg<double, 4> { static constexpr int R = 4, FPB = 32; };
template <> struct FrameCfg<double, 8> { static constexpr int R = 8, FPB = 16; };
template <> struct FrameCfg<double, 16> { static constexpr int R = 16, FPB = 8; };
template <> struct FrameCfg<double, 32> { static constexpr int R = 16, FPB = 2; };
template <> struct FrameCfg<double, 64> { static constexpr int R = 16, FPB = 1; };

// Streamed SWEEP kernel shapes (frame_stream.cuh) for the large frames.
template <typename T, int S>
struct StreamPick {
  using type = void;
};
template <> struct StreamPick<float, 128> { using type = StreamShape<128, 512, 8, 8>; };
// 64^2 complex64: 8 values per thread on both axes (two row batches of 32 rows,
// two column groups), 111 registers, two CTAs per SM.  16 row values per thread
// (row split 4) measured 0.375 vs 0.339 ms per config-3 iteration.
#ifndef PDD_S64_NT  // A/B builds: threads, row split, CTAs per SM
#define PDD_S64_NT 256
#define PDD_S64_GR 8
#define PDD_S64_MINB 2
#endif
template <> struct StreamPick<float, 64> { using type = StreamShape<64, PDD_S64_NT, PDD_S64_GR, 8, PDD_S64_MINB>; };
// complex128 128^2: 16 values per thread on both axes (64 registers), the
// transpose tile in global scratch (tile_in_global), 8 warps per CTA.
template <> struct StreamPick<double, 128> { using type = StreamShape<128, 256, 8, 8, 1>; };

template <typename T, class SH>
constexpr bool stream_tmem_probe() {  // TMEM probe cache where it keeps occupancy (one CTA per SM)
  return std::is_same_v<T, float> && SH::MINB == 1;
}

// Shapes whose BLIND frame pass runs as ONE streamed launch (RF2: the shared-probe
// R-factor transform inside the sweep): shared-memory tile, room for a second one.
template <typename T, class SH>
constexpr bool stream_rf2() {
  return !stream_tmem_probe<T, SH>() && !tile_in_global<T, SH>() && !amp_tile_staged<T, SH, false>() &&
         2 * sizeof(cx<T>) * static_cast<size_t>(SH::S) * SH::P * SH::MINB <= (size_t(200) << 10);
}

template <typename T, class SH, bool FAST, bool FWD = false, bool ADJ = false, bool RF2 = false>
static cudaError_t launch_stream(const FrameArgs<T>& a, cudaStream_t st) {
  auto kern = sweep_stream_kernel<T, SH, FAST, stream_tmem_probe<T, SH>(), FWD, ADJ, RF2>;
  const size_t smem = stream_smem_bytes<T, SH>(RF2);
  static int blocks_per_sm = 0;
  static int sms = 0;
  if (!blocks_per_sm) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, SH::NT, smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (blocks_per_sm < 1) return cudaErrorInvalidConfiguration;
  }
  if (a.nframes <= 0) return cudaSuccess;
  // SWEEP runs the host schedule, built for exactly this grid
  if (!FWD && !ADJ && (!a.cta_beg || a.ncta != blocks_per_sm * sms)) return cudaErrorInvalidConfiguration;
  // global transpose tiles: one per CTA of the full persistent grid
  if (tile_in_global<T, SH>() && !a.scratch) return cudaErrorInvalidValue;
  const int grid = (FWD || ADJ) ? std::min(a.nframes, blocks_per_sm * sms) : a.ncta;
  kern<<<grid, SH::NT, smem, st>>>(a);
#ifdef PDD_PHASE_TIMING  // diagnostic builds (not capturable): per-phase cycles summed over CTAs
  {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusNone) {
      cudaStreamSynchronize(st);
      unsigned long long h[4] = {0, 0, 0, 0}, z[4] = {0, 0, 0, 0};
      cudaMemcpyFromSymbol(h, g_phase_cycles, sizeof(h));
      cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
      fprintf(stderr, "PDD_PHASE S=%d FWD=%d grid=%d frames=%d: barrier+rfsum %.0f  columns %.0f  rows_inv %.0f  rows_fwd_next %.0f (cycles per CTA)\n",
              SH::S, int(FWD), grid, a.nframes, double(h[0]) / grid, double(h[1]) / grid, double(h[2]) / grid, double(h[3]) / grid);
    }
  }
#endif
  return cudaGetLastError();
}

// Persistent grid of the streamed SWEEP kernel for side S (0: not streamed);
// the host builds the back-projection piece schedule for exactly this grid.
template <typename T>
int sweep_stream_ctas(int S) {
  auto q = [](auto kern, int nt, size_t smem) {
    int bps = 0, sms = 0, dev = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, nt, smem) != cudaSuccess)
      return 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return bps * sms;
  };
  if constexpr (std::is_same_v<T, float>) {
    if (S == 128) {
      using SH = StreamPick<float, 128>::type;
      return q(sweep_stream_kernel<float, SH, true, SH::MINB == 1, false>, SH::NT, stream_smem_bytes<float, SH>());
    }
    if (S == 64) {
      using SH = StreamPick<float, 64>::type;
      return q(sweep_stream_kernel<float, SH, true, SH::MINB == 1, false>, SH::NT, stream_smem_bytes<float, SH>());
    }
  } else {
    if (S == 128) {
      using SH = StreamPick<double, 128>::type;
      return q(sweep_stream_kernel<double, SH, true, false, false>, SH::NT, stream_smem_bytes<double, SH>());
    }
  }
  return 0;
}
template int sweep_stream_ctas<float>(int);
template int sweep_stream_ctas<double>(int);

// Bytes of global transpose-tile scratch the streamed kernels of side S need
// (0: their tile lives in shared memory): one tile per CTA of the persistent grid.
template <typename T>
size_t stream_scratch_bytes(int S) {
  if constexpr (std::is_same_v<T, double>) {
    if (S == 128) {
      using SH = StreamPick<double, 128>::type;
      return sizeof(cx<double>) * static_cast<size_t>(SH::S) * SH::P * static_cast<size_t>(sweep_stream_ctas<T>(S));
    }
  }
  return 0;
}
template size_t stream_scratch_bytes<float>(int);
template size_t stream_scratch_bytes<double>(int);

template <typename T, int S, int MODE>
static cudaError_t launch_frame_s(const FrameArgs<T>& a, cudaStream_t st) {
  if constexpr (MODE == kSweep && !std::is_same_v<typename StreamPick<T, S>::type, void>) {
    using SH = typename StreamPick<T, S>::type;
    return a.fast_prox ? launch_stream<T, SH, true>(a, st) : launch_stream<T, SH, false>(a, st);
  }
  if constexpr (MODE == kFwd && !std::is_same_v<typename StreamPick<T, S>::type, void>) {
    using SH = typename StreamPick<T, S>::type;
    return a.fast_prox ? launch_stream<T, SH, true, true>(a, st) : launch_stream<T, SH, false, true>(a, st);
  }
  if constexpr (MODE == kAdj && !std::is_same_v<typename StreamPick<T, S>::type, void>) {
    using SH = typename StreamPick<T, S>::type;
    if constexpr (tile_in_global<T, SH>()) return launch_stream<T, SH, true, false, true>(a, st);
  }
  if constexpr (MODE == kBlind && !std::is_same_v<typename StreamPick<T, S>::type, void>) {
    using SH = typename StreamPick<T, S>::type;
    if constexpr (stream_rf2<T, SH>()) {
      // one pass: the sweep with the subdomain copies W_d (raw q_j output) and,
      // inside it, the R-factor transform with the shared probe w (probe2)
      if (a.rf_part && a.probe2) {
        FrameArgs<T> sw = a;
        sw.bp_raw = 1;
        return a.fast_prox ? launch_stream<T, SH, true, false, false, true>(sw, st)
                           : launch_stream<T, SH, false, false, false, true>(sw, st);
      }
    }
    if constexpr (!stream_tmem_probe<T, SH>()) {  // no TMEM probe cache: per-frame probe tiles are fine
      // BLIND = R-factor forward with the shared probe w (probe2), then the
      // SWEEP with the subdomain copies W_d and raw q_j output
      FrameArgs<T> rf = a;
      rf.probe = a.probe2;
      rf.probe_idx = nullptr;
      rf.frames_out = nullptr;
      rf.inten_out = nullptr;
      cudaError_t e = a.rf_part ? launch_frame_s<T, S, kFwd>(rf, st) : cudaSuccess;
      if (e != cudaSuccess) return e;
      FrameArgs<T> sw = a;
      sw.rf_part = nullptr;
      sw.bp_raw = 1;
      return a.fast_prox ? launch_stream<T, SH, true>(sw, st) : launch_stream<T, SH, false>(sw, st);
    }
  }
  if constexpr (std::is_same_v<T, double> && S == 128) {
    return cudaErrorInvalidValue;  // every mode runs the streamed kernel above
  } else {
  using C = FrameCfg<T, S>;
  using E = Fft2<T, S, C::R>;
  constexpr int threads = E::NT * C::FPB;
  constexpr int nw = (E::NT + 31) / 32;
  const size_t smem = sizeof(cx<T>) * (S + static_cast<size_t>(C::FPB) * E::TILE) + sizeof(double) * C::FPB * nw;
  auto kern = frame_kernel<T, S, C::R, C::FPB, MODE>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (a.nframes <= 0) return cudaSuccess;
  const int grid = (a.nframes + C::FPB - 1) / C::FPB;
  kern<<<grid, threads, smem, st>>>(a);
  return cudaGetLastError();
  }
}

template <typename T, int S>
static cudaError_t launch_frame_mode(int mode, const FrameArgs<T>& a, cudaStream_t st) {
  switch (mode) {
    case kFwd: return launch_frame_s<T, S, kFwd>(a, st);
    case kAdj: return launch_frame_s<T, S, kAdj>(a, st);
    case kSweep: return launch_frame_s<T, S, kSweep>(a, st);
    case kBlind: return launch_frame_s<T, S, kBlind>(a, st);
  }
  return cudaErrorInvalidValue;
}

template <>
bool frame_supported<float>(int S) {
  return S == 2 || S == 4 || S == 8 || S == 16 || S == 32 || S == 64 || S == 128;
}
template <>
bool frame_supported<double>(int S) {
  return S == 2 || S == 4 || S == 8 || S == 16 || S == 32 || S == 64 || S == 128;
}

template <>
cudaError_t launch_frame<float>(int mode, int S, const FrameArgs<float>& a, cudaStream_t st) {
  switch (S) {
    case 2: return launch_frame_mode<float, 2>(mode, a, st);
    case 4: return launch_frame_mode<float, 4>(mode, a, st);
    case 8: return launch_frame_mode<float, 8>(mode, a, st);
    case 16: return launch_frame_mode<float, 16>(mode, a, st);
    case 32: return launch_frame_mode<float, 32>(mode, a, st);
    case 64: return launch_frame_mode<float, 64>(mode, a, st);
    case 128: return launch_frame_mode<float, 128>(mode, a, st);
  }
  return cudaErrorInvalidValue;
}
template <>
cudaError_t launch_frame<double>(int mode, int S, const FrameArgs<double>& a, cudaStream_t st) {
  switch (S) {
    case 2: return launch_frame_mode<double, 2>(mode, a, st);
    case 4: return launch_frame_mode<double, 4>(mode, a, st);
    case 8: return launch_frame_mode<double, 8>(mode, a, st);
    case 16: return launch_frame_mode<double, 16>(mode, a, st);
    case 32: return launch_frame_mode<double, 32>(mode, a, st);
    case 64: return launch_frame_mode<double, 64>(mode, a, st);
    case 128: return launch_frame_mode<double, 128>(mode, a, st);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Blind w-step in one launch (blind.cpp:194-208): avg = sum_d (Delta_d + W_d) / D
// (d order) -> FFT2 -> support mask -> IFFT2 -> w.  One CTA, the frame engine
// of fft.cuh; replaces probe_avg + forward + apply_mask + adjoint launches.
template <typename T, int S, int R>
__global__ void __launch_bounds__(Fft2<T, S, R>::NT) wstep_kernel(const cx<T>* wd_all, int D, const T* mask,
                                                                  const cx<T>* twg, T scale, cx<T>* w,
                                                                  const int* skip) {
  using E = Fft2<T, S, R>;
  constexpr int G = E::G, NT = E::NT;
  extern __shared__ __align__(16) unsigned char wstep_smem[];
  cx<T>* tws = reinterpret_cast<cx<T>*>(wstep_smem);
  cx<T>* buf = tws + S;
  if (skip && *skip) return;
  const int t = threadIdx.x;
  for (int i = t; i < S; i += NT) tws[i] = twg[i];
  cx<T> v[R];
  {
    const int y = t / G, g = t % G;
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cx<T>{T(0), T(0)};
    const cx<T>* src = wd_all + y * S + g;
#pragma unroll 4
    for (int d = 0; d < D; ++d) {  // d order per pixel; the R loads of a tile are independent
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] += src[static_cast<int64_t>(d) * S * S + G * m];
    }
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cx<T>{v[m].x / static_cast<T>(D), v[m].y / static_cast<T>(D)};
  }
  __syncthreads();
  E::forward(v, buf, tws, t);
  {
    const int x = t % S, c = t / S;
#pragma unroll
    for (int q = 0; q < R / G; ++q)
#pragma unroll
      for (int k1 = 0; k1 < G; ++k1) {
        const int ky = (c + G * q) + R * k1;
        const cx<T> val = v[q * G + k1] * scale;
        v[q * G + k1] = mask[ky * S + x] == T(0) ? cx<T>{T(0), T(0)} : val;
      }
  }
  __syncthreads();
  E::inverse(v, buf, tws, t);
  {
    const int y = t / G, g = t % G;
#pragma unroll
    for (int m = 0; m < R; ++m) w[y * S + g + G * m] = v[m] * scale;
  }
}

template <typename T, int S>
static cudaError_t launch_wstep_s(const cx<T>* wd_all, int D, const T* mask, const cx<T>* tw, T scale, cx<T>* w,
                                  const int* skip, cudaStream_t st) {
  using C = FrameCfg<T, S>;
  using E = Fft2<T, S, C::R>;
  const size_t smem = sizeof(cx<T>) * (S + static_cast<size_t>(E::TILE));
  auto kern = wstep_kernel<T, S, C::R>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<1, E::NT, smem, st>>>(wd_all, D, mask, tw, scale, w, skip);
  return cudaGetLastError();
}

// cudaErrorNotSupported: no single-CTA engine for this shape (complex128 128^2,
// G == 1 shapes) -- the caller runs the four-launch w-step instead.
template <>
cudaError_t launch_wstep<float>(int S, const cx<float>* wd_all, int D, const float* mask, const cx<float>* tw,
                                float scale, cx<float>* w, const int* skip, cudaStream_t st) {
  switch (S) {
    case 16: return launch_wstep_s<float, 16>(wd_all, D, mask, tw, scale, w, skip, st);
    case 32: return launch_wstep_s<float, 32>(wd_all, D, mask, tw, scale, w, skip, st);
    case 64: return launch_wstep_s<float, 64>(wd_all, D, mask, tw, scale, w, skip, st);
  }
  return cudaErrorNotSupported;
}
template <>
cudaError_t launch_wstep<double>(int S, const cx<double>* wd_all, int D, const double* mask, const cx<double>* tw,
                                 double scale, cx<double>* w, const int* skip, cudaStream_t st) {
  switch (S) {
    case 16: return launch_wstep_s<double, 16>(wd_all, D, mask, tw, scale, w, skip, st);
    case 32: return launch_wstep_s<double, 32>(wd_all, D, mask, tw, scale, w, skip, st);
    case 64: return launch_wstep_s<double, 64>(wd_all, D, mask, tw, scale, w, skip, st);
  }
  return cudaErrorNotSupported;
}

// ---------------------------------------------------------------------------
// block reduction of two doubles, fixed tree; result in thread 0.
__device__ __forceinline__ void block_sum2(double& a, double& b, double* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    sm[2 * w] = a;
    sm[2 * w + 1] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    a = 0.0;
    b = 0.0;
    for (int i = 0; i < nw; ++i) {
      a += sm[2 * i];
      b += sm[2 * i + 1];
    }
  }
}


// Streaming (evict-first) load of a complex value: back-projection tiles are
// read exactly once.
template <typename T>
struct Vec2;
template <>
struct Vec2<float> {
  using type = float2;
};
template <>
struct Vec2<double> {
  using type = double2;
};
template <typename T>
__device__ __forceinline__ cx<T>& operator+=(cx<T>& a, typename Vec2<T>::type b) {
  a.x += b.x;
  a.y += b.y;
  return a;
}

// Gather tile: TW = 32*VEC columns x 8*NROW rows per CTA of 256 threads; lane
// tx owns VEC adjacent columns (VEC = 2: one 16-byte load per row per frame).
// MODE is a template parameter: the accumulation loop then holds no branches,
// so the NROW x unroll predicated loads of one trip are all in flight before
// the first add waits on one of them.
//
// Resident CTAs asked of ptxas: 4 (64 registers) for the overlap-add modes and
// for the small-tile float blind update (config 3: 59 -> 54 us; the larger
// tiles and complex128 would spill at 64 registers).
template <typename T, int NROW, int VEC, int MODE>
constexpr int gather_min_ctas() {
  if (MODE == kGatherNonblind || MODE == kGatherAdjoint) return 4;
  if (MODE == kGatherBlind && sizeof(T) == 4 && NROW * VEC <= 2) return 4;
  return 1;
}
template <typename T, int NROW, int VEC, int MODE>
__global__ void __launch_bounds__(256, gather_min_ctas<T, NROW, VEC, MODE>()) gather_kernel(const GatherArgs<T> a) {
  constexpr int kMeta = 256;  // covering frames staged in shared memory per chunk
  __shared__ double sm[16];
  __shared__ int s_fr[kMeta], s_r0[kMeta], s_c0[kMeta], s_h[kMeta];
  __shared__ int64_t s_base[kMeta];
  if (a.stop_flag && *a.stop_flag) return;
  const int4 td = a.tiles[blockIdx.x];
  const int sub = td.x, tr0 = td.y, tc0 = td.z;
  // covering partial images: back-projection pieces, or frames
  const bool items = (MODE == kGatherNonblind || MODE == kGatherAdjoint) && a.tile_items != nullptr;
  const bool flat = a.mbeg != nullptr;  // flattened per-tile lists (one dependent load level)
  const int fb = flat ? a.mbeg[blockIdx.x] : items ? a.tile_item_beg[blockIdx.x] : td.w;
  const int fe = flat ? a.mbeg[blockIdx.x + 1] : items ? a.tile_item_beg[blockIdx.x + 1] : a.tiles[blockIdx.x + 1].w;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int H = a.sub_h[sub], W = a.sub_w[sub];
  const int c = tc0 + VEC * tx;  // first of this lane's VEC columns
  const int S = a.S;
  const int64_t SS = static_cast<int64_t>(S) * S;
  const int nf = fe - fb;

  cx<T> acc[NROW][VEC];
  T wacc[NROW][VEC];
  double dacc[NROW][VEC];
#pragma unroll
  for (int i = 0; i < NROW; ++i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      acc[i][v] = cx<T>{T(0), T(0)};
      wacc[i][v] = T(0);
      dacc[i][v] = 0.0;
    }

  // Ascending frame order per pixel (the reference's embed_add order).
  // Predicated loads keep the unrolled frames' loads in flight together;
  // adding an exact zero for uncovered pixels leaves the sum unchanged.  With
  // VEC = 2 a frame covers both columns or neither (host guarantees even
  // window columns, S even).
  for (int kb = 0; kb < nf; kb += kMeta) {
    const int nk = min(kMeta, nf - kb);
    if (kb > 0) __syncthreads();
    for (int k = threadIdx.x; k < nk; k += blockDim.x) {
      if (flat) {
        const int4 m = a.meta[fb + kb + k];
        s_r0[k] = m.x;
        s_c0[k] = m.y;
        s_h[k] = m.z;
        s_fr[k] = m.w;
        s_base[k] = a.mbase[fb + kb + k];
      } else if (items) {
        const int it = a.tile_items[fb + kb + k];
        s_fr[k] = -1;
        s_r0[k] = a.it_r[it];
        s_c0[k] = a.it_c[it];
        s_h[k] = a.it_h[it];
        s_base[k] = a.it_base[it];
      } else {
        const int fr = a.tile_frames[fb + kb + k];
        s_fr[k] = fr;
        s_r0[k] = a.fr_r[fr];
        s_c0[k] = a.fr_c[fr];
        s_h[k] = S;
        s_base[k] = fr * SS;
      }
    }
    __syncthreads();
    if constexpr (MODE == kGatherAdjoint || MODE == kGatherNonblind) {
      // plain overlap-add: U frames x NROW rows of loads issued as one batch,
      // then added in ascending frame order
      using V = typename Vec2<T>::type;
      constexpr int NV = (VEC == 2 && std::is_same_v<T, float>) ? 1 : VEC;  // loads per row
      // frames per batch: about 8 loads in flight per thread (64-register cap)
      constexpr int U = (NROW * NV >= 4) ? 2 : 8 / (NROW * NV);
      using L = std::conditional_t<NV == 1 && VEC == 2, float4, V>;
      auto load = [&](int k, int i, int v) -> L {
        const int cc = c - s_c0[k];
        const int rr = tr0 + ty + 8 * i - s_r0[k];
        const bool ok = static_cast<unsigned>(cc) < static_cast<unsigned>(S) &&
                        static_cast<unsigned>(rr) < static_cast<unsigned>(s_h[k]);
        L q{};
        if (ok) q = __ldcs(reinterpret_cast<const L*>(a.bp + s_base[k] + static_cast<int64_t>(rr) * S + cc + v));
        return q;
      };
      auto add = [&](int i, int v, const L& q) {
        if constexpr (NV == 1 && VEC == 2) {
          const float4 f = reinterpret_cast<const float4&>(q);
          acc[i][0].x += f.x;
          acc[i][0].y += f.y;
          acc[i][VEC - 1].x += f.z;
          acc[i][VEC - 1].y += f.w;
        } else {
          acc[i][v] += reinterpret_cast<const V&>(q);
        }
      };
      int k = 0;
#pragma unroll 1
      for (; k + U <= nk; k += U) {
        L q[U][NROW][NV];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < NROW; ++i)
#pragma unroll
            for (int v = 0; v < NV; ++v) q[u][i][v] = load(k + u, i, v);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < NROW; ++i)
#pragma unroll
            for (int v = 0; v < NV; ++v) add(i, v, q[u][i][v]);
      }
#pragma unroll 1
      for (; k < nk; ++k)
#pragma unroll
        for (int i = 0; i < NROW; ++i)
#pragma unroll
          for (int v = 0; v < NV; ++v) add(i, v, load(k, i, v));
    } else {
#pragma unroll 4
      for (int k = 0; k < nk; ++k) {
        const int fr = s_fr[k], r0 = s_r0[k], c0 = s_c0[k];
        const int cc = c - c0;
        const bool cv = static_cast<unsigned>(cc) < static_cast<unsigned>(S);
#pragma unroll
        for (int i = 0; i < NROW; ++i) {
          const int rr = tr0 + ty + 8 * i - r0;
          const bool ok = cv && static_cast<unsigned>(rr) < static_cast<unsigned>(S);
          const int64_t pix = static_cast<int64_t>(rr) * S + cc;
          if constexpr (MODE == kGatherDensity) {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
              if (ok) dacc[i][v] += static_cast<double>(norm2(a.probe[pix + v]));
          } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
              cx<T> w{T(0), T(0)}, q{T(0), T(0)};
              if (ok) {
                w = a.probe[static_cast<int64_t>(sub) * SS + pix + v];
                q = a.bp[fr * SS + pix + v];
              }
              acc[i][v] += mul_conj(q, w);
              wacc[i][v] += norm2(w);
            }
          }
        }
      }
    }
  }

  double diff = 0.0, nrm = 0.0;
  const int64_t base = a.sub_off[sub];
  constexpr bool update = MODE == kGatherNonblind || MODE == kGatherBlind;
  const cx<T>* u_in = a.u_in ? a.u_in : a.u;
  const cx<T>* lam_in = a.lam_in ? a.lam_in : a.lam;
  // pair sides meeting this tile: the flattened per-tile list (usually empty)
  // or all of the subdomain's
  int pb = 0, pe = 0;
  const int32_t* plist = nullptr;
  if constexpr (update) {
    if (a.tps_beg) {
      pb = a.tps_beg[blockIdx.x];
      pe = a.tps_beg[blockIdx.x + 1];
      plist = a.tps;
    } else {
      pb = a.sub_pbeg[sub];
      pe = a.sub_pbeg[sub + 1];
    }
  }
#pragma unroll
  for (int i = 0; i < NROW; ++i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const int r = tr0 + ty + 8 * i, cv = c + v;
      if (r >= H || cv >= W) continue;
      const int64_t pi = base + static_cast<int64_t>(r) * W + cv;
      if constexpr (MODE == kGatherAdjoint) {
        a.out[pi] = acc[i][v];
      } else if constexpr (MODE == kGatherDensity) {
        a.dens_out[pi] = dacc[i][v];
      } else {
        cx<T> num = acc[i][v] * a.eta;
        for (int q = pb; q < pe; ++q) {
          const PairSide p = a.ps[plist ? plist[q] : q];
          if (r < p.r0 || r >= p.r1 || cv < p.c0 || cv >= p.c1) continue;
          const int64_t o = static_cast<int64_t>(r - p.r0) * (p.c1 - p.c0) + (cv - p.c0);
          num += (a.v[p.v_off + o] - lam_in[p.lam_off + o]) * a.r;
        }
        const cx<T> uo = u_in[pi];
        cx<T> un;
        if constexpr (MODE == kGatherNonblind) {
          const T d = a.denom[pi];
          un = d < T(0) ? cx<T>{T(1), T(0)} : cx<T>{num.x / d, num.y / d};
        } else {
          const T rp = a.rpen[pi];
          const T dd = a.eta * wacc[i][v] + rp + a.gamma;
          const cx<T> nn = num + uo * a.gamma;
          un = rp < T(0) ? cx<T>{T(1), T(0)} : cx<T>{nn.x / dd, nn.y / dd};
        }
        for (int q = pb; q < pe; ++q) {
          const PairSide p = a.ps[plist ? plist[q] : q];
          if (r < p.r0 || r >= p.r1 || cv < p.c0 || cv >= p.c1) continue;
          const int64_t o = static_cast<int64_t>(r - p.r0) * (p.c1 - p.c0) + (cv - p.c0);
          a.lam[p.lam_off + o] = lam_in[p.lam_off + o] + (un - a.v[p.v_off + o]);
        }
        a.u[pi] = un;
        const double dx = static_cast<double>(un.x) - static_cast<double>(uo.x);
        const double dy = static_cast<double>(un.y) - static_cast<double>(uo.y);
        diff += dx * dx + dy * dy;
        nrm += static_cast<double>(un.x) * un.x + static_cast<double>(un.y) * un.y;
      }
    }
  if constexpr (update) {
    if (a.re_part) {
      block_sum2(diff, nrm, sm);
      if (threadIdx.x == 0) {
        a.re_part[2 * blockIdx.x] = diff;
        a.re_part[2 * blockIdx.x + 1] = nrm;
      }
    }
  }
}

template <typename T, int MODE>
static cudaError_t launch_gather_mode(const GatherArgs<T>& a, cudaStream_t st) {
  if (a.tile_w == 64) {
    if (a.tile_h != 32) return cudaErrorInvalidValue;
    gather_kernel<T, 4, 2, MODE><<<a.ntiles, 256, 0, st>>>(a);
  } else if (a.tile_h == 8) {
    gather_kernel<T, 1, 1, MODE><<<a.ntiles, 256, 0, st>>>(a);
  } else if (a.tile_h == 16) {
    gather_kernel<T, 2, 1, MODE><<<a.ntiles, 256, 0, st>>>(a);
  } else if (a.tile_h == 32) {
    gather_kernel<T, 4, 1, MODE><<<a.ntiles, 256, 0, st>>>(a);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_gather(const GatherArgs<T>& a, cudaStream_t st) {
  if (a.ntiles <= 0) return cudaSuccess;
  switch (a.mode) {
    case kGatherAdjoint: return launch_gather_mode<T, kGatherAdjoint>(a, st);
    case kGatherNonblind: return launch_gather_mode<T, kGatherNonblind>(a, st);
    case kGatherBlind: return launch_gather_mode<T, kGatherBlind>(a, st);
    case kGatherDensity: return launch_gather_mode<T, kGatherDensity>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void pack_kernel(const PairGeom* pairs, const cx<T>* u, const cx<T>* lam, cx<T>* s,
                            const int* stop_flag) {
  if (stop_flag && *stop_flag) return;
  const PairGeom p = pairs[blockIdx.y];
  const int n = p.h * p.w;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int rr = i / p.w, cc = i % p.w;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      if (p.u_off[side] < 0) continue;
      s[p.s_off + static_cast<int64_t>(side) * n + i] =
          u[p.u_off[side] + static_cast<int64_t>(rr) * p.u_pitch[side] + cc] + lam[p.lam_off[side] + i];
    }
  }
}

template <typename T>
__global__ void vstep_kernel(const PairGeom* pairs, const cx<T>* s, cx<T>* v, const int* stop_flag) {
  if (stop_flag && *stop_flag) return;
  const PairGeom p = pairs[blockIdx.y];
  const int n = p.h * p.w;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v[p.v_off + i] = (s[p.s_off + i] + s[p.s_off + n + i]) * T(0.5);
}

template <typename T>
cudaError_t launch_pack(const PairGeom* pairs, int npairs, int maxpix, const cx<T>* u, const cx<T>* lam,
                        cx<T>* s, const int* stop_flag, cudaStream_t st) {
  if (npairs <= 0) return cudaSuccess;
  dim3 grid(std::min((maxpix + 255) / 256, 1184), npairs);
  pack_kernel<T><<<grid, 256, 0, st>>>(pairs, u, lam, s, stop_flag);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_vstep(const PairGeom* pairs, int npairs, int maxpix, const cx<T>* s, cx<T>* v,
                         const int* stop_flag, cudaStream_t st) {
  if (npairs <= 0) return cudaSuccess;
  dim3 grid(std::min((maxpix + 255) / 256, 1184), npairs);
  vstep_kernel<T><<<grid, 256, 0, st>>>(pairs, s, v, stop_flag);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void fill_kernel(cx<T>* p, int64_t n, cx<T> value) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = value;
}
template <typename T>
cudaError_t launch_fill(cx<T>* p, int64_t n, cx<T> value, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  fill_kernel<T><<<grid, 256, 0, st>>>(p, n, value);
  return cudaGetLastError();
}

template <typename T>
__global__ void merge_kernel(const cx<T>* u, const int64_t* rect, const int64_t* off, int D, int64_t H, int64_t W,
                             cx<double>* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < H * W;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / W, c = i % W;
    double sx = 0.0, sy = 0.0, cnt = 0.0;
    for (int d = 0; d < D; ++d) {
      const int64_t* q = rect + 4 * d;
      if (r < q[0] || r >= q[1] || c < q[2] || c >= q[3]) continue;
      const cx<T> v = u[off[d] + (r - q[0]) * (q[3] - q[2]) + (c - q[2])];
      sx += static_cast<double>(v.x);
      sy += static_cast<double>(v.y);
      cnt += 1.0;
    }
    out[i] = cnt > 0.0 ? cx<double>{sx / cnt, sy / cnt} : cx<double>{1.0, 0.0};
  }
}
template <typename T>
cudaError_t launch_merge(const cx<T>* u, const int64_t* sub_rect, const int64_t* sub_off, int D, int64_t H, int64_t W,
                         cx<double>* out, cudaStream_t st) {
  const int64_t n = H * W;
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  merge_kernel<T><<<grid, 256, 0, st>>>(u, sub_rect, sub_off, D, H, W, out);
  return cudaGetLastError();
}
template cudaError_t launch_merge<float>(const cx<float>*, const int64_t*, const int64_t*, int, int64_t, int64_t,
                                         cx<double>*, cudaStream_t);
template cudaError_t launch_merge<double>(const cx<double>*, const int64_t*, const int64_t*, int, int64_t, int64_t,
                                          cx<double>*, cudaStream_t);

// pin = (no window covers the pixel) | user mask  -- from the gather tiles
__global__ void pins_kernel(const int4* tiles, int tile_h, int tile_w, const int32_t* tile_frames, const int32_t* fr_r,
                            const int32_t* fr_c, int S, const int64_t* sub_off, const int32_t* sub_h,
                            const int32_t* sub_w, const uint8_t* user_pin, uint8_t* pin) {
  const int4 td = tiles[blockIdx.x];
  const int sub = td.x, fb = td.w, fe = tiles[blockIdx.x + 1].w;
  const int H = sub_h[sub], W = sub_w[sub];
  for (int e = threadIdx.x; e < tile_h * tile_w; e += blockDim.x) {
    const int r = td.y + e / tile_w, c = td.z + e % tile_w;
    if (r >= H || c >= W) continue;
    bool covered = false;
    for (int k = fb; k < fe && !covered; ++k) {
      const int fr = tile_frames[k];
      covered = r >= fr_r[fr] && r < fr_r[fr] + S && c >= fr_c[fr] && c < fr_c[fr] + S;
    }
    const int64_t i = sub_off[sub] + static_cast<int64_t>(r) * W + c;
    pin[i] = !covered || (user_pin && user_pin[i]);
  }
}
cudaError_t launch_pins(const int4* tiles, int ntiles, int tile_h, int tile_w, const int32_t* tile_frames,
                        const int32_t* fr_r, const int32_t* fr_c, int S, const int64_t* sub_off, const int32_t* sub_h,
                        const int32_t* sub_w, const uint8_t* user_pin, uint8_t* pin, cudaStream_t st) {
  if (ntiles <= 0) return cudaSuccess;
  pins_kernel<<<ntiles, 256, 0, st>>>(tiles, tile_h, tile_w, tile_frames, fr_r, fr_c, S, sub_off, sub_h, sub_w,
                                      user_pin, pin);
  return cudaGetLastError();
}

__global__ void widen_cx_kernel(const cx<float>* in, cx<double>* out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = cx<double>{static_cast<double>(in[i].x), static_cast<double>(in[i].y)};
}
cudaError_t launch_widen_cx(const cx<float>* in, cx<double>* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  widen_cx_kernel<<<grid, 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
__global__ void segsum_kernel(const double* in, int stride, int comp, const int64_t* beg, const int* map,
                              double* out, const int* skip) {
  __shared__ double sm[16];
  if (skip && *skip) return;
  const int64_t b = beg[blockIdx.x], e = beg[blockIdx.x + 1];
  double acc = 0.0, dummy = 0.0;
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) acc += in[i * stride + comp];
  block_sum2(acc, dummy, sm);
  if (threadIdx.x == 0) out[map ? map[blockIdx.x] : blockIdx.x] = acc;
}
cudaError_t launch_segsum(const double* in, int stride, int comp, const int64_t* beg, int nseg, const int* map,
                          double* out, const int* skip, cudaStream_t st) {
  if (nseg <= 0) return cudaSuccess;
  segsum_kernel<<<nseg, 256, 0, st>>>(in, stride, comp, beg, map, out, skip);
  return cudaGetLastError();
}

template <typename T>
__global__ void frame_sums_kernel(const T* amp, int64_t per, double* out) {
  __shared__ double sm[16];
  const T* p = amp + blockIdx.x * per;
  double acc = 0.0, dummy = 0.0;
  for (int64_t i = threadIdx.x; i < per; i += blockDim.x) acc += static_cast<double>(p[i]);
  block_sum2(acc, dummy, sm);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}
template <typename T>
cudaError_t launch_frame_sums(const T* amp, int64_t nfr, int64_t per, double* out, cudaStream_t st) {
  if (nfr <= 0) return cudaSuccess;
  frame_sums_kernel<T><<<static_cast<unsigned>(nfr), 256, 0, st>>>(amp, per, out);
  return cudaGetLastError();
}

// Augmented Lagrangian terms (metrics.cpp:73-101), fp64 accumulation.
// Frame term per frame j: sum_i g_eps(z_i; b_i) + eta (Re(conj(G_i)(au_i - z_i)) + |au_i - z_i|^2 / 2),
// g_eps = stagm::pixel_value (stagm.cpp:29-35) with b = amp^2.
template <typename T>
__global__ void lagrangian_frames_kernel(const cx<T>* au, const cx<T>* z, const cx<T>* gamma, const T* amp,
                                         int64_t per, double eps, double eta, double* out) {
  __shared__ double sm[16];
  const int64_t base = blockIdx.x * per;
  double acc = 0.0, dummy = 0.0;
  for (int64_t i = threadIdx.x; i < per; i += blockDim.x) {
    const cx<T> zi = z[base + i], ai = au[base + i], gi = gamma[base + i];
    const double zx = zi.x, zy = zi.y;
    const double ax = hypot(zx, zy), rb = static_cast<double>(amp[base + i]), b = rb * rb;
    double g;
    if (ax < eps * rb) {
      g = 0.5 * (1.0 - eps) * (b - ax * ax / eps);
    } else {
      const double d = ax - rb;
      g = 0.5 * d * d;
    }
    const double rx = static_cast<double>(ai.x) - zx, ry = static_cast<double>(ai.y) - zy;
    acc += g + eta * (static_cast<double>(gi.x) * rx + static_cast<double>(gi.y) * ry + 0.5 * (rx * rx + ry * ry));
  }
  block_sum2(acc, dummy, sm);
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}
template <typename T>
cudaError_t launch_lagrangian_frames(const cx<T>* au, const cx<T>* z, const cx<T>* gamma, const T* amp, int64_t nfr,
                                     int64_t per, double eps, double eta, double* out, cudaStream_t st) {
  if (nfr <= 0) return cudaSuccess;
  lagrangian_frames_kernel<T><<<static_cast<unsigned>(nfr), 256, 0, st>>>(au, z, gamma, amp, per, eps, eta, out);
  return cudaGetLastError();
}

// Overlap term per (local pair, side): r (Re(conj(Lambda_s)(pi u_s - v)) + |pi u_s - v|^2 / 2);
// out[2 lp + side] (0 where the side's subdomain lives on another rank).
template <typename T>
__global__ void lagrangian_pairs_kernel(const PairGeom* pairs, const cx<T>* u, const cx<T>* v, const cx<T>* lam,
                                        double r, double* out) {
  __shared__ double sm[16];
  const PairGeom p = pairs[blockIdx.x];
  const int side = blockIdx.y;
  double acc = 0.0, dummy = 0.0;
  if (p.u_off[side] >= 0) {
    const int64_t n = static_cast<int64_t>(p.h) * p.w;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const int64_t rr = i / p.w, cc = i % p.w;
      const cx<T> ui = u[p.u_off[side] + rr * p.u_pitch[side] + cc], vi = v[p.v_off + i],
                  li = lam[p.lam_off[side] + i];
      const double rx = static_cast<double>(ui.x) - static_cast<double>(vi.x);
      const double ry = static_cast<double>(ui.y) - static_cast<double>(vi.y);
      acc += r * (static_cast<double>(li.x) * rx + static_cast<double>(li.y) * ry + 0.5 * (rx * rx + ry * ry));
    }
  }
  block_sum2(acc, dummy, sm);
  if (threadIdx.x == 0) out[2 * blockIdx.x + side] = acc;
}
template <typename T>
cudaError_t launch_lagrangian_pairs(const PairGeom* pairs, int npairs, const cx<T>* u, const cx<T>* v,
                                    const cx<T>* lam, double r, double* out, cudaStream_t st) {
  if (npairs <= 0) return cudaSuccess;
  lagrangian_pairs_kernel<T><<<dim3(npairs, 2), 256, 0, st>>>(pairs, u, v, lam, r, out);
  return cudaGetLastError();
}
template cudaError_t launch_lagrangian_frames<float>(const cx<float>*, const cx<float>*, const cx<float>*,
                                                     const float*, int64_t, int64_t, double, double, double*,
                                                     cudaStream_t);
template cudaError_t launch_lagrangian_frames<double>(const cx<double>*, const cx<double>*, const cx<double>*,
                                                      const double*, int64_t, int64_t, double, double, double*,
                                                      cudaStream_t);
template cudaError_t launch_lagrangian_pairs<float>(const PairGeom*, int, const cx<float>*, const cx<float>*,
                                                    const cx<float>*, double, double*, cudaStream_t);
template cudaError_t launch_lagrangian_pairs<double>(const PairGeom*, int, const cx<double>*, const cx<double>*,
                                                     const cx<double>*, double, double*, cudaStream_t);

template <typename T>
__global__ void convert_amp_kernel(const void* src, int kind, T* amp, int64_t n, unsigned long long* neg) {
  unsigned long long bad = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = kind == 1 ? static_cast<double>(static_cast<const float*>(src)[i]) : static_cast<const double*>(src)[i];
    if (v < 0.0) {
      ++bad;
      v = 0.0;
    }
    amp[i] = static_cast<T>(kind == 0 ? sqrt(v) : v);
  }
  if (bad && neg) atomicAdd(neg, bad);
}
template <typename T>
cudaError_t launch_convert_amp(const void* src, int kind, T* amp, int64_t n, unsigned long long* neg,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  convert_amp_kernel<T><<<grid, 256, 0, st>>>(src, kind, amp, n, neg);
  return cudaGetLastError();
}

// float64 intensities of global frames [g0, g0+count) -> T amplitudes at
// their local positions (glob2loc: -1 = owned by another rank).
template <typename T>
__global__ void scatter_amp_kernel(const double* src, int64_t g0, int64_t count, int64_t per, const int32_t* glob2loc,
                                   T* amp, unsigned long long* neg) {
  unsigned long long bad = 0;
  const int64_t n = count * per;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t f = i / per;
    const int32_t loc = glob2loc[g0 + f];
    if (loc < 0) continue;
    double v = src[i];
    if (v < 0.0) {
      ++bad;
      v = 0.0;
    }
    amp[static_cast<int64_t>(loc) * per + (i - f * per)] = static_cast<T>(sqrt(v));
  }
  if (bad && neg) atomicAdd(neg, bad);
}
template <typename T>
cudaError_t launch_scatter_amp(const double* src, int64_t g0, int64_t count, int64_t per, const int32_t* glob2loc,
                               T* amp, unsigned long long* neg, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((count * per + 255) / 256, 148 * 16));
  scatter_amp_kernel<T><<<grid, 256, 0, st>>>(src, g0, count, per, glob2loc, amp, neg);
  return cudaGetLastError();
}
template cudaError_t launch_scatter_amp<float>(const double*, int64_t, int64_t, int64_t, const int32_t*, float*,
                                               unsigned long long*, cudaStream_t);
template cudaError_t launch_scatter_amp<double>(const double*, int64_t, int64_t, int64_t, const int32_t*, double*,
                                                unsigned long long*, cudaStream_t);

template <typename T>
__global__ void denom_sub_kernel(const double* dens, const uint8_t* pin, const PairSide* ps, int nps, int H, int W,
                                 T eta, T r, T* denom, unsigned long long* bad, int blind) {
  const int64_t n = static_cast<int64_t>(H) * W;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int rr = static_cast<int>(i / W), cc = static_cast<int>(i % W);
    double d = blind ? 0.0 : static_cast<double>(eta) * dens[i];
    for (int k = 0; k < nps; ++k) {
      const PairSide p = ps[k];
      if (rr >= p.r0 && rr < p.r1 && cc >= p.c0 && cc < p.c1) d += static_cast<double>(r);
    }
    if (!blind && !pin[i] && dens[i] <= 0.0) atomicAdd(bad, 1ull);
    denom[i] = pin[i] ? T(-1) : static_cast<T>(d);
  }
}
template <typename T>
cudaError_t launch_denom_sub(const double* dens, const uint8_t* pin, const PairSide* ps, int nps, int H, int W,
                             T eta, T r, T* denom, unsigned long long* bad, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(H) * W;
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  denom_sub_kernel<T><<<grid, 256, 0, st>>>(dens, pin, ps, nps, H, W, eta, r, denom, bad, 0);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_rpen_sub(const uint8_t* pin, const PairSide* ps, int nps, int H, int W, T r, T* rpen,
                            cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(H) * W;
  if (n <= 0) return cudaSuccess;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  denom_sub_kernel<T><<<grid, 256, 0, st>>>(nullptr, pin, ps, nps, H, W, T(0), r, rpen, nullptr, 1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// iteration control: stop rules of run() (solver.cpp:225-262) on the device
// Switches of the NEXT iteration's passes from the run state.  Runs at the end
// of every RE finalize step (so an iteration needs no launch of its own for
// it) and as gate_kernel before the trailing R-factor pass.
__device__ __forceinline__ void gate_body(RunCtl* c) {
  c->skipA = !(c->stop == 0 || (c->stop == c->iter && !c->done));
  c->skipB = c->stop != 0;
  c->skipC = c->stop != 0;
}
__global__ void gate_kernel(RunCtl* c) { gate_body(c); }
__device__ __forceinline__ void rf_finalize_body(RunCtl* c, const double* rf_sub, int D, double* rec) {
  if (c->skipA) return;
  double s = 0.0;
  for (int d = 0; d < D; ++d) s += rf_sub[d];
  const double rf = s / c->l1;
  const int n = c->iter;
  if (n >= 1) {
    rec[2 * ((n - 1) % c->rec_cap)] = rf;
    if (c->stop == n) {
      c->done = 1;
    } else if (!isfinite(rf)) {
      c->diverged = n;
      c->stop = n;
      c->done = 1;
    } else if (c->rule == 0 && rf <= c->tol_rf) {
      c->stop = n;
      c->done = 1;
    }
  }
  c->skipB = c->stop != 0;
}
__global__ void rf_finalize_kernel(RunCtl* c, const double* rf_sub, int D, double* rec) {
  rf_finalize_body(c, rf_sub, D, rec);
}
__device__ __forceinline__ void re_finalize_body(RunCtl* c, const double* diff, const double* norm, int D, double* rec) {
  if (c->skipB) {
    gate_body(c);
    return;
  }
  double re = 0.0;
  bool finite = true;
  for (int d = 0; d < D; ++d) {
    const double e = sqrt(diff[d]) / sqrt(norm[d]);
    if (!isfinite(e)) finite = false;
    re = e > re ? e : re;
  }
  const int n = c->iter + 1;
  rec[2 * ((n - 1) % c->rec_cap) + 1] = finite ? re : NAN;
  c->iter = n;
  if (!finite) {
    c->diverged = n;
    c->stop = n;
  } else if (c->rule == 1 && re <= c->tol_re) {
    c->stop = n;
  } else if (n >= c->max_iters) {
    c->stop = n;
  }
  gate_body(c);
}
__global__ void re_finalize_kernel(RunCtl* c, const double* diff, const double* norm, int D, double* rec) {
  re_finalize_body(c, diff, norm, D, rec);
}

// Segment sums and the finalize step in ONE launch (single-rank solvers: no
// all-reduce sits between them): block b sums segment b exactly as
// segsum_kernel does (same strided accumulation and tree, so the sums are
// bit-identical to the two-launch path of multi-rank solvers), and the block
// that finishes last -- a device counter it resets -- runs the finalize body
// on the D sums.  NCOMP = 1: R-factor numerators; NCOMP = 2: RE (diff, norm).
constexpr int kFusedMaxD = 64;
template <int NCOMP>
__global__ void segsum_finalize_kernel(const double* in, const int64_t* beg, const int* map, double* out0, double* out1,
                                       const int* skip, unsigned* counter, RunCtl* c, int D, double* rec) {
  __shared__ double sm[16];
  __shared__ double fin[2 * kFusedMaxD];
  __shared__ int last;
  if (skip && *skip) {  // pass disabled: only the RE step's closing gate remains to do
    if (NCOMP == 2 && blockIdx.x == 0 && threadIdx.x == 0) gate_body(c);
    return;
  }
  const int64_t b = beg[blockIdx.x], e = beg[blockIdx.x + 1];
  double acc0 = 0.0, acc1 = 0.0;
  // (the two components of block_sum2 are summed independently, each with
  // the per-thread order and tree segsum_kernel gives it)
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    acc0 += in[NCOMP * i];
    if constexpr (NCOMP == 2) acc1 += in[2 * i + 1];
  }
  block_sum2(acc0, acc1, sm);
  if (threadIdx.x == 0) {
    const int o = map ? map[blockIdx.x] : blockIdx.x;
    out0[o] = acc0;
    if constexpr (NCOMP == 2) out1[o] = acc1;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < D) {
    fin[threadIdx.x] = __ldcg(out0 + threadIdx.x);
    if constexpr (NCOMP == 2) fin[kFusedMaxD + threadIdx.x] = __ldcg(out1 + threadIdx.x);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *counter = 0u;
    if constexpr (NCOMP == 1) rf_finalize_body(c, fin, D, rec);
    else re_finalize_body(c, fin, fin + kFusedMaxD, D, rec);
  }
}
cudaError_t launch_segsum_finalize(int ncomp, const double* in, const int64_t* beg, int nseg, const int* map,
                                   double* out0, double* out1, const int* skip, unsigned* counter, RunCtl* c, int D,
                                   double* rec, cudaStream_t st) {
  if (nseg <= 0 || D > kFusedMaxD || D > 256) return cudaErrorInvalidValue;
  if (ncomp == 1) segsum_finalize_kernel<1><<<nseg, 256, 0, st>>>(in, beg, map, out0, out1, skip, counter, c, D, rec);
  else segsum_finalize_kernel<2><<<nseg, 256, 0, st>>>(in, beg, map, out0, out1, skip, counter, c, D, rec);
  return cudaGetLastError();
}
int fused_finalize_max_subdomains() { return kFusedMaxD; }
cudaError_t launch_gate(RunCtl* c, cudaStream_t st) {
  gate_kernel<<<1, 1, 0, st>>>(c);
  return cudaGetLastError();
}
cudaError_t launch_rf_finalize(RunCtl* c, const double* rf_sub, int D, double* rec, cudaStream_t st) {
  rf_finalize_kernel<<<1, 1, 0, st>>>(c, rf_sub, D, rec);
  return cudaGetLastError();
}
cudaError_t launch_re_finalize(RunCtl* c, const double* diff, const double* norm, int D, double* rec,
                               cudaStream_t st) {
  re_finalize_kernel<<<1, 1, 0, st>>>(c, diff, norm, D, rec);
  return cudaGetLastError();
}

// explicit instantiations
template cudaError_t launch_gather<float>(const GatherArgs<float>&, cudaStream_t);
template cudaError_t launch_gather<double>(const GatherArgs<double>&, cudaStream_t);
template cudaError_t launch_pack<float>(const PairGeom*, int, int, const cx<float>*, const cx<float>*, cx<float>*,
                                        const int*, cudaStream_t);
template cudaError_t launch_pack<double>(const PairGeom*, int, int, const cx<double>*, const cx<double>*,
                                         cx<double>*, const int*, cudaStream_t);
template cudaError_t launch_vstep<float>(const PairGeom*, int, int, const cx<float>*, cx<float>*, const int*,
                                         cudaStream_t);
template cudaError_t launch_vstep<double>(const PairGeom*, int, int, const cx<double>*, cx<double>*, const int*,
                                          cudaStream_t);
template cudaError_t launch_fill<float>(cx<float>*, int64_t, cx<float>, cudaStream_t);
template cudaError_t launch_fill<double>(cx<double>*, int64_t, cx<double>, cudaStream_t);
template cudaError_t launch_frame_sums<float>(const float*, int64_t, int64_t, double*, cudaStream_t);
template cudaError_t launch_frame_sums<double>(const double*, int64_t, int64_t, double*, cudaStream_t);
template cudaError_t launch_convert_amp<float>(const void*, int, float*, int64_t, unsigned long long*, cudaStream_t);
template cudaError_t launch_convert_amp<double>(const void*, int, double*, int64_t, unsigned long long*,
                                                cudaStream_t);
template cudaError_t launch_denom_sub<float>(const double*, const uint8_t*, const PairSide*, int, int, int, float,
                                             float, float*, unsigned long long*, cudaStream_t);
template cudaError_t launch_denom_sub<double>(const double*, const uint8_t*, const PairSide*, int, int, int, double,
                                              double, double*, unsigned long long*, cudaStream_t);
template cudaError_t launch_rpen_sub<float>(const uint8_t*, const PairSide*, int, int, int, float, float*,
                                            cudaStream_t);
template cudaError_t launch_rpen_sub<double>(const uint8_t*, const PairSide*, int, int, int, double, double*,
                                             cudaStream_t);

}  // namespace pdd
