// Per-frame fused kernel: the data-parallel heart of the OD²P iteration.
//
// One frame per Fft2<T,S,R>::NT threads, FPB frames per CTA.  Modes:
//   FWD    : patch gather S_j u (field.cpp:5-16) x probe -> FFT2 -> A u
//            (forward.cpp:28-41); optional outputs: frames, intensities
//            (forward.cpp:95-106), per-frame R-factor partials
//            sum | |A u| - sqrt f | (solver.cpp:207-214).
//   ADJ    : frames -> IFFT2 -> x conj(probe) (forward.cpp:43-54 minus the
//            overlap-add, which the deterministic gather kernel does).
//   SWEEP  : the nonblind z/Gamma step (solver.cpp:125-139) fused between the
//            two transforms: y = Gamma + A u, z = prox(y) (stagm.cpp:45-73),
//            Gamma' = y - z, then resid = z - Gamma' -> IFFT2 -> x conj(P)
//            (solver.cpp:157-164).  R-factor partials of u^n ride along.
//   BLIND  : like SWEEP with the subdomain probe copy W_d (blind.cpp:224-242);
//            additionally keeps q_j = IFFT2(resid) (the probe update needs it
//            before conj(W^{n+1}) is known) and the shared-probe R-factor of
//            u^n via a second forward transform (blind.cpp:320-332).
#pragma once

#include "fft.cuh"

namespace pdd {

enum FrameMode : int { kFwd = 1, kAdj = 2, kSweep = 3, kBlind = 4 };

// One position of the streamed sweep schedule with everything the kernel needs
// about its frame (32 bytes: staged in shared memory a frame ahead, so no
// dependent global load sits behind a CTA barrier).
struct alignas(16) PosRec {
  int32_t f;        // frame index
  int32_t lo;       // rows y < lo are final after this frame (layout.hpp pc_pos.y)
  int32_t nw_rot;   // newfrom | rot << 16 (pc_pos.z, .w)
  int32_t pitch;    // image row pitch of the frame's subdomain (elements)
  int64_t ofs;      // element offset of the frame's window row 0 in the partials (pc_ofs)
  int64_t woff;     // element offset of the window corner in the image buffer (fr_off)
};

template <typename T>
struct FrameArgs {
  int nframes = 0;
  const cx<T>* probe = nullptr;       // [S][S] (or per-frame probes via probe_idx)
  const int32_t* probe_idx = nullptr; // optional [nframes] -> index into probe tiles (blind: subdomain copy)
  const cx<T>* probe2 = nullptr;      // blind: shared probe w for the R-factor transform
  const cx<T>* tw = nullptr;          // [S] W_S^k forward twiddles
  const cx<T>* img = nullptr;         // concatenated images
  const int64_t* off = nullptr;       // [nframes] element offset of window corner
  const int32_t* pitch = nullptr;     // [nframes] image row pitch (elements)
  const cx<T>* frames_in = nullptr;   // ADJ input [nframes][S][S]
  cx<T>* frames_out = nullptr;        // FWD output A u
  T* inten_out = nullptr;             // FWD |A u|^2
  const T* amp = nullptr;             // sqrt(f)  [nframes][S][S]
  const cx<T>* gamma_in = nullptr;
  cx<T>* gamma_out = nullptr;
  cx<T>* z_out = nullptr;             // diagnostic z (SWEEP/BLIND)
  cx<T>* bp_out = nullptr;            // conj(P) . IFFT(.)  (ADJ/SWEEP) or q_j = IFFT(resid) (BLIND)
  double* rf_part = nullptr;          // [nframes]
  const int* stop_flag = nullptr;     // if non-null and *stop_flag != 0: skip (device-side early stop)
  T lam = T(0), eps = T(0.5);
  int fast_prox = 1;
  T scale = T(1);                     // 1/S (unitary normalisation per transform)
  unsigned long long* phase_cycles = nullptr;  // PDD_PHASE_TIMING builds: per-phase SM cycles
  int rows_al16 = 0;                  // every window row starts 16-byte aligned (streamed kernel: TMA rows)
  int bp_raw = 0;                     // SWEEP: bp_out = IFFT(.) without conj(probe) (the blind q_j)
  // Streamed sweep schedule (required by the streamed SWEEP kernel; layout.hpp):
  // CTA b of ncta runs positions [cta_beg[b], cta_beg[b+1]), frames in
  // back-projection piece order.  Unchained layouts: one piece per frame,
  // written whole to bp_out + f * S * S.
  const int32_t* cta_beg = nullptr;   // [ncta+1]
  int ncta = 0;
  const int4* pc_pos = nullptr;       // [nframes] {frame, lo, newfrom, rot}
  const int64_t* pc_ofs = nullptr;    // [nframes]
  const PosRec* pc_rec = nullptr;     // [nframes] the same schedule as records (streamed SWEEP reads these)
  int64_t img_elems = 0;              // PDD_BOUNDS builds: image buffer size (elements)
  cx<T>* scratch = nullptr;           // global transpose tiles of the streamed kernel when its
                                      // tile exceeds shared memory (stream_scratch_bytes)
};

// ST-AGM per-pixel prox, stagm.cpp:45-73.  amp = sqrt(b).  The fast form is
// exact whenever lam <= (1-eps)/eps: then the outer candidate never falls
// below eps*sqrt(b) and neither the origin nor the inner point can win
// (SURVEY.md sec. 0 item 3); the host selects it from (lam, eps).
template <typename T>
__device__ __forceinline__ T mag_obj(T m, T absy, T b, T root_b, T lam, T eps) {
  T g;
  if (m < eps * root_b) {
    g = T(0.5) * (T(1) - eps) * (b - m * m / eps);
  } else {
    const T d = m - root_b;
    g = T(0.5) * d * d;
  }
  const T e = m - absy;
  return g + T(0.5) * lam * e * e;
}

template <typename T>
__device__ __forceinline__ cx<T> stagm_prox(cx<T> y, T amp, T lam, T eps, bool fast) {
  const T absy = sqrt(norm2(y));
  T m = (amp + lam * absy) / (T(1) + lam);
  if (!fast) {
    const T b = amp * amp, inner_edge = eps * amp;
    if (m < inner_edge) m = inner_edge;
    T best = mag_obj(m, absy, b, amp, lam, eps);
    const T o0 = mag_obj(T(0), absy, b, amp, lam, eps);
    if (o0 < best) {
      best = o0;
      m = T(0);
    }
    const T ic = lam - (T(1) - eps) / eps;
    if (ic > T(0)) {
      const T mi = lam * absy / ic;
      if (mi < inner_edge) {
        const T oi = mag_obj(mi, absy, b, amp, lam, eps);
        if (oi < best) m = mi;
      }
    }
  }
  if (absy > T(0)) return cx<T>{y.x / absy * m, y.y / absy * m};
  return cx<T>{m, T(0)};
}

// float32 fast form of the prox (valid when lam <= (1-eps)/eps, see above):
// one rsqrt replaces sqrt + two IEEE divisions; |y| and the scale factor carry
// <= 2 ulp extra error (well inside the 1e-5 float32 parity bound).
// Hardware rsqrt (<= 2 ulp): a Newton refinement was measured to change
// nothing in the parity errors (Gamma's float32 error is set by cancellation
// in y - prox(y)) while costing 5% of the frame kernel.
__device__ __forceinline__ float rsqrt_ftz(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// The argument is clamped to FLT_MIN so the flush-to-zero rsqrt (one MUFU, no
// denormal rescaling branch) stays finite: n2 = 0 gives |y| = 0 and the
// reference's (m, 0) exactly; 0 < n2 < FLT_MIN (|y| < 1.1e-19, far below any
// float32 Fourier coefficient of a frame) is treated as n2 = FLT_MIN.
__device__ __forceinline__ cx<float> prox_fast_f32(cx<float> y, float amp, float lam, float inv1pl) {
  const float n2 = norm2(y);
  const float ri = rsqrt_ftz(fmaxf(n2, 1.17549435e-38f));
  const float m = (amp + lam * (n2 * ri)) * inv1pl;
  const cx<float> z = y * (m * ri);
  return n2 > 0.f ? z : cx<float>{m, 0.f};
}
__device__ __forceinline__ float abs_fast_f32(cx<float> a) {
  const float n2 = norm2(a);
  return n2 * rsqrt_ftz(fmaxf(n2, 1.17549435e-38f));
}

// Sum a per-thread double over the NT threads of one frame slot; result valid
// in the slot's thread 0.  Fixed shuffle tree => deterministic.
template <int NT>
__device__ __forceinline__ double slot_sum(double v, double* red, int t, int slot) {
  if constexpr (NT <= 32) {
#pragma unroll
    for (int o = NT / 2; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, NT);
    return v;
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    constexpr int NW = NT / 32;
    if ((t & 31) == 0) red[slot * NW + t / 32] = v;
    __syncthreads();
    double s = 0.0;
    if (t == 0)
      for (int w = 0; w < NW; ++w) s += red[slot * NW + w];
    return s;
  }
}

template <typename T, int S, int R, int FPB, int MODE>
__global__ void __launch_bounds__(Fft2<T, S, R>::NT* FPB)
    frame_kernel(const FrameArgs<T> a) {
  using E = Fft2<T, S, R>;
  constexpr int G = E::G, NT = E::NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cx<T>* tws = reinterpret_cast<cx<T>*>(smem_raw);
  cx<T>* bufs = tws + S;
  double* red = reinterpret_cast<double*>(bufs + FPB * E::TILE);

  if (a.stop_flag && *a.stop_flag) return;  // uniform across the grid

  const int tid = threadIdx.x;
  const int slot = tid / NT, t = tid % NT;
  cx<T>* buf = bufs + slot * E::TILE;
  for (int i = tid; i < S; i += NT * FPB) tws[i] = a.tw[i];
  const int f = blockIdx.x * FPB + slot;
  const bool live = f < a.nframes;
  __syncthreads();

  cx<T> v[R];
  const int y = t / G, g = t % G;      // row layout
  const int x = t % S, c = t / S;      // Fourier layout
  const int64_t fbase = static_cast<int64_t>(f) * S * S;

  const cx<T>* probe = a.probe;
  if (a.probe_idx && live) probe = a.probe + static_cast<int64_t>(a.probe_idx[f]) * S * S;

  double rf = 0.0;
  if constexpr (MODE != kAdj) {
    cx<T> patch[MODE == kBlind ? R : 1];
    if (live) {
      const cx<T>* src = a.img + a.off[f] + static_cast<int64_t>(y) * a.pitch[f] + g;
      const cx<T>* pr = probe + y * S + g;
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const cx<T> u = src[G * m];
        if constexpr (MODE == kBlind) patch[m] = u;
        v[m] = u * pr[G * m];
      }
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = cx<T>{T(0), T(0)};
    }

    if constexpr (MODE == kBlind) {
      // Shared-probe forward transform for the lagged R-factor of u^n.
      cx<T> w2[R];
      const cx<T>* pr2 = a.probe2 + y * S + g;
#pragma unroll
      for (int m = 0; m < R; ++m) w2[m] = patch[m] * pr2[G * m];
      E::forward(w2, buf, tws, t);
      if (live && a.rf_part) {
        T acc = T(0);
#pragma unroll
        for (int q = 0; q < R / G; ++q)
#pragma unroll
          for (int k1 = 0; k1 < G; ++k1) {
            const int ky = c + G * q + R * k1;
            const cx<T> au = w2[q * G + k1] * a.scale;
            acc += fabs(sqrt(norm2(au)) - a.amp[fbase + ky * S + x]);
          }
        rf = static_cast<double>(acc);
      }
      __syncthreads();
    }

    E::forward(v, buf, tws, t);

    if (live) {
      T acc = T(0);
#pragma unroll
      for (int q = 0; q < R / G; ++q) {
        // Compiler fence per chunk of G elements: bounds the number of
        // Gamma/amp loads in flight (and so live registers) without giving
        // up the G-wide memory-level parallelism.
        if constexpr (MODE != kFwd) asm volatile("" ::: "memory");
#pragma unroll
        for (int k1 = 0; k1 < G; ++k1) {
          const int ky = c + G * q + R * k1;
          const int64_t idx = fbase + ky * S + x;
          const cx<T> au = v[q * G + k1] * a.scale;
          if constexpr (MODE == kFwd) {
            if (a.frames_out) a.frames_out[idx] = au;
            if (a.inten_out) a.inten_out[idx] = norm2(au);
            if (a.rf_part) acc += fabs(sqrt(norm2(au)) - a.amp[idx]);
          } else {
            const T am = a.amp[idx];
            if constexpr (MODE == kSweep) acc += fabs(sqrt(norm2(au)) - am);
            const cx<T> yv = a.gamma_in[idx] + au;
            const cx<T> z = stagm_prox(yv, am, a.lam, a.eps, a.fast_prox != 0);
            const cx<T> gn = yv - z;
            a.gamma_out[idx] = gn;
            if (a.z_out) a.z_out[idx] = z;
            v[q * G + k1] = z - gn;
          }
        }
      }
      if constexpr (MODE != kBlind) rf = static_cast<double>(acc);
    } else if constexpr (MODE != kFwd) {
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = cx<T>{T(0), T(0)};
    }
  } else {
    if (live) {
#pragma unroll
      for (int q = 0; q < R / G; ++q)
#pragma unroll
        for (int k1 = 0; k1 < G; ++k1) {
          const int ky = c + G * q + R * k1;
          v[q * G + k1] = a.frames_in[fbase + ky * S + x];
        }
    } else {
#pragma unroll
      for (int m = 0; m < R; ++m) v[m] = cx<T>{T(0), T(0)};
    }
  }

  if constexpr (MODE != kFwd) {
    E::inverse(v, buf, tws, t);
    if (live) {
      cx<T>* dst = a.bp_out + fbase + y * S + g;
      const cx<T>* pr = probe + y * S + g;
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const cx<T> q = v[m] * a.scale;
        // BLIND keeps q_j itself: conj(W^{n+1}) is applied in the gather.
        if constexpr (MODE == kBlind) dst[G * m] = q;
        else dst[G * m] = mul_conj(q, pr[G * m]);
      }
    }
  }

  if constexpr (MODE != kAdj) {
    if (a.rf_part) {
      const double s = slot_sum<NT>(rf, red, t, slot);
      if (t == 0 && live) a.rf_part[f] = s;
    }
  }
}

}  // namespace pdd
