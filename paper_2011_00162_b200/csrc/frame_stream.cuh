// Streamed per-frame SWEEP kernel for large frames (S = 64, 128).
//
// Same arithmetic as frame_kernel<..., kSweep> (the nonblind z/Gamma step of
// solver.cpp:125-139 fused between the two transforms, then the
// back-projection of solver.cpp:157-164), restructured around what limits a
// 128^2 complex64 frame on one SM: the frame (128 KB) fills the shared-memory
// transpose tile, so memory latency must be hidden *inside* the frame.
//
//   rows forward   : patch x probe -> 1-D FFTs of all rows -> smem (natural)
//   column groups  : for each group of CG columns (columns are independent
//                    once the rows are done): column FFT -> prox against
//                    Gamma/amplitude values PREFETCHED into registers one
//                    group ahead -> inverse column FFT -> smem
//   rows inverse   : 1-D inverse FFTs of all rows -> x conj(probe) -> HBM
// The Gamma/amplitude loads of group g+1 (or of the next frame's first group)
// are issued right after group g's prox, so they land while the inverse and
// forward column transforms run; stores are fire-and-forget.  Persistent CTAs
// walk frames with a grid stride.  Loops over row batches and column groups
// are not unrolled, which keeps the SASS inside the instruction cache (the
// fully unrolled engine spent a quarter of its stall samples on
// no_instructions in its ncu capture).
#pragma once

#include <type_traits>

#include "frame_kernel.cuh"
#include "tmem.cuh"

namespace pdd {

template <int S_, int NT_, int GR_, int GC_, int MINB_ = 1>
struct StreamShape {
  static constexpr int S = S_, NT = NT_, GR = GR_, GC = GC_, MINB = MINB_;
  static constexpr int RR = S / GR;          // row elements per thread
  static constexpr int RPB = NT / GR;        // rows per batch
  static constexpr int NRB = S / RPB;        // row batches
  static constexpr int RC = S / GC;          // column elements per thread
  static constexpr int CG = NT / GC;         // columns per group
  static constexpr int NG = S / CG;          // column groups
  static constexpr int P = S + GR;           // smem pitch (bank-conflict-free with the rotation swizzle)
  static constexpr int RW = 32 / GR;         // rows per warp in the row phases
  static_assert(RR >= GR && RR % GR == 0, "row split");
  static_assert(RC >= GC && RC % GC == 0, "column split");
  static_assert(S % RPB == 0 && S % CG == 0 && CG >= 32, "grouping");
};

// TMEM columns holding one thread's probe values for all its row batches
// (32-bit words): the probe is identical for every frame, so it is staged once
// per persistent CTA in tensor memory instead of being re-read from L2 twice
// per frame (64 loads/thread/frame).
template <class SH>
struct ProbeTmem {
  static constexpr int PER_THREAD = SH::NRB * 2 * SH::RR;
  static constexpr int SLOTS = (SH::NT / 32) / 4;  // warps sharing a lane quarter
  static constexpr int RAW = PER_THREAD * SLOTS;
  static constexpr int NCOLS = RAW <= 32 ? 32 : RAW <= 64 ? 64 : RAW <= 128 ? 128 : RAW <= 256 ? 256 : 512;
  static_assert(RAW <= 512, "probe does not fit in TMEM");
};

// FWD = true: the forward half only (FrameMode kFwd: A u -> frames_out,
// |A u|^2 -> inten_out, R-factor partials), e.g. the trailing R-factor pass.
template <typename T, class SH, bool FAST, bool TMEMP = false, bool FWD = false>
__global__ void __launch_bounds__(SH::NT, SH::MINB) sweep_stream_kernel(const FrameArgs<T> a) {
  constexpr int S = SH::S, NT = SH::NT, GR = SH::GR, GC = SH::GC, RR = SH::RR, RC = SH::RC;
  constexpr int RPB = SH::RPB, NRB = SH::NRB, CG = SH::CG, NG = SH::NG, P = SH::P;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cx<T>* tw = reinterpret_cast<cx<T>*>(smem_raw);
  cx<T>* twr = tw + S;  // row-phase inter-stage twiddles, [k][g] = W_S^(g k): lane-consecutive reads
  cx<T>* buf = twr + S;
  double* red = reinterpret_cast<double*>(buf + S * P);

  if (a.stop_flag && *a.stop_flag) return;
  const int t = threadIdx.x;
  for (int i = t; i < S; i += NT) {
    tw[i] = a.tw[i];
    twr[i] = a.tw[(i % GR) * (i / GR)];
  }

  __shared__ uint32_t tmem_slot;
  uint32_t tmem_base = 0;
  const int warp = t >> 5;
  if constexpr (TMEMP) {
    static_assert(std::is_same_v<T, float> && 2 * RR == 32, "TMEM probe path: float, 16 values per row batch");
    if (warp == 0) tmem_alloc<ProbeTmem<SH>::NCOLS>(&tmem_slot);
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    tmem_base = tmem_slot;
    const int col0 = (warp >> 2) * ProbeTmem<SH>::PER_THREAD;
#pragma unroll 1
    for (int rb = 0; rb < NRB; ++rb) {
      const int y = rb * RPB + t / GR, g = t % GR;
      uint32_t raw[32];
#pragma unroll
      for (int m = 0; m < RR; ++m) {
        // the unitary 1/S of both transforms folded into the cached probe
        // (S a power of two: exact, results unchanged)
        const cx<T> p = a.probe[y * S + g + GR * m] * a.scale;
        raw[2 * m] = __float_as_uint(p.x);
        raw[2 * m + 1] = __float_as_uint(p.y);
      }
      tmem_st32(tmem_addr(tmem_base, warp, col0 + 32 * rb), raw);
    }
    tmem_wait_st();
  }
  __syncthreads();
  // this thread's probe values for row batch rb, from TMEM or global memory
  auto probe_row = [&](int ff, int rb, int y, int g, cx<T>* pv) {
    if constexpr (TMEMP) {
      uint32_t raw[32];
      tmem_ld32(tmem_addr(tmem_base, warp, (warp >> 2) * ProbeTmem<SH>::PER_THREAD + 32 * rb), raw);
      tmem_wait_ld();
#pragma unroll
      for (int m = 0; m < RR; ++m) pv[m] = cx<T>{__uint_as_float(raw[2 * m]), __uint_as_float(raw[2 * m + 1])};
    } else {
      // per-frame probe tiles (blind: the subdomain's copy W_d) via probe_idx
      const cx<T>* pr =
          a.probe + (a.probe_idx ? static_cast<int64_t>(a.probe_idx[ff]) * S * S : int64_t(0)) + y * S + g;
#pragma unroll
      for (int m = 0; m < RR; ++m) pv[m] = pr[GR * m];
    }
  };

  // Patch rows by bulk TMA: in the inverse row phase each warp's own rows of
  // buf fall free; 4 lanes then copy the next frame's patch rows for the same
  // warp and row batch into them (1 KB each, completion on a per-(warp, batch)
  // mbarrier), so the forward row phase reads them from shared memory instead
  // of waiting on HBM.  Needs 16-byte aligned rows (even window offsets and
  // pitches; checked on the host).
  constexpr int NW = NT / 32;
  __shared__ __align__(8) uint64_t s_rowbar[NW * NRB];
  const bool tma_rows = !FWD && a.rows_al16 != 0 && sizeof(cx<T>) * S % 16 == 0;
  if (tma_rows) {
    if (t < NW * NRB) mbar_init(s_rowbar + t, 1);
    mbar_init_fence();
    __syncthreads();
  }
  auto issue_rows = [&](int ff, int rb) {  // whole warp; rows rb*RPB + RW*warp + [0, RW)
    const int lane = t & 31;
    uint64_t* bar = s_rowbar + rb * NW + warp;
    if (lane == 0) mbar_arrive_expect_tx(bar, SH::RW * S * sizeof(cx<T>));
    __syncwarp();
    if (lane < SH::RW) {
      const int y = rb * RPB + SH::RW * warp + lane;
      bulk_g2s(buf + y * P, a.img + a.off[ff] + static_cast<int64_t>(y) * a.pitch[ff], S * sizeof(cx<T>), bar);
    }
  };
  uint32_t row_phase = 0;  // parity of the frames consumed so far

  const T scale = TMEMP ? T(1) : a.scale;  // TMEM probe carries the 1/S
  const T inv1pl = T(1) / (T(1) + a.lam);
  const int cx_ = t % CG, gc = t / CG;  // column-phase coordinates

  // Prefetch registers: Gamma and amplitude of one column group.
  cx<T> pg[RC];
  T pa[RC];
  auto prefetch = [&](int ff, int grp) {
    if (ff >= a.nframes) return;
    // one base pointer per array; the (ky - gc) * S offsets are immediates
    const int64_t base = static_cast<int64_t>(ff) * S * S + gc * S + grp * CG + cx_;
    const cx<T>* gsrc = a.gamma_in + base;
    const T* asrc = a.amp + base;
#pragma unroll
    for (int q = 0; q < RC / GC; ++q)
#pragma unroll
      for (int k1 = 0; k1 < GC; ++k1) {
        const int oy = GC * q + RC * k1;
        if constexpr (!FWD) pg[q * GC + k1] = gsrc[oy * S];
        if (!FWD || a.rf_part) pa[q * GC + k1] = asrc[oy * S];
      }
  };
  prefetch(blockIdx.x, 0);
  if (tma_rows && blockIdx.x < a.nframes)
#pragma unroll 1
    for (int rb = 0; rb < NRB; ++rb) issue_rows(blockIdx.x, rb);

#ifdef PDD_PHASE_TIMING
  unsigned long long tph[4] = {0, 0, 0, 0};
#define PDD_TICK(i)                                 \
  do {                                              \
    const unsigned long long now = clock64();       \
    tph[i] += now - tlast;                          \
    tlast = now;                                    \
  } while (0)
  unsigned long long tlast = clock64();
#else
#define PDD_TICK(i) \
  do {              \
  } while (0)
#endif
  for (int f = blockIdx.x; f < a.nframes; f += gridDim.x) {
    const int64_t fbase = static_cast<int64_t>(f) * S * S;
    // ---------------- rows, forward
#pragma unroll 1
    for (int rb = 0; rb < NRB; ++rb) {
      const int y = rb * RPB + t / GR, g = t % GR;
      cx<T> v[RR], pv[RR];
      if (tma_rows) {
        mbar_wait(s_rowbar + rb * NW + warp, row_phase);
#pragma unroll
        for (int m = 0; m < RR; ++m) v[m] = buf[y * P + g + GR * m];
        __syncwarp();  // all lanes hold their row elements before the row is overwritten
      } else {
        const cx<T>* src = a.img + a.off[f] + static_cast<int64_t>(y) * a.pitch[f] + g;
#pragma unroll
        for (int m = 0; m < RR; ++m) v[m] = src[GR * m];
      }
      probe_row(f, rb, y, g, pv);
#pragma unroll
      for (int m = 0; m < RR; ++m) v[m] = v[m] * pv[m];
      dft<RR, false>(v);
#pragma unroll
      for (int k = 0; k < RR; ++k) {
        const int k2 = k;
        buf[y * P + k2 * GR + ((g + k2) & (GR - 1))] = (k == 0) ? v[k] : v[k] * twr[k * GR + g];
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < RR / GR; ++q) {
        const int k2 = g + GR * q;
#pragma unroll
        for (int gp = 0; gp < GR; ++gp) v[q * GR + gp] = buf[y * P + k2 * GR + ((gp + k2) & (GR - 1))];
        dft<GR, false>(v + q * GR);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < RR / GR; ++q) {
        const int k2 = g + GR * q;
#pragma unroll
        for (int k1 = 0; k1 < GR; ++k1) buf[y * P + k2 + RR * k1] = v[q * GR + k1];
      }
    }
    __syncthreads();
    PDD_TICK(0);

    // ---------------- column groups: forward, prox, inverse
    T rf_acc = T(0);  // <= 2*RC terms per thread: float is ample; the tree below is double
#pragma unroll 1
    for (int grp = 0; grp < NG; ++grp) {
      const int x = grp * CG + cx_;
      cx<T> w[RC];
#pragma unroll
      for (int m = 0; m < RC; ++m) w[m] = buf[(gc + GC * m) * P + x];
      dft<RC, false>(w);
#pragma unroll
      for (int k = 0; k < RC; ++k) buf[(k * GC + gc) * P + x] = (k == 0) ? w[k] : w[k] * tw[gc * k];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < RC / GC; ++q) {
        const int k2 = gc + GC * q;
#pragma unroll
        for (int gp = 0; gp < GC; ++gp) w[q * GC + gp] = buf[(k2 * GC + gp) * P + x];
        dft<GC, false>(w + q * GC);
      }
      // Fourier-domain step: w[q*GC + k1] = X(ky = gc + GC q + RC k1, kx = x)
      T acc = T(0);
      const int64_t fx = fbase + gc * S + x;  // + (ky - gc) * S below, immediates
      if constexpr (FWD) {
#pragma unroll
        for (int q = 0; q < RC / GC; ++q)
#pragma unroll
          for (int k1 = 0; k1 < GC; ++k1) {
            const int e = q * GC + k1;
            const int64_t idx = fx + (GC * q + RC * k1) * S;
            const cx<T> au = w[e] * scale;
            if (a.frames_out) a.frames_out[idx] = au;
            if (a.inten_out) a.inten_out[idx] = norm2(au);
            if (a.rf_part) {
              if constexpr (FAST && std::is_same_v<T, float>) acc += fabsf(abs_fast_f32(au) - pa[e]);
              else acc += fabs(sqrt(norm2(au)) - pa[e]);
            }
          }
        rf_acc += acc;
        if (grp + 1 < NG) prefetch(f, grp + 1);
        else prefetch(f + gridDim.x, 0);
        continue;  // groups own disjoint columns of buf: no barrier between them
      }
#pragma unroll
      for (int q = 0; q < RC / GC; ++q)
#pragma unroll
        for (int k1 = 0; k1 < GC; ++k1) {
          const int e = q * GC + k1;
          const int64_t idx = fx + (GC * q + RC * k1) * S;
          const cx<T> au = w[e] * scale;
          const cx<T> yv = pg[e] + au;
          cx<T> z;
          if constexpr (FAST && std::is_same_v<T, float>) {
            acc += fabsf(abs_fast_f32(au) - pa[e]);
            z = prox_fast_f32(yv, pa[e], a.lam, inv1pl);
          } else {
            acc += fabs(sqrt(norm2(au)) - pa[e]);
            z = stagm_prox(yv, pa[e], a.lam, a.eps, FAST);
          }
          const cx<T> gn = yv - z;
          a.gamma_out[idx] = gn;
          if (a.z_out) a.z_out[idx] = z;
          w[e] = z - gn;
        }
      rf_acc += acc;
      if (grp + 1 < NG) prefetch(f, grp + 1);
      else prefetch(f + gridDim.x, 0);
#pragma unroll
      for (int q = 0; q < RC / GC; ++q) {
        const int k2 = gc + GC * q;
        dft<GC, true>(w + q * GC);
#pragma unroll
        for (int gp = 0; gp < GC; ++gp) buf[(k2 * GC + gp) * P + x] = w[q * GC + gp];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < RC; ++k) {
        const cx<T> v = buf[(k * GC + gc) * P + x];
        w[k] = (k == 0) ? v : mul_conj(v, tw[gc * k]);
      }
      dft<RC, true>(w);
#pragma unroll
      for (int m = 0; m < RC; ++m) buf[(gc + GC * m) * P + x] = w[m];
    }
    __syncthreads();
    PDD_TICK(1);

    // ---------------- rows, inverse -> x conj(probe) -> back-projection tile
#pragma unroll 1
    for (int rb = 0; rb < (FWD ? 0 : NRB); ++rb) {
      const int y = rb * RPB + t / GR, g = t % GR;
      cx<T> v[RR], pv[RR];
      probe_row(f, rb, y, g, pv);
#pragma unroll
      for (int q = 0; q < RR / GR; ++q) {
        const int k2 = g + GR * q;
#pragma unroll
        for (int k1 = 0; k1 < GR; ++k1) v[q * GR + k1] = buf[y * P + k2 + RR * k1];
        dft<GR, true>(v + q * GR);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < RR / GR; ++q) {
        const int k2 = g + GR * q;
#pragma unroll
        for (int gp = 0; gp < GR; ++gp) buf[y * P + k2 * GR + ((gp + k2) & (GR - 1))] = v[q * GR + gp];
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < RR; ++k) {
        const cx<T> b = buf[y * P + k * GR + ((g + k) & (GR - 1))];
        v[k] = (k == 0) ? b : mul_conj(b, twr[k * GR + g]);
      }
      if (tma_rows && f + static_cast<int>(gridDim.x) < a.nframes) {
        __syncwarp();             // this warp's rows are consumed
        fence_proxy_async_smem();  // ... before the async proxy overwrites them
        issue_rows(f + gridDim.x, rb);
      }
      dft<RR, true>(v);
      cx<T>* dst = a.bp_out + fbase + y * S + g;
#pragma unroll
      if (a.bp_raw) {  // blind: q_j = IFFT(.) itself; conj(W^{n+1}) is applied in the gather
#pragma unroll
        for (int m = 0; m < RR; ++m) dst[GR * m] = v[m] * scale;
      } else {
#pragma unroll
        for (int m = 0; m < RR; ++m) dst[GR * m] = mul_conj(v[m] * scale, pv[m]);
      }
    }

    PDD_TICK(2);
    row_phase ^= 1u;
    // per-frame R-factor partial (deterministic tree)
    double rf = static_cast<double>(rf_acc);
    if (a.rf_part) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rf += __shfl_down_sync(0xffffffffu, rf, o);
      if ((t & 31) == 0) red[t >> 5] = rf;
    }
    __syncthreads();  // also: rows of the next frame overwrite buf
    if (a.rf_part && t == 0) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += red[w];
      a.rf_part[f] = s;
    }
    PDD_TICK(3);
  }
#ifdef PDD_PHASE_TIMING
  if (a.phase_cycles && t == 0)
    for (int i = 0; i < 4; ++i) atomicAdd(a.phase_cycles + i, tph[i]);
#endif
#undef PDD_TICK
  if constexpr (TMEMP) {
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    if (warp == 0) tmem_dealloc<ProbeTmem<SH>::NCOLS>(tmem_base);
  }
}

template <typename T, class SH>
size_t stream_smem_bytes() {
  return sizeof(cx<T>) * (2 * SH::S + static_cast<size_t>(SH::S) * SH::P) + sizeof(double) * (SH::NT / 32);
}

}  // namespace pdd
