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

#include <cstdio>
#include <type_traits>

#include "frame_kernel.cuh"
#include "tmem.cuh"

#ifndef PDD_ACC_ON
#define PDD_ACC_ON true  // tensor-memory back-projection accumulation (false: A/B builds)
#endif

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
  // Back-projection accumulator ring after the probe: per thread (image row
  // Y mod 16, column residue g) 8 ring slots of 16-row bands x RR complex.
  static constexpr int ACC0 = NCOLS;
  static constexpr int ACC_COLS = 8 * 2 * SH::RR;
  static constexpr int NCOLS_ACC = ACC0 + ACC_COLS;
};

#ifndef PDD_TW128
#define PDD_TW128 0  // twiddles by 16-byte shared loads (two per instruction)
#endif
#ifndef PDD_ROWFUSE
#define PDD_ROWFUSE 1  // inverse rows of frame i and forward rows of frame i+1 without a CTA barrier
#endif
#ifndef PDD_COLSPLIT
#define PDD_COLSPLIT 2  // column groups: independent warp sets exchanging through named barriers
#endif

#ifdef PDD_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[4];  // summed over CTAs; printed by launch_stream
#endif
#ifndef PDD_SMETA
#define PDD_SMETA 1  // schedule records staged in shared memory a frame ahead (no global metadata loads behind barriers)
#endif
#ifndef PDD_SKEW
#define PDD_SKEW 2000  // cycles by which column warp set k starts after set k-1 (see "Staggered warps")
#endif
#ifndef PDD_CHAINR
#define PDD_CHAINR 1  // row phases chained by warp rank on the scheduler: rank k starts when rank k-1 issued its first exchange
#endif

// Two twiddles W[k], W[k+1] (k even) by one 16-byte shared-memory load.
__device__ __forceinline__ void tw_pair(const cx<float>* p, cx<float>& a, cx<float>& b) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  a = cx<float>{v.x, v.y};
  b = cx<float>{v.z, v.w};
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

#ifndef PDD_STAGE64
#define PDD_STAGE64 0  // A/B builds: stage the S = 64 amplitudes too
#endif
// Which shapes stage the column group's amplitudes in shared memory.
template <typename T, class SH, bool FWD>
constexpr bool amp_tile_staged() {
  return (SH::S == 128 || PDD_STAGE64) && std::is_same_v<T, float>;
}

template <typename T, class SH>
constexpr size_t stream_smem_bytes_base();

// Shapes whose transpose tile does not fit in shared memory (complex128
// 128^2: 272 KB) keep it in a per-CTA global scratch slice instead
// (a.scratch + blockIdx.x * S * P; L2-resident: ~80 MB for the whole grid).
template <typename T, class SH>
constexpr bool tile_in_global() {
  return sizeof(cx<T>) * static_cast<size_t>(SH::S) * SH::P > (size_t(160) << 10);
}

// FWD = true: the forward half only (FrameMode kFwd: A u -> frames_out,
// |A u|^2 -> inten_out, R-factor partials), e.g. the trailing R-factor pass.
// ADJ = true: the inverse half only (FrameMode kAdj: frames_in -> IFFT2 ->
// x conj(probe) -> bp_out per frame), global-tile shapes only.
// RF2 = true (blind, blind.cpp:320-332 inside the sweep): the R-factor of u^n is
// taken with the SHARED probe a.probe2 through a second forward transform of
// the same patch (second transpose tile; one pass over patches and amplitudes
// instead of a separate FWD launch), while the sweep itself runs with the
// subdomain copies (a.probe / probe_idx).
template <typename T, class SH, bool FAST, bool TMEMP = false, bool FWD = false, bool ADJ = false, bool RF2 = false>
__global__ void __launch_bounds__(SH::NT, SH::MINB) sweep_stream_kernel(const FrameArgs<T> a) {
  constexpr int S = SH::S, NT = SH::NT, GR = SH::GR, GC = SH::GC, RR = SH::RR, RC = SH::RC;
  constexpr int RPB = SH::RPB, NRB = SH::NRB, CG = SH::CG, NG = SH::NG, P = SH::P;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 16-byte twiddle loads: float, RR/RC even
  constexpr bool TWV = PDD_TW128 && std::is_same_v<T, float> && RR % 2 == 0 && RC % 2 == 0;
  // column phase split into NSPLIT independent warp sets (S = 128 float sweep)
  constexpr int NSPLIT = (std::is_same_v<T, float> && S == 128 && CG % PDD_COLSPLIT == 0 &&
                          (NT / 32) % PDD_COLSPLIT == 0) ? PDD_COLSPLIT : 1;
  cx<T>* tw = reinterpret_cast<cx<T>*>(smem_raw);
  cx<T>* twr = tw + S;  // row-phase inter-stage twiddles, [k][g] = W_S^(g k): lane-consecutive reads
  cx<T>* twc = twr + S;  // column-phase twiddles, [gc][k] = W_S^(gc k): immediate offsets in k
  constexpr bool GTILE = tile_in_global<T, SH>();
  static_assert(!ADJ || GTILE, "ADJ: global-tile shapes only");
  static_assert(!(GTILE && TMEMP), "global tile: no tensor-memory paths");
  constexpr bool STRIDED = FWD || ADJ;  // frames blockIdx.x + k * gridDim.x (no piece schedule)
  constexpr bool SMETA = PDD_SMETA && !STRIDED;
  __shared__ PosRec s_rec[3];
  cx<T>* buf = GTILE ? a.scratch + static_cast<int64_t>(blockIdx.x) * S * P : twc + S;
  double* red = reinterpret_cast<double*>(GTILE ? twc + S : buf + S * P);
  // S = 128: the amplitudes of the next column group land by cp.async straight
  // in shared memory ([element][thread], conflict-free, read back only by the
  // thread that copied them) -- the column phase sits at the 128-register cap
  // and a register prefetch spilled.
  T* ampst = reinterpret_cast<T*>(red + NT / 32);
  static_assert(!RF2 || (!FWD && !ADJ && !TMEMP && !tile_in_global<T, SH>() && !amp_tile_staged<T, SH, false>()),
                "RF2: shared-memory tile shapes without staged amplitudes");
  cx<T>* buf2 = reinterpret_cast<cx<T>*>(smem_raw + stream_smem_bytes_base<T, SH>());  // RF2 only

  if (a.stop_flag && *a.stop_flag) return;
  const int t = threadIdx.x;
  for (int i = t; i < S; i += NT) {
    tw[i] = a.tw[i];
    if constexpr (TWV) twr[i] = a.tw[((i >> 1) % GR) * ((i / (2 * GR)) * 2 + (i & 1))];  // [k/2][g][k%2]
    else twr[i] = a.tw[(i % GR) * (i / GR)];
    twc[i] = a.tw[(i / RC) * (i % RC)];
  }

  __shared__ uint32_t tmem_slot;
  uint32_t tmem_base = 0;
  const int warp = t >> 5;
  // tensor-memory back-projection accumulation across the frames of a piece
  // (S = 128: the 16-row ring maps an image row to a fixed lane, see layout.hpp)
  constexpr bool ACC = PDD_ACC_ON && TMEMP && !FWD && S == 128 && SH::GR == 8;
  constexpr int TCOLS = ACC ? 512 : ProbeTmem<SH>::NCOLS;
  if constexpr (ACC) static_assert(ProbeTmem<SH>::NCOLS_ACC <= 512, "TMEM: probe + accumulator");
  if constexpr (TMEMP) {
    static_assert(std::is_same_v<T, float> && 2 * RR == 32, "TMEM probe path: float, 16 values per row batch");
    if (warp == 0) tmem_alloc<TCOLS>(&tmem_slot);
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
  if constexpr (SMETA) {
    if (t < 2) {
      const int j = a.cta_beg[blockIdx.x] + t;
      if (j < a.cta_beg[blockIdx.x + 1]) s_rec[t] = a.pc_rec[j];
      else s_rec[t].f = -1;
    }
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
  const bool tma_rows = !FWD && !ADJ && !GTILE && a.rows_al16 != 0 && sizeof(cx<T>) * S % 16 == 0;
  if (tma_rows) {
    if (t < NW * NRB) mbar_init(s_rowbar + t, 1);
    mbar_init_fence();
    __syncthreads();
  }
  auto issue_rows = [&](int ff, int64_t woff, int wpitch, int rb) {  // whole warp; rows rb*RPB + RW*warp + [0, RW)
    const int lane = t & 31;
    uint64_t* bar = s_rowbar + rb * NW + warp;
    if (lane == 0) mbar_arrive_expect_tx(bar, SH::RW * S * sizeof(cx<T>));
    __syncwarp();
    if (lane < SH::RW) {
      const int y = rb * RPB + SH::RW * warp + lane;
#ifdef PDD_BOUNDS
      if (ff < 0 || ff >= a.nframes || woff != a.off[ff] || wpitch != a.pitch[ff] ||
          woff + static_cast<int64_t>(y) * wpitch + S > a.img_elems || ((woff + static_cast<int64_t>(y) * wpitch) & 1)) {
        printf("PDD_BOUNDS issue_rows: cta %d ff %d y %d off %lld pitch %d\n", blockIdx.x, ff, y, (long long)woff, wpitch);
        __trap();
      }
#endif
      bulk_g2s(buf + y * P, a.img + woff + static_cast<int64_t>(y) * wpitch, S * sizeof(cx<T>), bar);
    }
  };
  uint32_t row_phase = 0;  // parity of the frames consumed so far

  const T scale = TMEMP ? T(1) : a.scale;  // TMEM probe carries the 1/S
  const T inv1pl = T(1) / (T(1) + a.lam);
  // column-phase coordinates.  The warps form NSPLIT sets; set k owns columns
  // [k CG/NSPLIT, (k+1) CG/NSPLIT) of every group, so a set exchanges only
  // within itself (named barrier 1 + k) and the sets drift apart in time.
  constexpr int SETT = NT / NSPLIT, SETC = CG / NSPLIT;  // threads, columns per set
  const int cx_ = (t / SETT) * SETC + (t % SETT) % SETC;
  const int gc = (t % SETT) / SETC;
  auto col_sync = [&]() {
    if constexpr (NSPLIT == 1) __syncthreads();
    else if constexpr (SETT == 32) __syncwarp();
    else named_bar(1 + t / SETT, SETT);
  };

  // Prefetch registers: Gamma and amplitude of one column group.
  cx<T> pg[RC];
  constexpr bool STAGE = amp_tile_staged<T, SH, FWD>();
  T pa[STAGE ? 1 : RC];
  auto pa_at = [&](int e) {
    if constexpr (STAGE) return ampst[e * NT + t];
    else return pa[e];
  };
  auto prefetch = [&](int ff, int grp) {
    if (ff < 0) return;
#ifdef PDD_BOUNDS
    if (ff >= a.nframes) {
      printf("PDD_BOUNDS prefetch: cta %d ff %d grp %d\n", blockIdx.x, ff, grp);
      __trap();
    }
#endif
    // one base pointer per array; the (ky - gc) * S offsets are immediates
    const int64_t base = static_cast<int64_t>(ff) * S * S + gc * S + grp * CG + cx_;
    const cx<T>* gsrc = (ADJ ? a.frames_in : a.gamma_in) + base;
    const T* asrc = a.amp + base;
#pragma unroll
    for (int q = 0; q < RC / GC; ++q)
#pragma unroll
      for (int k1 = 0; k1 < GC; ++k1) {
        const int oy = GC * q + RC * k1;
        if constexpr (!FWD) pg[q * GC + k1] = gsrc[oy * S];
        if constexpr (ADJ) continue;
        if (!FWD || a.rf_part) {
          if constexpr (STAGE) cp_async4(ampst + (q * GC + k1) * NT + t, asrc + oy * S);
          else pa[q * GC + k1] = asrc[oy * S];
        }
      }
    if constexpr (STAGE) cp_async_commit();
  };
#ifdef PDD_CANARY  // debug builds: detect shared-memory writes past the working set
  uint32_t* canary = reinterpret_cast<uint32_t*>(smem_raw + stream_smem_bytes_base<T, SH>() +
                                                 (RF2 ? sizeof(cx<T>) * static_cast<size_t>(S) * P : 0));
  for (int k = t; k < (48 << 10) / 4; k += NT) canary[k] = 0xDEADBEEFu;
  __syncthreads();
#endif
  // Work order.  SWEEP: this CTA's positions [cta_beg[b], cta_beg[b+1]) of the
  // host schedule (frames in back-projection piece order; layout.hpp).
  // FWD: frames blockIdx.x + k * gridDim.x.
  int i = STRIDED ? static_cast<int>(blockIdx.x) : a.cta_beg[blockIdx.x];
  const int iend = STRIDED ? a.nframes : a.cta_beg[blockIdx.x + 1];
  constexpr int kStepOne = 1;
  auto next_of = [&](int j) { return STRIDED ? j + static_cast<int>(gridDim.x) : j + kStepOne; };
  // SMETA: the schedule records of positions i, i+1 (and i+2, in flight) sit in
  // the ring s_rec; c0 is the slot of position i.
  int c0 = 0;
  auto slot = [&](int k) { return c0 + k >= 3 ? c0 + k - 3 : c0 + k; };
  auto frame_cur = [&]() -> int {  // frame of position i (-1: none)
    if constexpr (SMETA) return s_rec[c0].f;
    else if constexpr (STRIDED) return i < iend ? i : -1;
    else return i < iend ? a.pc_pos[i].x : -1;
  };
  auto frame_nxt = [&]() -> int {  // frame of the position after i
    const int j = next_of(i);
    if constexpr (SMETA) return s_rec[slot(1)].f;
    else if constexpr (STRIDED) return j < iend ? j : -1;
    else return j < iend ? a.pc_pos[j].x : -1;
  };
  // window corner offset / row pitch of frame ff held in ring slot k (SMETA) or from the frame tables
  auto win_off = [&](int ff, int k) -> int64_t {
    if constexpr (SMETA) return s_rec[slot(k)].woff;
    else return a.off[ff];
  };
  auto win_pitch = [&](int ff, int k) -> int {
    if constexpr (SMETA) return s_rec[slot(k)].pitch;
    else return a.pitch[ff];
  };
  {
    const int f0 = frame_cur();
    prefetch(f0, 0);
    if (tma_rows && f0 >= 0) {
      const int64_t wo = win_off(f0, 0);
      const int wp = win_pitch(f0, 0);
#pragma unroll 1
      for (int rb = 0; rb < NRB; ++rb) issue_rows(f0, wo, wp, rb);
    }
  }

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
  // ---------------- rows, forward (frame f): warp-local (each warp owns its rows)
  auto fwd_rows = [&](int f, int k) {  // k: ring slot offset of f's record (SMETA)
#pragma unroll 1
    for (int rb = 0; rb < NRB; ++rb) {
      const int y = rb * RPB + t / GR, g = t % GR;
      cx<T> v[RR], pv[RR];
      cx<T> pw2[RF2 ? RR : 1];
      if constexpr (!TMEMP) {  // probe values from L2: in flight while the patch rows arrive
        probe_row(f, rb, y, g, pv);
        if constexpr (RF2) {
          const cx<T>* pw = a.probe2 + y * S + g;
#pragma unroll
          for (int m = 0; m < RR; ++m) pw2[m] = pw[GR * m];
        }
      }
      if (tma_rows) {
        mbar_wait(s_rowbar + rb * NW + warp, row_phase);
#pragma unroll
        for (int m = 0; m < RR; ++m) v[m] = buf[y * P + g + GR * m];
        __syncwarp();  // all lanes hold their row elements before the row is overwritten
      } else {
        const cx<T>* src = a.img + win_off(f, k) + static_cast<int64_t>(y) * win_pitch(f, k) + g;
#pragma unroll
        for (int m = 0; m < RR; ++m) v[m] = src[GR * m];
      }
      // 1-D transform of this thread's row elements through the warp's rows of dst
      auto row_fft = [&](cx<T>* vv, cx<T>* dst) {
        dft<RR, false>(vv);
#pragma unroll
        for (int k = 0; k < RR; k += 2) {
          cx<T> t0, t1;
          if constexpr (TWV) tw_pair(twr + (k >> 1) * 2 * GR + 2 * g, t0, t1);
          else t0 = twr[k * GR + g], t1 = twr[(k + 1) * GR + g];
          dst[y * P + k * GR + ((g + k) & (GR - 1))] = (k == 0) ? vv[k] : vv[k] * t0;
          dst[y * P + (k + 1) * GR + ((g + k + 1) & (GR - 1))] = vv[k + 1] * t1;
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < RR / GR; ++q) {
          const int k2 = g + GR * q;
#pragma unroll
          for (int gp = 0; gp < GR; ++gp) vv[q * GR + gp] = dst[y * P + k2 * GR + ((gp + k2) & (GR - 1))];
          dft<GR, false>(vv + q * GR);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < RR / GR; ++q) {
          const int k2 = g + GR * q;
#pragma unroll
          for (int k1 = 0; k1 < GR; ++k1) dst[y * P + k2 + RR * k1] = vv[q * GR + k1];
        }
      };
      if constexpr (RF2) {  // patch x shared probe -> rows of the second tile
        cx<T> v2[RR];
#pragma unroll
        for (int m = 0; m < RR; ++m) v2[m] = v[m] * pw2[m];
        row_fft(v2, buf2);
      }
      if constexpr (TMEMP) probe_row(f, rb, y, g, pv);
#pragma unroll
      for (int m = 0; m < RR; ++m) v[m] = v[m] * pv[m];
      row_fft(v, buf);
    }
  };
  constexpr bool FUSE = PDD_ROWFUSE && !FWD && !ADJ;
  int pend_f = -1;  // FUSE: frame whose R-factor warp partials sit in red[]
  if constexpr (FUSE) {
    if (i < iend) fwd_rows(frame_cur(), 0);
  }
  for (; i < iend; i = next_of(i)) {
    const int f = frame_cur();
    const int64_t fbase = static_cast<int64_t>(f) * S * S;
#ifdef PDD_BOUNDS
    if (f < 0 || f >= a.nframes) {
      printf("PDD_BOUNDS frame: cta %d i %d iend %d f %d\n", blockIdx.x, i, iend, f);
      __trap();
    }
#endif
    if constexpr (!FUSE && !ADJ) fwd_rows(f, 0);
    if constexpr (ACC) tmem_fence_before_sync();
    __syncthreads();
    if constexpr (ACC) tmem_fence_after_sync();
    if constexpr (FUSE) {
      // summed by the first thread of the LAST warp set, which starts its
      // columns late anyway (staggered sets below)
      if (pend_f >= 0 && a.rf_part && t == NT - NT / NSPLIT) {
        double s = 0.0;
        for (int w = 0; w < NT / 32; ++w) s += red[w];
        a.rf_part[pend_f] = s;
      }
    }
    if constexpr (SMETA) {
      // the record of position i+2 lands during this column phase (its slot
      // held position i-1, last read before the barrier above)
      if (t == NT - 1) {
        PosRec* dst = s_rec + slot(2);
        if (i + 2 < iend) {
          cp_async16(dst, a.pc_rec + i + 2);
          cp_async16(reinterpret_cast<char*>(dst) + 16, reinterpret_cast<const char*>(a.pc_rec + i + 2) + 16);
          cp_async_commit();
        } else {
          dst->f = -1;
        }
      }
    }
    PDD_TICK(0);

#if PDD_SKEW
    // Staggered warps: after a CTA barrier all 16 warps run the same
    // shared-memory burst / FMA burst sequence in lockstep, so the two pipes
    // take turns instead of overlapping.  Starting warp set k late by
    // k * PDD_SKEW cycles keeps one set in its exchange while the other
    // computes (measured on config 4: K1 7.63 -> 7.30 ms at 2000 cycles).
    if (NSPLIT >= 2 && t >= SETT) {
      const long long t0 = clock64();
      const long long d = static_cast<long long>(PDD_SKEW) * (t / SETT);
      while (clock64() - t0 < d) {
      }
    }
#endif
    // ---------------- column groups: forward, prox, inverse
    T rf_acc = T(0);  // <= 2*RC terms per thread: float is ample; the tree below is double
#pragma unroll 1
    for (int grp = 0; grp < NG; ++grp) {
      const int x = grp * CG + cx_;
      cx<T> w[RC];
      if constexpr (ADJ) {
        // frames_in of this column group, in the layout the forward column
        // transform ends in: w[q*GC + k1] = X(ky = gc + GC q + RC k1, kx = x)
#pragma unroll
        for (int e = 0; e < RC; ++e) w[e] = pg[e];
        if (grp + 1 < NG) prefetch(f, grp + 1);
        else prefetch(frame_nxt(), 0);
      } else {
      T acc2 = T(0);
      if constexpr (RF2) {  // forward column transform of the shared-probe tile -> R-factor terms
        cx<T> w2[RC];
#pragma unroll
        for (int m = 0; m < RC; ++m) w2[m] = buf2[(gc + GC * m) * P + x];
        dft<RC, false>(w2);
#pragma unroll
        for (int k = 0; k < RC; k += 2) {
          const cx<T> t0 = twc[gc * RC + k], t1 = twc[gc * RC + k + 1];
          buf2[(k * GC + gc) * P + x] = (k == 0) ? w2[k] : w2[k] * t0;
          buf2[((k + 1) * GC + gc) * P + x] = w2[k + 1] * t1;
        }
        col_sync();
#pragma unroll
        for (int q = 0; q < RC / GC; ++q) {
          const int k2 = gc + GC * q;
#pragma unroll
          for (int gp = 0; gp < GC; ++gp) w2[q * GC + gp] = buf2[(k2 * GC + gp) * P + x];
          dft<GC, false>(w2 + q * GC);
        }
#pragma unroll
        for (int e = 0; e < RC; ++e) {
          const cx<T> au2 = w2[e] * scale;
          if constexpr (FAST && std::is_same_v<T, float>) acc2 += fabsf(abs_fast_f32(au2) - pa_at(e));
          else acc2 += fabs(sqrt(norm2(au2)) - pa_at(e));
        }
      }
#pragma unroll
      for (int m = 0; m < RC; ++m) w[m] = buf[(gc + GC * m) * P + x];
      dft<RC, false>(w);
#pragma unroll
      for (int k = 0; k < RC; k += 2) {
        cx<T> t0, t1;
        if constexpr (TWV) tw_pair(twc + gc * RC + k, t0, t1);
        else t0 = twc[gc * RC + k], t1 = twc[gc * RC + k + 1];
        buf[(k * GC + gc) * P + x] = (k == 0) ? w[k] : w[k] * t0;
        buf[((k + 1) * GC + gc) * P + x] = w[k + 1] * t1;
      }
      col_sync();
#pragma unroll
      for (int q = 0; q < RC / GC; ++q) {
        const int k2 = gc + GC * q;
#pragma unroll
        for (int gp = 0; gp < GC; ++gp) w[q * GC + gp] = buf[(k2 * GC + gp) * P + x];
        dft<GC, false>(w + q * GC);
      }
      // Fourier-domain step: w[q*GC + k1] = X(ky = gc + GC q + RC k1, kx = x)
      if constexpr (STAGE) cp_async_wait_all();  // this thread's staged amplitudes
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
              if constexpr (FAST && std::is_same_v<T, float>) acc += fabsf(abs_fast_f32(au) - pa_at(e));
              else acc += fabs(sqrt(norm2(au)) - pa_at(e));
            }
          }
        rf_acc += acc;
        if (grp + 1 < NG) prefetch(f, grp + 1);
        else prefetch(frame_nxt(), 0);
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
            acc += fabsf(abs_fast_f32(au) - pa_at(e));
            z = prox_fast_f32(yv, pa_at(e), a.lam, inv1pl);
          } else {
            acc += fabs(sqrt(norm2(au)) - pa_at(e));
            z = stagm_prox(yv, pa_at(e), a.lam, a.eps, FAST);
          }
          const cx<T> gn = yv - z;
          a.gamma_out[idx] = gn;
          if (a.z_out) a.z_out[idx] = z;
          w[e] = z - gn;
        }
      rf_acc += RF2 ? acc2 : acc;
      if (grp + 1 < NG) prefetch(f, grp + 1);
      else prefetch(frame_nxt(), 0);
      }  // !ADJ
#pragma unroll
      for (int q = 0; q < RC / GC; ++q) {
        const int k2 = gc + GC * q;
        dft<GC, true>(w + q * GC);
#pragma unroll
        for (int gp = 0; gp < GC; ++gp) buf[(k2 * GC + gp) * P + x] = w[q * GC + gp];
      }
      col_sync();
#pragma unroll
      for (int k = 0; k < RC; k += 2) {
        cx<T> t0, t1;
        if constexpr (TWV) tw_pair(twc + gc * RC + k, t0, t1);
        else t0 = twc[gc * RC + k], t1 = twc[gc * RC + k + 1];
        const cx<T> v0 = buf[(k * GC + gc) * P + x], v1 = buf[((k + 1) * GC + gc) * P + x];
        w[k] = (k == 0) ? v0 : mul_conj(v0, t0);
        w[k + 1] = mul_conj(v1, t1);
      }
      dft<RC, true>(w);
#pragma unroll
      for (int m = 0; m < RC; ++m) buf[(gc + GC * m) * P + x] = w[m];
    }
    if constexpr (SMETA && !STAGE) {
      if (t == NT - 1) cp_async_wait_all();
    }
    __syncthreads();
    PDD_TICK(1);

    // ---------------- rows, inverse -> x conj(probe) -> back-projection tile
    // this frame's piece bookkeeping: rows y < lo are final, rows y >= newfrom new
    int p_lo = S, p_new = 0, p_rot = 0;
    int64_t p_ofs = fbase;
    if constexpr (SMETA) {
      const PosRec r = s_rec[c0];
      p_lo = r.lo;
      p_new = r.nw_rot & 0xffff;
      p_rot = r.nw_rot >> 16;
      p_ofs = r.ofs;
    } else if constexpr (!STRIDED) {
      const int4 pi = a.pc_pos[i];
      p_lo = pi.y;
      p_new = pi.z;
      p_rot = pi.w;
      p_ofs = a.pc_ofs[i];
    }
    const int fn = frame_nxt();
    int64_t n_off = 0;
    int n_pitch = 0;
    if (tma_rows && fn >= 0) {
      n_off = win_off(fn, 1);
      n_pitch = win_pitch(fn, 1);
    }
#ifdef PDD_BOUNDS
    if (p_ofs < 0 || p_lo <= 0 || p_lo > S || p_new < 0 || p_new > S || fn >= a.nframes) {
      printf("PDD_BOUNDS piece: cta %d i %d f %d ofs %lld lo %d new %d fn %d\n", blockIdx.x, i, f, (long long)p_ofs, p_lo,
             p_new, fn);
      __trap();
    }
#endif
    // Staggered row phases: the four warps of a scheduler (ranks warp / 4)
    // start one after the other -- rank k once rank k-1 has issued its first
    // exchange -- so their shared-memory bursts and FFT arithmetic interleave
    // instead of coinciding (config 4: K1 7.30 -> 6.99 ms with the column stagger).
    constexpr bool CHR = PDD_CHAINR != 0 && !FWD && NW == 16;
    if constexpr (CHR) {
      if ((warp >> 2) > 0) named_bar(8 + (warp >> 2), 256);  // rank k waits for rank k-1
    }
#pragma unroll 1
    for (int rb = 0; rb < (FWD ? 0 : NRB); ++rb) {
      const int y = rb * RPB + t / GR, g = t % GR;
      cx<T> v[RR], pv[RR];
      if (TMEMP || !a.bp_raw) probe_row(f, rb, y, g, pv);  // blind: q_j is written without conj(probe)
#pragma unroll
      for (int q = 0; q < RR / GR; ++q) {
        const int k2 = g + GR * q;
#pragma unroll
        for (int k1 = 0; k1 < GR; ++k1) v[q * GR + k1] = buf[y * P + k2 + RR * k1];
        dft<GR, true>(v + q * GR);
      }
      if constexpr (CHR) {
        if (rb == 0 && (warp >> 2) < 3) named_arrive(9 + (warp >> 2), 256);
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
      for (int k = 0; k < RR; k += 2) {
        cx<T> t0, t1;
        if constexpr (TWV) tw_pair(twr + (k >> 1) * 2 * GR + 2 * g, t0, t1);
        else t0 = twr[k * GR + g], t1 = twr[(k + 1) * GR + g];
        const cx<T> b0 = buf[y * P + k * GR + ((g + k) & (GR - 1))];
        const cx<T> b1 = buf[y * P + (k + 1) * GR + ((g + k + 1) & (GR - 1))];
        v[k] = (k == 0) ? b0 : mul_conj(b0, t0);
        v[k + 1] = mul_conj(b1, t1);
      }
      if (tma_rows && fn >= 0) {
        __syncwarp();             // this warp's rows are consumed
        fence_proxy_async_smem();  // ... before the async proxy overwrites them
        issue_rows(fn, n_off, n_pitch, rb);
      }
      dft<RR, true>(v);
      if (a.bp_raw) {  // blind: q_j = IFFT(.) itself; conj(W^{n+1}) is applied in the gather
#pragma unroll
        for (int m = 0; m < RR; ++m) v[m] = v[m] * scale;
      } else {
#pragma unroll
        for (int m = 0; m < RR; ++m) v[m] = mul_conj(v[m] * scale, pv[m]);
      }
      if constexpr (ACC) {
        // warp-uniform: p_lo, p_new are multiples of 4 and a warp holds 4 rows
        const uint32_t ta = tmem_addr(tmem_base, warp, ProbeTmem<SH>::ACC0 + (((y >> 4) + p_rot) & 7) * (2 * RR));
        if (y < p_new) {  // rows already holding earlier frames of the piece
          uint32_t raw[32];
          tmem_ld32(ta, raw);
          tmem_wait_ld();
#pragma unroll
          for (int m = 0; m < RR; ++m) v[m] = v[m] + cx<T>{__uint_as_float(raw[2 * m]), __uint_as_float(raw[2 * m + 1])};
        }
        if (y >= p_lo) {  // later frames of the piece still add to this row
          uint32_t raw[32];
#pragma unroll
          for (int m = 0; m < RR; ++m) {
            raw[2 * m] = __float_as_uint(v[m].x);
            raw[2 * m + 1] = __float_as_uint(v[m].y);
          }
          tmem_st32(ta, raw);
          tmem_wait_st();
          continue;
        }
      }
      cx<T>* dst = a.bp_out + p_ofs + y * S + g;
#pragma unroll
      for (int m = 0; m < RR; ++m) dst[GR * m] = v[m];
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
    if constexpr (FUSE) {
      // the next frame's forward rows follow at once: a warp touches only its
      // own rows of buf, and the accumulator rows that change warps between
      // frames are ordered by the two barriers of the next frame
      pend_f = f;
      if (fn >= 0) fwd_rows(fn, 1);
    } else {
      if constexpr (ACC) tmem_fence_before_sync();  // accumulator rows change warps between frames
      __syncthreads();  // also: rows of the next frame overwrite buf
      if constexpr (ACC) tmem_fence_after_sync();
      if (a.rf_part && t == 0) {
        double s = 0.0;
        for (int w = 0; w < NT / 32; ++w) s += red[w];
        a.rf_part[f] = s;
      }
    }
    PDD_TICK(3);
    if constexpr (SMETA) c0 = slot(1);
  }
  if constexpr (FUSE) {
    __syncthreads();
    if (pend_f >= 0 && a.rf_part && t == 0) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += red[w];
      a.rf_part[pend_f] = s;
    }
  }
#ifdef PDD_CANARY
  __syncthreads();
  for (int k = t; k < (48 << 10) / 4; k += NT)
    if (canary[k] != 0xDEADBEEFu) {
      printf("PDD_CANARY cta %d: word %d past the end = %08x\n", blockIdx.x, k, canary[k]);
      break;
    }
#endif
#ifdef PDD_PHASE_TIMING
  if (t == 0)
    for (int i = 0; i < 4; ++i) atomicAdd(g_phase_cycles + i, tph[i]);
#endif
#undef PDD_TICK
  if constexpr (TMEMP) {
    tmem_fence_before_sync();
    __syncthreads();
    tmem_fence_after_sync();
    if (warp == 0) tmem_dealloc<TCOLS>(tmem_base);
  }
}

template <typename T, class SH>
constexpr size_t stream_smem_bytes_base() {
  return sizeof(cx<T>) * (3 * SH::S + (tile_in_global<T, SH>() ? 0 : static_cast<size_t>(SH::S) * SH::P)) +
         sizeof(double) * (SH::NT / 32) +
         (amp_tile_staged<T, SH, false>() ? sizeof(T) * static_cast<size_t>(SH::RC) * SH::NT : 0);
}
template <typename T, class SH>
size_t stream_smem_bytes(bool rf2 = false) {
  return stream_smem_bytes_base<T, SH>() + (rf2 ? sizeof(cx<T>) * static_cast<size_t>(SH::S) * SH::P : 0)
#ifdef PDD_CANARY
         + (size_t(48) << 10)  // debug builds: a canary region after the working set
#endif
      ;
}

}  // namespace pdd
