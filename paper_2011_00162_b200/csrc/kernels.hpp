// Host-side launch interface between the C++ drivers and the CUDA kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cx.cuh"

namespace pdd {

template <typename T>
struct FrameArgs;

// One rectangle of one overlap pair, seen from one side, in that side's
// subdomain-local coordinates (ddplan.cpp:14-19).
struct PairSide {
  int32_t r0, r1, c0, c1;
  int64_t v_off;    // element offset of v_p in the concatenated v buffer
  int64_t lam_off;  // element offset of Lambda_{p,side}
};

enum GatherMode : int {
  kGatherAdjoint = 0,  // out = sum_j bp_j (forward.cpp:43-54 overlap-add)
  kGatherNonblind = 1, // u-update + Lambda-update + RE partials (solver.cpp:154-193)
  kGatherBlind = 2,    // blind u-update with W^{n+1} (blind.cpp:253-272)
  kGatherDensity = 3,  // rho = sum_j |P|^2 (forward.cpp:56-66), double
};

template <typename T>
struct GatherArgs {
  int mode = 0;
  int ntiles = 0;
  int tile_h = 8;                       // rows per tile (multiple of 8)
  int tile_w = 32;                      // columns per tile: 32, or 64 (float, 16-byte column pairs)
  const int4* tiles = nullptr;          // {sub, r0, c0, frame_begin}; end = tiles[i+1].w
  const int32_t* tile_frames = nullptr; // local frame ids, ascending j per tile
  const int32_t* fr_r = nullptr;        // [nframes] window corner (subdomain coords)
  const int32_t* fr_c = nullptr;
  const int32_t* fr_sub = nullptr;      // [nframes] owning local subdomain
  // Nonblind update over back-projection pieces (layout.hpp) instead of
  // frames: partial image k is [it_h[k]][S] at bp + it_base[k], window corner
  // (it_r[k], it_c[k]); per tile the covering pieces tile_items[tile_item_beg[t] ..].
  const int32_t* tile_items = nullptr;
  const int32_t* tile_item_beg = nullptr;
  const int32_t* it_r = nullptr;
  const int32_t* it_c = nullptr;
  const int32_t* it_h = nullptr;
  const int64_t* it_base = nullptr;
  // Flattened per-tile lists (layout.cpp, preferred when set): covering
  // partial images of tile t are entries [mbeg[t], mbeg[t+1]) of meta
  // {r0, c0, h, frame} and mbase (element offset) -- one dependent load level
  // fewer than the tile_items -> it_* chain; the pair sides whose overlap
  // rectangle meets tile t are ps[tps[tps_beg[t] ..]] (usually none).
  const int32_t* mbeg = nullptr;
  const int4* meta = nullptr;
  const int64_t* mbase = nullptr;
  const int32_t* tps_beg = nullptr;
  const int32_t* tps = nullptr;
  int S = 0;
  const cx<T>* bp = nullptr;            // [nframes][S][S]
  const cx<T>* probe = nullptr;         // density: P; blind: W copies [nsub][S][S]
  const int64_t* sub_off = nullptr;     // [nsub] offset into image buffers
  const int32_t* sub_h = nullptr;
  const int32_t* sub_w = nullptr;
  cx<T>* u = nullptr;                   // updates: output image (u^{n+1})
  const cx<T>* u_in = nullptr;          // updates: u^n when not in place (nullptr: u)
  const T* denom = nullptr;             // nonblind: eta*rho + r*npairs (< 0: pinned)
  const T* rpen = nullptr;              // blind: r*npairs (< 0: pinned)
  const int32_t* sub_pbeg = nullptr;    // CSR over PairSide per subdomain (ascending p)
  const PairSide* ps = nullptr;
  const cx<T>* v = nullptr;
  cx<T>* lam = nullptr;                 // updates: Lambda^{n+1}
  const cx<T>* lam_in = nullptr;        // Lambda^n when not in place (nullptr: lam)
  T eta = T(0), r = T(0), gamma = T(0);
  cx<T>* out = nullptr;                 // adjoint output (image layout)
  double* dens_out = nullptr;           // density output (image layout)
  double* re_part = nullptr;            // [ntiles][2] (diff, norm)
  const int* stop_flag = nullptr;
};

// Overlap pair with both sides' image addressing (for v / s packing).
struct PairGeom {
  int32_t h, w;
  int64_t u_off[2];    // element offset of the overlap's top-left in each side's image buffer (-1: remote side)
  int32_t u_pitch[2];
  int64_t v_off;       // offset into v (and into the s exchange buffers: s[side] = s_off + side*h*w)
  int64_t lam_off[2];
  int64_t s_off;
};

template <typename T>
cudaError_t launch_frame(int mode, int S, const FrameArgs<T>& a, cudaStream_t st);
// blind w-step (average of the D probe tiles -> FFT2 -> mask -> IFFT2 -> w) in one launch;
// cudaErrorNotSupported for shapes without a single-CTA engine
template <typename T>
cudaError_t launch_wstep(int S, const cx<T>* wd_all, int D, const T* mask, const cx<T>* tw, T scale, cx<T>* w,
                         const int* skip, cudaStream_t st);
template <typename T>
int sweep_stream_ctas(int S);  // persistent grid of the streamed SWEEP kernel (0: not streamed)
template <typename T>
size_t stream_scratch_bytes(int S);  // global transpose tiles the streamed kernels need (0: none)
template <typename T>
bool frame_supported(int S);

template <typename T>
cudaError_t launch_gather(const GatherArgs<T>& a, cudaStream_t st);

// s_{p,side} = u_side|overlap + Lambda_{p,side} for the sides present locally.
template <typename T>
cudaError_t launch_pack(const PairGeom* pairs, int npairs, int maxpix, const cx<T>* u, const cx<T>* lam,
                        cx<T>* s, const int* stop_flag, cudaStream_t st);
// v_p = 0.5 * (s_{p,0} + s_{p,1})
template <typename T>
cudaError_t launch_vstep(const PairGeom* pairs, int npairs, int maxpix, const cx<T>* s, cx<T>* v,
                         const int* stop_flag, cudaStream_t st);

template <typename T>
cudaError_t launch_fill(cx<T>* p, int64_t n, cx<T> value, cudaStream_t st);

// merge (ddplan.cpp:104-121) on the device: mean over covering subdomains,
// vacuum 1 elsewhere; subdomain rects [D][4] (r0,r1,c0,c1) with image offsets.
template <typename T>
cudaError_t launch_merge(const cx<T>* u, const int64_t* sub_rect, const int64_t* sub_off, int D, int64_t H, int64_t W,
                         cx<double>* out, cudaStream_t st);
// scan_coverage (scan.cpp:36-44) of one subdomain from its gather tiles -> pins.
cudaError_t launch_pins(const int4* tiles, int ntiles, int tile_h, int tile_w, const int32_t* tile_frames,
                        const int32_t* fr_r, const int32_t* fr_c, int S, const int64_t* sub_off, const int32_t* sub_h,
                        const int32_t* sub_w, const uint8_t* user_pin, uint8_t* pin, cudaStream_t st);

// complex64 -> complex128 on the device (state downloads without host loops)
cudaError_t launch_widen_cx(const cx<float>* in, cx<double>* out, int64_t n, cudaStream_t st);

// Deterministic segmented sums: out[map[s]] = sum_{i in [beg[s], beg[s+1])} in[i*stride+comp]
// (fixed tree; map == nullptr means identity).  Skipped when *skip != 0.
cudaError_t launch_segsum(const double* in, int stride, int comp, const int64_t* beg, int nseg, const int* map,
                          double* out, const int* skip, cudaStream_t st);

// Augmented Lagrangian (metrics.cpp:73-101): per-frame terms [nfr] and
// per-(local pair, side) overlap terms [2 npairs], fp64.
template <typename T>
cudaError_t launch_lagrangian_frames(const cx<T>* au, const cx<T>* z, const cx<T>* gamma, const T* amp, int64_t nfr,
                                     int64_t per, double eps, double eta, double* out, cudaStream_t st);
template <typename T>
cudaError_t launch_lagrangian_pairs(const PairGeom* pairs, int npairs, const cx<T>* u, const cx<T>* v,
                                    const cx<T>* lam, double r, double* out, cudaStream_t st);

// Per-frame sums of amplitudes (for the R-factor denominator), double.
template <typename T>
cudaError_t launch_frame_sums(const T* amp, int64_t nfr, int64_t per, double* out, cudaStream_t st);

// amp[i] = sqrt(src) (kind 0: f64 intensity) or src (kind 1: f32 amplitude, kind 2: f64 amplitude);
// negative inputs are counted into *neg (FrameStack::validate, scan.cpp:46-56).
template <typename T>
cudaError_t launch_scatter_amp(const double* src, int64_t g0, int64_t count, int64_t per, const int32_t* glob2loc,
                               T* amp, unsigned long long* neg, cudaStream_t st);
template <typename T>
cudaError_t launch_convert_amp(const void* src, int kind, T* amp, int64_t n, unsigned long long* neg,
                               cudaStream_t st);

// Denominators for one subdomain: d = eta*rho (+ r per covering pair side); pinned -> -1;
// counts interior pixels with rho <= 0 into *bad.  (solver.cpp:53-75)
template <typename T>
cudaError_t launch_denom_sub(const double* dens, const uint8_t* pin, const PairSide* ps, int nps, int H, int W,
                             T eta, T r, T* denom, unsigned long long* bad, cudaStream_t st);
// Blind penalty: rpen = r per covering pair side, pinned -> -1 (blind.cpp:100-107).
template <typename T>
cudaError_t launch_rpen_sub(const uint8_t* pin, const PairSide* ps, int nps, int H, int W, T r, T* rpen,
                            cudaStream_t st);

// Iteration control (device-side stop logic; see nonblind.cpp).
struct RunCtl {
  int iter;      // completed iterations (state is u^iter)
  int stop;      // 0 or the final iteration
  int done;      // final R-factor recorded
  int diverged;  // iteration at which a non-finite RF/RE appeared
  int max_iters;
  int rule;      // 0: R-factor, 1: relative error
  int skipA;     // frame pass disabled
  int skipB;     // update pass disabled
  int rec_cap;   // records ring capacity (iterations)
  int skipC;     // stop from earlier iterations only (set by the gate): the forked consensus branch
  double tol_rf, tol_re, l1;
};
cudaError_t launch_gate(RunCtl* c, cudaStream_t st);
cudaError_t launch_rf_finalize(RunCtl* c, const double* rf_sub, int D, double* rec, cudaStream_t st);
cudaError_t launch_re_finalize(RunCtl* c, const double* diff, const double* norm, int D, double* rec,
                               cudaStream_t st);
// segsum + finalize in one launch (single-rank solvers, D <= fused_finalize_max_subdomains()):
// ncomp 1 = R-factor (out0), 2 = RE (out0 = diff, out1 = norm); counter: a zeroed device word
cudaError_t launch_segsum_finalize(int ncomp, const double* in, const int64_t* beg, int nseg, const int* map,
                                   double* out0, double* out1, const int* skip, unsigned* counter, RunCtl* c, int D,
                                   double* rec, cudaStream_t st);
int fused_finalize_max_subdomains();

}  // namespace pdd
