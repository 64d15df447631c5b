/*
 * ptychodd_cuda.h -- C-ABI of the B200-native OD²P hot path.
 *
 * Drop-in boundary for the reference C++ API of arXiv 2011.00162 "ptychodd"
 * (/root/reference/proj/include/ptychodd/*.hpp).  Plain pointers and sizes
 * only; no exception crosses this boundary.  Every function returns a status:
 *   PDD_OK 0, PDD_INVALID_ARGUMENT 1 (std::invalid_argument),
 *   PDD_OUT_OF_RANGE 2 (std::out_of_range), PDD_RUNTIME_ERROR 3
 *   (std::runtime_error), PDD_DIVERGENCE 4 (ptychodd::DivergenceError,
 *   solver.hpp:62-68; iteration index via the out-parameter), PDD_CUDA_ERROR 5,
 *   PDD_FORMAT_ERROR 6 (ptychodd::FormatError, io.hpp:12-18)
 * and pdd_last_error() returns the thread-local message.  A C++ or Python shim
 * rethrows the reference's exception types from these codes.
 *
 * Data conventions (the reference's, field.hpp:48-91):
 *   complex arrays: interleaved (re, im) float64 pairs, row-major;
 *   frame stacks:   [J][s][s] in scan order (scan.hpp:38-43, packed);
 *   solver state:   per owned subdomain in ascending d: images [H_d][W_d];
 *                   frames [J_d][s][s] in frames_of order; overlap variables
 *                   per pair in ascending p; Lambda side 0 then side 1
 *                   (solver.hpp:41-51).
 * Precision: dtype PDD_F32 computes in float/complex64 (amplitudes stored as
 * float), PDD_F64 in double/complex128.
 */
#ifndef PTYCHODD_CUDA_H
#define PTYCHODD_CUDA_H

#include <stdint.h>

#if defined(__GNUC__)
#define PDD_API __attribute__((visibility("default")))
#else
#define PDD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PDD_OK = 0,
  PDD_INVALID_ARGUMENT = 1,
  PDD_OUT_OF_RANGE = 2,
  PDD_RUNTIME_ERROR = 3,
  PDD_DIVERGENCE = 4,
  PDD_CUDA_ERROR = 5,
  PDD_FORMAT_ERROR = 6 /* ptychodd::FormatError (io.hpp:12-18): malformed PTYA input */
};
enum { PDD_F32 = 1, PDD_F64 = 2 };
enum { PDD_AXIS_AUTO = 0, PDD_AXIS_COLUMNS = 1, PDD_AXIS_ROWS = 2 }; /* ddplan.hpp:7 SplitAxis */
enum { PDD_STOP_RFACTOR = 0, PDD_STOP_RELATIVE_ERROR = 1 };           /* solver.hpp:11-14 StopRule */
/* Measured data handed to the solver constructors: a [J][s][s] array in global
 * scan order, or (PDD_DATA_PTYA_FRAMES_F64, host only) `data` is the
 * NUL-terminated path of a frames.ptya stack of float64 intensities -- the
 * file the reference's CLI loads with read_frames (io.cpp:186-202) -- streamed
 * from disk through page-locked chunks to the device, where it is converted to
 * amplitudes; validated like read_frames + FrameStack::validate. */
enum { PDD_DATA_INTENSITY_F64 = 0, PDD_DATA_AMPLITUDE_F32 = 1, PDD_DATA_AMPLITUDE_F64 = 2,
       PDD_DATA_PTYA_FRAMES_F64 = 3 };

PDD_API const char* pdd_last_error(void);
PDD_API int pdd_version(void);
PDD_API int pdd_device_count(int32_t* n);

/* ---- scan geometry and decomposition plans (host integer work) ----------
 * pdd_plan_stripes   <- make_raster_scan (scan.hpp:31-33) + plan_stripes (ddplan.hpp:37-41)
 * pdd_plan_grid      <- 2-D block plan (extension; configs 2 and 3)
 * pdd_plan_from_arrays <- any DecompositionPlan (ddplan.hpp:12-35) given as arrays */
typedef struct pdd_plan pdd_plan;
typedef struct {
  int64_t frame_side, step, image_height, image_width, grid_rows, grid_cols, n_frames;
  int32_t n_sub, n_pairs;
} pdd_plan_info;

PDD_API int pdd_plan_stripes(int64_t image_height, int64_t image_width, int64_t frame_side, int64_t step, int32_t D,
                     int32_t axis, pdd_plan** out);
PDD_API int pdd_plan_grid(int64_t image_height, int64_t image_width, int64_t frame_side, int64_t step, int32_t Dr,
                  int32_t Dc, pdd_plan** out);
PDD_API int pdd_plan_from_arrays(int64_t frame_side, int64_t step, int64_t image_height, int64_t image_width,
                         int64_t n_frames, const int64_t* positions, int32_t D, const int32_t* assignment,
                         const int64_t* subdomains, int32_t n_pairs, const int32_t* pairs, const int64_t* regions,
                         pdd_plan** out);
PDD_API int pdd_plan_info_get(const pdd_plan* plan, pdd_plan_info* info);
/* positions [J][2], assignment [J], subdomains [D][4] (r0,r1,c0,c1), pairs [P][2] (d1<d2),
 * regions [P][4], local_grid [D][2]; any pointer may be NULL. */
PDD_API int pdd_plan_arrays(const pdd_plan* plan, int64_t* positions, int32_t* assignment, int64_t* subdomains,
                    int32_t* pairs, int64_t* regions, int64_t* local_grid);
PDD_API int pdd_plan_destroy(pdd_plan* plan);
/* Host-only: one rank's share of a plan -- owned subdomains (d with floor(d*world/D) == rank),
 * pairs touching them (ascending p), and the NCCL exchange schedule: one (local pair index,
 * peer rank, my side) triple per cut pair.  Arrays sized D, n_pairs, n_pairs*3. */
PDD_API int pdd_rank_layout(const pdd_plan* plan, int32_t rank, int32_t world, int32_t* n_local_sub,
                            int32_t* local_subs, int32_t* n_local_pairs, int32_t* local_pairs, int32_t* n_exchange,
                            int32_t* exchange);
/* scan_coverage (scan.hpp:35-36): int32 [H][W] */
PDD_API int pdd_scan_coverage(const pdd_plan* plan, int32_t* out);

/* ---- operators on host buffers ------------------------------------------- */
/* fft2_normalized / ifft2_normalized (fft.hpp:8-15): unitary, in place */
PDD_API int pdd_fft2(double* data, int64_t h, int64_t w, int32_t inverse, int32_t dtype);
/* forward (forward.hpp:8-10): frames_out [J][s][s] c128 (may be NULL); intensity_out [J][s][s] f64
 * (intensity(), forward.hpp:26-27; may be NULL) */
PDD_API int pdd_forward(const double* probe, int64_t s, const double* image, int64_t H, int64_t W, const int64_t* positions,
                int64_t J, double* frames_out, double* intensity_out, int32_t dtype);
/* adjoint (forward.hpp:12-14) */
PDD_API int pdd_adjoint(const double* probe, int64_t s, const double* frames, const int64_t* positions, int64_t J,
                int64_t H, int64_t W, double* image_out, int32_t dtype);
/* illumination_density (forward.hpp:16-17): f64 [H][W] */
PDD_API int pdd_illumination_density(const double* probe, int64_t s, const int64_t* positions, int64_t J, int64_t H,
                             int64_t W, double* out, int32_t dtype);
/* adjoint_probe (forward.hpp:22-24) -> num [s][s] c128 and probe_density (forward.hpp:19-20) -> den [s][s];
 * frames may be NULL (density only). */
PDD_API int pdd_probe_sums(const double* image, int64_t H, int64_t W, const double* frames, const int64_t* positions,
                   int64_t J, int64_t s, double* num_out, double* den_out, int32_t dtype);
/* simulate_frames (simulate.hpp:56-58) on the device: intensity |F(probe o image|w_j)|^2 of every
 * window, written as float64 [J][s][s] into DEVICE memory intensity_dev (input synthesis for
 * large configurations). */
PDD_API int pdd_simulate_intensity_device(const double* probe, int64_t s, const double* image, int64_t H, int64_t W,
                                          const int64_t* positions, int64_t J, double* intensity_dev, int32_t dtype);
/* intensity of n complex values */
PDD_API int pdd_intensity(const double* z, int64_t n, double* out, int32_t dtype);
/* stagm::pixel_prox over n pixels (stagm.hpp:26-29; b = intensity) */
PDD_API int pdd_stagm_prox(const double* y, const double* b, int64_t n, double lambda, double epsilon, double* out,
                   int32_t dtype);
/* stagm::pixel_value / pixel_gradient (stagm.hpp:19-24) */
PDD_API int pdd_stagm_value_gradient(const double* x, const double* b, int64_t n, double epsilon, double* value,
                             double* gradient, int32_t dtype);
/* r_factor (metrics.hpp:9-10): subs = local images concatenated in d order, intensities [J][s][s] */
PDD_API int pdd_r_factor(const pdd_plan* plan, const double* subs, const double* intensities, const double* probe,
                 double* out, int32_t dtype);
/* relative_error (metrics.hpp:12-14) over D images given as one concatenation + sizes */
PDD_API int pdd_relative_error(const double* current, const double* previous, int32_t D, const int64_t* sizes, double* out,
                       int32_t dtype);
/* merge (ddplan.hpp:47-50): host, exact */
PDD_API int pdd_merge(const pdd_plan* plan, const double* subs, double* out);

/* ---- nonblind OD²P solver (solver.hpp:72-107) ----------------------------- */
typedef struct {
  double epsilon, eta, r, tol_rf, tol_re;
  int32_t max_iters, stop_rule, record_lagrangian, threads;
} pdd_nonblind_config;

typedef struct pdd_nonblind pdd_nonblind;

/* NonblindSolver(plan, frames, probe, config, pin_ones): data [J][s][s] of data_kind in
 * global scan order (host memory unless data_on_device); probe [s][s] c128; pin_ones
 * [H][W] f64 or NULL.  device = CUDA ordinal.
 * Ordering contract for data_on_device: the solver copies the data on its own
 * stream, which is not ordered after the caller's streams -- every write to the
 * buffer must be complete (e.g. cudaStreamSynchronize of the producing stream)
 * before the call.  The buffer may be reused or freed when the call returns. */
PDD_API int pdd_nonblind_create(const pdd_plan* plan, const void* data, int32_t data_kind, int32_t data_on_device,
                        const double* probe, const pdd_nonblind_config* cfg, const double* pin_ones, int32_t dtype,
                        int32_t device, pdd_nonblind** out);
/* Rank-sharded variant: this process owns subdomains d with floor(d*world/D) == rank and
 * exchanges overlap strips with NCCL.  nccl_id: 128 bytes from pdd_nccl_unique_id on rank 0. */
PDD_API int pdd_nccl_unique_id(void* out128);
PDD_API int pdd_nonblind_create_rank(const pdd_plan* plan, const void* data, int32_t data_kind, int32_t data_on_device,
                             const double* probe, const pdd_nonblind_config* cfg, const double* pin_ones,
                             int32_t dtype, int32_t device, int32_t rank, int32_t world, const void* nccl_id,
                             pdd_nonblind** out);
/* One handle driving n_devices ranks of this process -- the reference's worker
 * pool (NonblindConfig::threads, solver.hpp:25; WorkerPool, parallel.hpp:14-90)
 * mapped onto GPUs: rank r on devices[r] owns subdomains d with
 * floor(d*n_devices/D) == r (n_devices <= D), each rank on its own host thread,
 * stream and CUDA graphs; NCCL between distinct devices, the in-process host
 * transport when a device repeats (several ranks on one GPU: the multi-rank
 * code path without NCCL).  Iterates are bit-identical for every n_devices at
 * fixed D.  State arrays use the single-handle layout above. */
PDD_API int pdd_nonblind_create_multi(const pdd_plan* plan, const void* data, int32_t data_kind,
                                      int32_t data_on_device, const double* probe, const pdd_nonblind_config* cfg,
                                      const double* pin_ones, int32_t dtype, const int32_t* devices,
                                      int32_t n_devices, pdd_nonblind** out);
/* PTYA header (io.cpp:80-115): dtype code to expect (1 f64, 2 c128), ndim,
 * dims (up to 4, zero-padded), payload byte offset.  PDD_FORMAT_ERROR with the
 * byte offset in the message on malformed input. */
PDD_API int pdd_ptya_header(const char* path, int32_t want_dtype, int32_t* ndim, int64_t* dims4,
                            int64_t* payload_offset);
/* A 128-byte id for the in-process host transport, usable in place of an NCCL
 * id by pdd_*_create_rank when the ranks are threads of one process (tests of
 * the rank-sharded path on one device).  No reference counterpart. */
PDD_API int pdd_host_transport_id(void* out128);
/* Sizes of the state arrays held by this handle (complex element counts). */
typedef struct {
  int32_t n_local_sub, n_local_pairs;
  int64_t frame_side, image_elems, frame_elems, v_elems, lambda_elems;
} pdd_nonblind_layout;
PDD_API int pdd_nonblind_layout_get(const pdd_nonblind* h, pdd_nonblind_layout* out);
/* local_subs [n_local_sub], sub_hw [n_local_sub][2], sub_frames [n_local_sub],
 * local_pairs [n_local_pairs], pair_hw [n_local_pairs][2] */
PDD_API int pdd_nonblind_layout_arrays(const pdd_nonblind* h, int32_t* local_subs, int64_t* sub_hw, int64_t* sub_frames,
                               int32_t* local_pairs, int64_t* pair_hw);
PDD_API int pdd_nonblind_init_state(pdd_nonblind* h);                  /* solver.cpp:96-116 */
PDD_API int pdd_nonblind_step(pdd_nonblind* h, int32_t store_z);       /* solver.cpp:118-205 */
/* run() (solver.cpp:216-267) from a fresh init_state.  records: [max_iters][3] (rf, re, t_ms);
 * returns PDD_DIVERGENCE with *diverged_at set if RF/RE became non-finite. */
PDD_API int pdd_nonblind_run(pdd_nonblind* h, int64_t* iterations, double* records, int64_t* diverged_at);
/* run() with the reference's per-iteration callback (solver.hpp:88
 * on_iteration): cb(iteration, rf, re, t_ms, lagrangian, user) is called on the
 * calling thread while the device loop runs -- in order, once per iteration,
 * at most one poll window (16 iterations) behind the device, never for
 * iterations a stop rule rolls back.  lagrangian is NaN unless
 * record_lagrangian.  cb may be NULL (== pdd_nonblind_run).  It runs on the
 * thread that drives the device loop: the caller's, or rank 0's worker thread
 * for pdd_nonblind_create_multi handles. */
typedef void (*pdd_record_cb)(int64_t iteration, double rf, double re, double t_ms, double lagrangian, void* user);
PDD_API int pdd_nonblind_run_cb(pdd_nonblind* h, pdd_record_cb cb, void* user, int64_t* iterations, double* records,
                                int64_t* diverged_at);
/* Exactly n iterations from the current state (no stop rule, no host round trip). */
PDD_API int pdd_nonblind_iterate(pdd_nonblind* h, int32_t n);
/* Same, reporting the device time of the n iterations (CUDA events on the solver stream). */
PDD_API int pdd_nonblind_iterate_timed(pdd_nonblind* h, int32_t n, double* ms);
/* n eager iterations with CUDA events around the kernels: ms[3] = {frame kernel, gather kernel,
 * whole iteration} averages (roofline accounting). */
PDD_API int pdd_nonblind_profile(pdd_nonblind* h, int32_t n, double* ms);
PDD_API int pdd_nonblind_last_rf(pdd_nonblind* h, double* rf);
PDD_API int pdd_nonblind_get_state(pdd_nonblind* h, double* u, double* z, double* gamma, double* v, double* lambda,
                           int64_t* iteration);
PDD_API int pdd_nonblind_set_state(pdd_nonblind* h, const double* u, const double* z, const double* gamma, const double* v,
                           const double* lambda, int64_t iteration);
/* A_d u_d of the current iterate for the local frames ([J_local][s][s] c128) */
PDD_API int pdd_nonblind_forward(pdd_nonblind* h, double* au);
/* augmented_lagrangian (metrics.hpp:16-19, metrics.cpp:73-101) of the handle's current state
 * (u, z, Gamma, v, Lambda) with au = A u recomputed on the device.  Needs a stored z (init_state,
 * set_state with z, or step with store_z); otherwise PDD_INVALID_ARGUMENT.  Collective over ranks. */
PDD_API int pdd_nonblind_lagrangian(pdd_nonblind* h, double* out);
/* ConvergenceRecord::lagrangian history of the last run() with record_lagrangian (solver.cpp:258-260):
 * copies min(cap, n) values, *n = recorded count (0 when record_lagrangian was off). */
PDD_API int pdd_nonblind_lagrangian_history(pdd_nonblind* h, double* out, int64_t cap, int64_t* n);
/* merge() of the current sub-solutions on the device -> host [H][W] c128 (single-rank handles) */
PDD_API int pdd_nonblind_merged(pdd_nonblind* h, double* out);
PDD_API int pdd_nonblind_sync(pdd_nonblind* h);
PDD_API int pdd_nonblind_launches_per_iteration(const pdd_nonblind* h, int64_t* n);
PDD_API int pdd_nonblind_destroy(pdd_nonblind* h);

/* ---- blind OD²BP solver (blind.hpp:58-85) --------------------------------- */
typedef struct {
  double epsilon, eta, r, mu, gamma, support_energy, tol_rf, tol_re;
  int32_t max_iters, stop_rule, threads;
} pdd_blind_config;

typedef struct pdd_blind pdd_blind;

/* BlindSolver(plan, frames, config, pin_ones); support_mask [s][s] 0/1 or NULL (estimate). */
PDD_API int pdd_blind_create(const pdd_plan* plan, const void* data, int32_t data_kind, int32_t data_on_device,
                     const pdd_blind_config* cfg, const double* support_mask, const double* pin_ones, int32_t dtype,
                     int32_t device, pdd_blind** out);
PDD_API int pdd_blind_create_rank(const pdd_plan* plan, const void* data, int32_t data_kind, int32_t data_on_device,
                          const pdd_blind_config* cfg, const double* support_mask, const double* pin_ones,
                          int32_t dtype, int32_t device, int32_t rank, int32_t world, const void* nccl_id,
                          pdd_blind** out);
/* Multi-device blind handle (see pdd_nonblind_create_multi). */
PDD_API int pdd_blind_create_multi(const pdd_plan* plan, const void* data, int32_t data_kind, int32_t data_on_device,
                                   const pdd_blind_config* cfg, const double* support_mask, const double* pin_ones,
                                   int32_t dtype, const int32_t* devices, int32_t n_devices, pdd_blind** out);
PDD_API int pdd_blind_layout_get(const pdd_blind* h, pdd_nonblind_layout* out);
/* init_state (blind.cpp:169-192); w0 [s][s] c128 replaces the amplitude-based initial probe, or NULL */
PDD_API int pdd_blind_init_state(pdd_blind* h, const double* w0);
PDD_API int pdd_blind_step(pdd_blind* h, int32_t store_z);
/* run() from the current state; records [max_iters][3] */
PDD_API int pdd_blind_run(pdd_blind* h, int64_t* iterations, double* records, int64_t* diverged_at);
/* Blind run() with the per-iteration callback (see pdd_nonblind_run_cb). */
PDD_API int pdd_blind_run_cb(pdd_blind* h, pdd_record_cb cb, void* user, int64_t* iterations, double* records,
                             int64_t* diverged_at);
PDD_API int pdd_blind_iterate(pdd_blind* h, int32_t n);
/* device time of exactly n iterations (CUDA events on the solver stream) */
PDD_API int pdd_blind_iterate_timed(pdd_blind* h, int32_t n, double* ms);
/* n eager iterations: ms[3] = {BLIND frame kernel, u-gather, whole iteration} averages */
PDD_API int pdd_blind_profile(pdd_blind* h, int32_t n, double* ms);
/* w, w_copies [D_local][s][s], delta [D_local][s][s], then as nonblind */
PDD_API int pdd_blind_get_state(pdd_blind* h, double* w, double* w_copies, double* delta, double* u, double* z,
                        double* gamma, double* v, double* lambda, int64_t* iteration);
PDD_API int pdd_blind_set_state(pdd_blind* h, const double* w, const double* w_copies, const double* delta,
                                const double* u, const double* z, const double* gamma, const double* v,
                                const double* lambda, int64_t iteration);
/* result.probe / probe_fourier (blind.cpp:440), support_mask(), the solver's own w0 */
PDD_API int pdd_blind_get_probe(pdd_blind* h, double* probe, double* probe_fourier, double* mask, double* w0);
PDD_API int pdd_blind_merged(pdd_blind* h, double* out);
PDD_API int pdd_blind_sync(pdd_blind* h);
PDD_API int pdd_blind_launches_per_iteration(const pdd_blind* h, int64_t* n);
PDD_API int pdd_blind_destroy(pdd_blind* h);

/* disk_support_mask (blind.hpp:47-48): centred disk in wrapped Fourier coordinates, out [side][side] */
PDD_API int pdd_disk_support_mask(int64_t side, double radius, double* out);
/* estimate_support_mask (blind.hpp:50-52): smallest centred disk holding energy_fraction of the
 * Fourier energy of probe_guess [side][side] c128 (FFT on the device); out [side][side] */
PDD_API int pdd_estimate_support_mask(const double* probe_guess, int64_t side, double energy_fraction, double* out);

/* ---- pinned host memory for end-to-end staging ----------------------------- */
PDD_API int pdd_host_alloc(void** p, int64_t bytes);
PDD_API int pdd_host_free(void* p);
/* Reserve the library's page-locked download staging buffer now (idempotent).
 * Large results (sub-solutions, merged image, state) are copied out through it
 * by several host threads; the Python front end calls this on its helper thread
 * while the device loop of run() executes, so the first download does not pay
 * for the allocation.  No reference counterpart (reference results are host
 * values already). */
PDD_API int pdd_host_stage_reserve(void);
/* Device memory is drawn from a library-private stream-ordered pool per device
 * whose freed blocks stay mapped for the next solver (repeated solves skip the
 * page mapping of multi-GB buffers); the device's default pool and other
 * allocators in the process are untouched.  This returns every unused block
 * of every pool to the driver now (synchronises the devices used); with
 * PDD_POOL_TRIM_ON_IDLE=1 it happens automatically when the last solver on a
 * device is destroyed.  No reference counterpart. */
PDD_API int pdd_release_cached_memory(void);

#ifdef __cplusplus
}
#endif

#endif /* PTYCHODD_CUDA_H */
