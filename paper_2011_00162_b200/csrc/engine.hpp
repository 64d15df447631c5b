// C++ host drivers of the OD²P iteration (the layer between the C-ABI and the
// kernels).  Semantics follow the reference solvers:
//   NonblindSolver (proj/include/ptychodd/solver.hpp:72-107, solver.cpp)
//   BlindSolver    (proj/include/ptychodd/blind.hpp:58-85, blind.cpp)
// with the WorkerPool (parallel.hpp:14-90) replaced by one CUDA stream per
// rank, one CUDA graph per iteration pair, and NCCL for the overlap-strip
// exchange when subdomains are spread over several GPUs.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

#include "plan.hpp"

namespace pdd {

struct NonblindConfig {  // solver.hpp:16-28
  double epsilon = 0.5, eta = 0.1, r = 4.0e3, tol_rf = 1.0e-5, tol_re = 1.0e-3;
  int32_t max_iters = 1000, stop_rule = 0, record_lagrangian = 0, threads = 0;
  void validate() const;
};

struct BlindConfig {  // blind.hpp:7-22
  double epsilon = 0.5, eta = 0.1, r = 5.0e3, mu = 2.0e2, gamma = 1.0e-4, support_energy = 0.995;
  double tol_rf = 1.0e-5, tol_re = 1.0e-3;
  int32_t max_iters = 1000, stop_rule = 0, threads = 0;
  void validate(int64_t s, const double* mask) const;
};

enum DataKind { kIntensityF64 = 0, kAmplitudeF32 = 1, kAmplitudeF64 = 2, kPtyaFramesF64 = 3 };

// Frames in global scan order, [J][s][s]; host or device memory -- or, for
// kPtyaFramesF64, ptr is a NUL-terminated path of a frames.ptya file
// (float64 intensities) streamed from disk (ptya.hpp).
struct DataSpec {
  const void* ptr = nullptr;
  int kind = kIntensityF64;
  bool device = false;
};

// Per-iteration record delivered while run() executes (solver.hpp:88
// on_iteration): 1-based iteration, R-factor, relative error, iteration time
// (device ms), augmented Lagrangian (NaN unless record_lagrangian).  Records
// arrive in order, each once, at most a poll window (16 iterations) after the
// device produced them, and never for iterations a stop rule rolls back.
using RecordFn = std::function<void(int64_t iteration, double rf, double re, double t_ms, double lag)>;

struct RunRecords {
  int64_t iterations = 0;
  int64_t diverged_at = 0;  // > 0: non-finite RF/RE at this iteration
  std::vector<double> rf, re, t_ms;
  std::vector<double> lag;  // augmented Lagrangian per iteration (record_lagrangian runs)
};

// Peer transport for the overlap exchange and the scalar all-reduce
// (implemented over NCCL in comm.cpp).  nullptr = single rank.
struct Comm {
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  // Enqueue on `stream`: send/recv complex buffers (elem_bytes per element).
  virtual void group_start() = 0;
  virtual void group_end() = 0;
  virtual void send(const void* buf, size_t bytes, int peer, void* stream) = 0;
  virtual void recv(void* buf, size_t bytes, int peer, void* stream) = 0;
  virtual void allreduce_sum_f64(double* buf, size_t n, void* stream) = 0;
  virtual void allreduce_sum_f32(float* buf, size_t n, void* stream) = 0;
  // false: calls block on the host (they synchronise the stream and wait for
  // peers), so the iteration runs eagerly instead of as a CUDA graph
  virtual bool capturable() const { return true; }
};

std::unique_ptr<Comm> make_nccl_comm(const void* unique_id, int rank, int world, int device);
void nccl_unique_id(void* out128);
// In-process host-staged transport between ranks that are threads of one
// process (any devices, including one device shared by every rank): the
// multi-rank path of the solvers without NCCL, for testing it on one GPU.
// Ranks passing the same hub id form one world.
std::unique_ptr<Comm> make_host_comm(const void* hub_id128, int rank, int world);
void host_hub_id(void* out128);
bool is_host_hub_id(const void* id128);

struct StateLayout {
  std::vector<int> local_subs;        // global subdomain ids owned here
  std::vector<int64_t> sub_h, sub_w;  // per local subdomain
  std::vector<int64_t> sub_frames;    // per local subdomain
  std::vector<int> local_pairs;       // global pair ids with at least one local side
  std::vector<int64_t> pair_h, pair_w;
  int64_t S = 0;
};

class NonblindGpu {
 public:
  virtual ~NonblindGpu() = default;
  virtual const StateLayout& layout() const = 0;
  virtual void init_state() = 0;
  // One iteration (solver.cpp:118-205).  store_z keeps z for get_state.
  virtual void step(bool store_z) = 0;
  // Config-driven solve from the current state (solver.cpp:216-267), stop rules on device.
  virtual RunRecords run(const RecordFn& on_record = {}) = 0;
  // Exactly n iterations from the current state, no stop rule (benchmark path).
  virtual void iterate(int n) = 0;
  // Same, returning the device time (CUDA events on the solver stream) in ms.
  virtual double iterate_timed(int n) = 0;
  // n eager iterations with CUDA events around each kernel on the solver stream:
  // ms[0] frame kernel, ms[1] gather kernel, ms[2] whole iteration (averages).
  virtual void profile(int n, double* ms) = 0;
  virtual double last_rf() = 0;  // R-factor of the current iterate
  // State transfer (reference layout: complex128 interleaved; see StateLayout).
  virtual void get_state(double* u, double* z, double* gamma, double* v, double* lam, int64_t* iteration) = 0;
  virtual void set_state(const double* u, const double* z, const double* gamma, const double* v, const double* lam,
                         int64_t iteration) = 0;
  virtual void forward_frames(double* au) = 0;  // A_d u_d for the local frames
  // Augmented Lagrangian (metrics.cpp:73-101) of the current state; needs z
  // (init_state, set_state with z, or step with store_z).
  virtual double lagrangian() = 0;
  // Per-iteration values recorded by the last run() with record_lagrangian.
  virtual std::vector<double> lagrangian_history() const = 0;
  virtual void merged(double* out) = 0;         // merge() of the current sub-solutions (single rank)
  virtual void sync() = 0;
  virtual void* stream() const = 0;  // cudaStream_t of this rank's work
  virtual int64_t kernel_launches_per_iteration() const = 0;
};

// disk_support_mask / estimate_support_mask (blind.cpp:46-75): [side][side] 0/1;
// the estimate's spectrum comes from the GPU FFT.
std::vector<double> disk_mask(int64_t side, double radius);
std::vector<double> estimate_mask(const std::vector<double>& w0, int64_t side, double frac);

std::unique_ptr<NonblindGpu> make_nonblind(const Plan& plan, const DataSpec& data, const double* probe,
                                           const NonblindConfig& cfg, const double* pin_ones, int dtype,
                                           int device, Comm* comm);

class BlindGpu {
 public:
  virtual ~BlindGpu() = default;
  virtual const StateLayout& layout() const = 0;
  virtual void init_state(const double* w0) = 0;  // nullptr: the solver's amplitude-based w0
  virtual void step(bool store_z) = 0;
  virtual RunRecords run(const RecordFn& on_record = {}) = 0;
  virtual void iterate(int n) = 0;
  virtual double iterate_timed(int n) = 0;          // device ms of exactly n iterations
  virtual void profile(int n, double* ms) = 0;      // {frame kernel, u-gather, iteration} averages
  virtual void get_state(double* w, double* w_copies, double* delta, double* u, double* z, double* gamma, double* v,
                         double* lam, int64_t* iteration) = 0;
  virtual void set_state(const double* w, const double* w_copies, const double* delta, const double* u,
                         const double* z, const double* gamma, const double* v, const double* lam,
                         int64_t iteration) = 0;
  virtual void get_probe(double* probe, double* probe_fourier, double* mask, double* w0) = 0;
  virtual void merged(double* out) = 0;
  virtual void sync() = 0;
  virtual void* stream() const = 0;  // cudaStream_t of this rank's work
  virtual int64_t kernel_launches_per_iteration() const = 0;
};

std::unique_ptr<BlindGpu> make_blind(const Plan& plan, const DataSpec& data, const BlindConfig& cfg,
                                     const double* mask, const double* pin_ones, int dtype, int device, Comm* comm);

// One handle over G = devices.size() ranks of this process (multi.cpp): rank
// r on devices[r], NCCL between distinct devices, the host transport when a
// device repeats.  State in the single-handle layout.
std::unique_ptr<NonblindGpu> make_nonblind_multi(const Plan& plan, const DataSpec& data, const double* probe,
                                                 const NonblindConfig& cfg, const double* pin_ones, int dtype,
                                                 const std::vector<int>& devices);
std::unique_ptr<BlindGpu> make_blind_multi(const Plan& plan, const DataSpec& data, const BlindConfig& cfg,
                                           const double* mask, const double* pin_ones, int dtype,
                                           const std::vector<int>& devices);

}  // namespace pdd
