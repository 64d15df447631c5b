// NCCL transport for the multi-GPU OD²P iteration.
//
// The reference has no distributed backend: its workers read the neighbour's
// overlap strip straight out of shared memory (solver.cpp:145-146,186-187).
// Across GPUs the same data flow is one grouped ncclSend/ncclRecv of
// s_d = pi u_d + Lambda_d per cut overlap pair and one all-reduce of the
// per-subdomain (RF, RE) partial sums -- both enqueued on the solver stream so
// they are captured in the iteration's CUDA graph.  NCCL is resolved with
// dlopen at communicator creation, so single-GPU use never loads it; whichever
// libnccl.so.2 torch already mapped is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "device.hpp"
#include "engine.hpp"

namespace pdd {
namespace {

struct NcclApi {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;

  // Resolved once per process (thread-safe); a failed resolution leaves no
  // half-initialised table behind and is reported again on every use.
  static NcclApi& get() {
    static NcclApi api;
    static std::string failure;
    static std::once_flag once;
    std::call_once(once, [] {
      try {
        api.load();
      } catch (const std::exception& e) {
        failure = e.what();
      }
    });
    if (!failure.empty()) throw RuntimeError(failure);
    return api;
  }
  void load() {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) throw RuntimeError(std::string("NCCL unavailable: ") + dlerror());
    auto sym = [&](const char* n) {
      void* p = dlsym(lib, n);
      if (!p) {
        dlclose(lib);
        throw RuntimeError(std::string("NCCL symbol missing: ") + n);
      }
      return p;
    };
    get_unique_id = reinterpret_cast<decltype(get_unique_id)>(sym("ncclGetUniqueId"));
    init_rank = reinterpret_cast<decltype(init_rank)>(sym("ncclCommInitRank"));
    destroy = reinterpret_cast<decltype(destroy)>(sym("ncclCommDestroy"));
    group_start = reinterpret_cast<decltype(group_start)>(sym("ncclGroupStart"));
    group_end = reinterpret_cast<decltype(group_end)>(sym("ncclGroupEnd"));
    send = reinterpret_cast<decltype(send)>(sym("ncclSend"));
    recv = reinterpret_cast<decltype(recv)>(sym("ncclRecv"));
    allreduce = reinterpret_cast<decltype(allreduce)>(sym("ncclAllReduce"));
    error_string = reinterpret_cast<decltype(error_string)>(sym("ncclGetErrorString"));
    h = lib;  // published only once every symbol resolved
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + error_string(r));
  }
};

class NcclComm final : public Comm {
 public:
  NcclComm(const void* uid, int rank, int world, int device) : rank_(rank), world_(world) {
    auto& api = NcclApi::get();
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    DeviceGuard g(device);
    api.check(api.init_rank(&comm_, world, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) NcclApi::get().destroy(comm_);
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void group_start() override { NcclApi::get().check(NcclApi::get().group_start(), "ncclGroupStart"); }
  void group_end() override { NcclApi::get().check(NcclApi::get().group_end(), "ncclGroupEnd"); }
  void send(const void* buf, size_t bytes, int peer, void* stream) override {
    auto& a = NcclApi::get();
    a.check(a.send(buf, bytes, ncclUint8, peer, comm_, static_cast<cudaStream_t>(stream)), "ncclSend");
  }
  void recv(void* buf, size_t bytes, int peer, void* stream) override {
    auto& a = NcclApi::get();
    a.check(a.recv(buf, bytes, ncclUint8, peer, comm_, static_cast<cudaStream_t>(stream)), "ncclRecv");
  }
  void allreduce_sum_f64(double* buf, size_t n, void* stream) override {
    auto& a = NcclApi::get();
    a.check(a.allreduce(buf, buf, n, ncclFloat64, ncclSum, comm_, static_cast<cudaStream_t>(stream)),
            "ncclAllReduce");
  }
  void allreduce_sum_f32(float* buf, size_t n, void* stream) override {
    auto& a = NcclApi::get();
    a.check(a.allreduce(buf, buf, n, ncclFloat32, ncclSum, comm_, static_cast<cudaStream_t>(stream)),
            "ncclAllReduce");
  }

 private:
  int rank_, world_;
  ncclComm_t comm_ = nullptr;
};

}  // namespace

void nccl_unique_id(void* out128) {
  auto& api = NcclApi::get();
  ncclUniqueId id;
  api.check(api.get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
}

std::unique_ptr<Comm> make_nccl_comm(const void* uid, int rank, int world, int device) {
  if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("comm: bad rank/world");
  return std::make_unique<NcclComm>(uid, rank, world, device);
}

}  // namespace pdd
