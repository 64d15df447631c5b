// Host-staged in-process transport (engine.hpp make_host_comm).
//
// Ranks are threads of one process; each call first drains the caller's
// stream, then moves bytes through host memory: send posts a message into the
// (src, dst) mailbox and returns, recv waits for the matching message (per
// (src, dst) pair messages are matched in posting order, which both sides
// produce in ascending global pair order, layout.cpp), all-reduce waits for
// every rank and sums the contributions in rank order.  The solver kernels of
// different ranks never wait on one another -- only the host threads do -- so
// every rank may share one device.  It exists to run the product's
// multi-rank code (cut-pair exchange, D-vector reductions, the stop-rule
// agreement) on one GPU; NCCL (comm.cpp) is the transport between GPUs.
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <tuple>
#include <vector>

#include "device.hpp"
#include "engine.hpp"

namespace pdd {
namespace {

constexpr char kMagic[8] = {'P', 'D', 'D', 'H', 'O', 'S', 'T', '1'};

struct Hub {
  explicit Hub(int w) : world(w), seq_send(w * w, 0), seq_recv(w * w, 0), contrib(w) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::tuple<int, int, uint64_t>, std::vector<char>> box;  // (src, dst, seq) -> bytes
  std::vector<uint64_t> seq_send, seq_recv;                         // [src * world + dst]
  // all-reduce rounds
  std::vector<std::vector<char>> contrib;
  int arrived = 0;
  uint64_t round = 0;
  std::vector<double> result_f64;
  std::vector<float> result_f32;
};

std::mutex g_reg_mu;
std::map<uint64_t, std::weak_ptr<Hub>> g_hubs;

std::shared_ptr<Hub> hub_for(uint64_t key, int world) {
  std::lock_guard<std::mutex> lock(g_reg_mu);
  auto& w = g_hubs[key];
  auto h = w.lock();
  if (!h) {
    h = std::make_shared<Hub>(world);
    w = h;
  } else if (h->world != world) {
    throw InvalidArgument("host transport: ranks of one hub disagree on the world size");
  }
  return h;
}

class HostComm final : public Comm {
 public:
  HostComm(std::shared_ptr<Hub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {}
  int rank() const override { return rank_; }
  int world() const override { return hub_->world; }
  bool capturable() const override { return false; }
  void group_start() override {}
  void group_end() override {}

  void send(const void* buf, size_t bytes, int peer, void* stream) override {
    auto st = static_cast<cudaStream_t>(stream);
    std::vector<char> msg(bytes);
    if (bytes) PDD_CUDA(cudaMemcpyAsync(msg.data(), buf, bytes, cudaMemcpyDeviceToHost, st));
    PDD_CUDA(cudaStreamSynchronize(st));
    std::lock_guard<std::mutex> lock(hub_->mu);
    const uint64_t seq = hub_->seq_send[rank_ * world() + peer]++;
    hub_->box[{rank_, peer, seq}] = std::move(msg);
    hub_->cv.notify_all();
  }

  void recv(void* buf, size_t bytes, int peer, void* stream) override {
    auto st = static_cast<cudaStream_t>(stream);
    std::vector<char> msg;
    {
      std::unique_lock<std::mutex> lock(hub_->mu);
      const uint64_t seq = hub_->seq_recv[peer * world() + rank_]++;
      const auto key = std::make_tuple(peer, rank_, seq);
      hub_->cv.wait(lock, [&] { return hub_->box.count(key) != 0; });
      msg = std::move(hub_->box[key]);
      hub_->box.erase(key);
    }
    if (msg.size() != bytes) throw RuntimeError("host transport: message size mismatch");
    if (bytes) PDD_CUDA(cudaMemcpyAsync(buf, msg.data(), bytes, cudaMemcpyHostToDevice, st));
    PDD_CUDA(cudaStreamSynchronize(st));  // msg is released on return
  }

  void allreduce_sum_f64(double* buf, size_t n, void* stream) override { allreduce(buf, n, stream); }
  void allreduce_sum_f32(float* buf, size_t n, void* stream) override { allreduce(buf, n, stream); }

 private:
  template <typename T>
  void allreduce(T* buf, size_t n, void* stream) {
    auto st = static_cast<cudaStream_t>(stream);
    std::vector<char> mine(sizeof(T) * n);
    if (n) PDD_CUDA(cudaMemcpyAsync(mine.data(), buf, mine.size(), cudaMemcpyDeviceToHost, st));
    PDD_CUDA(cudaStreamSynchronize(st));
    std::vector<T> out;
    {
      std::unique_lock<std::mutex> lock(hub_->mu);
      hub_->contrib[rank_] = std::move(mine);
      const uint64_t round = hub_->round;
      if (++hub_->arrived == world()) {
        std::vector<T> sum(n, T(0));
        for (int r = 0; r < world(); ++r) {  // fixed rank order
          if (hub_->contrib[r].size() != sizeof(T) * n) throw RuntimeError("host transport: all-reduce size mismatch");
          const T* c = reinterpret_cast<const T*>(hub_->contrib[r].data());
          for (size_t i = 0; i < n; ++i) sum[i] += c[i];
        }
        if constexpr (sizeof(T) == 8) hub_->result_f64 = sum;
        else hub_->result_f32 = sum;
        hub_->arrived = 0;
        ++hub_->round;
        hub_->cv.notify_all();
      } else {
        hub_->cv.wait(lock, [&] { return hub_->round != round; });
      }
      if constexpr (sizeof(T) == 8) out = hub_->result_f64;
      else out = hub_->result_f32;
    }
    if (n) PDD_CUDA(cudaMemcpyAsync(buf, out.data(), sizeof(T) * n, cudaMemcpyHostToDevice, st));
    PDD_CUDA(cudaStreamSynchronize(st));
  }

  std::shared_ptr<Hub> hub_;
  int rank_;
};

}  // namespace

void host_hub_id(void* out128) {
  std::random_device rd;
  uint64_t key = (static_cast<uint64_t>(rd()) << 32) ^ rd();
  char id[128] = {};
  std::memcpy(id, kMagic, sizeof(kMagic));
  std::memcpy(id + 8, &key, sizeof(key));
  std::memcpy(out128, id, sizeof(id));
}

bool is_host_hub_id(const void* id128) { return id128 && std::memcmp(id128, kMagic, sizeof(kMagic)) == 0; }

std::unique_ptr<Comm> make_host_comm(const void* hub_id128, int rank, int world) {
  if (!is_host_hub_id(hub_id128)) throw InvalidArgument("host transport: not a host hub id");
  if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("comm: bad rank/world");
  uint64_t key = 0;
  std::memcpy(&key, static_cast<const char*>(hub_id128) + 8, sizeof(key));
  return std::make_unique<HostComm>(hub_for(key, world), rank);
}

}  // namespace pdd
