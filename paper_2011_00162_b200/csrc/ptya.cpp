// PTYA header parsing and the streamed frame upload (ptya.hpp).
#include "ptya.hpp"

#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>

#include "device.hpp"

namespace pdd {
namespace {

constexpr uint16_t kVersion = 1;

class File {
 public:
  explicit File(const std::string& path) : fd_(::open(path.c_str(), O_RDONLY | O_CLOEXEC)) {
    if (fd_ < 0) throw RuntimeError("cannot open: " + path);
  }
  ~File() {
    if (fd_ >= 0) ::close(fd_);
  }
  uint64_t size() const {
    struct stat st {};
    if (::fstat(fd_, &st) != 0) throw RuntimeError("cannot stat PTYA file");
    return static_cast<uint64_t>(st.st_size);
  }
  // Reads exactly n bytes at offset (short file: the bytes available).
  uint64_t read_at(void* dst, uint64_t n, uint64_t off) const {
    uint64_t done = 0;
    while (done < n) {
      const ssize_t r = ::pread(fd_, static_cast<char*>(dst) + done, n - done, static_cast<off_t>(off + done));
      if (r < 0) throw RuntimeError("read failed on PTYA file");
      if (r == 0) break;
      done += static_cast<uint64_t>(r);
    }
    return done;
  }

 private:
  int fd_;
};

uint16_t le16(const unsigned char* b) { return static_cast<uint16_t>(b[0] | (b[1] << 8)); }
uint64_t le64(const unsigned char* b) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(b[i]) << (8 * i);
  return v;
}

// Process-wide page-locked chunk ring (allocated once: a first page-locked
// allocation costs tens of ms).
struct Ring {
  static constexpr int kSlots = 6;
  static constexpr size_t kBytes = size_t(32) << 20;
  std::mutex mu;
  void* buf[kSlots] = {};
  static Ring& get() {
    static Ring r;
    return r;
  }
  void reserve_locked() {
    for (auto& b : buf)
      if (!b) PDD_CUDA(cudaHostAlloc(&b, kBytes, cudaHostAllocPortable));
  }
};

}  // namespace

PtyaHeader ptya_read_header(const std::string& path, uint16_t want_dtype) {
  File f(path);
  PtyaHeader h;
  h.file_bytes = f.size();
  unsigned char b[8 + 8 * 4];
  const uint64_t got = f.read_at(b, sizeof(b), 0);
  // io.cpp:95-115: magic, version, dtype, ndim in [1, 4], dims in [1, 2^32]
  if (got < 4 || std::memcmp(b, "PTYA", 4) != 0) throw FormatError("bad magic, not a PTYA file", 0);
  if (got < 6) throw FormatError("truncated PTYA file", 4);
  h.version = le16(b + 4);
  if (h.version != kVersion) throw FormatError("unsupported PTYA version " + std::to_string(h.version), 4);
  if (got < 8) throw FormatError("truncated PTYA file", 6);
  h.dtype = le16(b + 6);
  if (h.dtype != want_dtype)
    throw FormatError("dtype mismatch: file has code " + std::to_string(h.dtype) + ", expected " +
                          std::to_string(want_dtype),
                      6);
  if (got < 10) throw FormatError("truncated PTYA file", 8);
  const uint16_t ndim = le16(b + 8);
  if (ndim < 1 || ndim > 4) throw FormatError("unsupported ndim " + std::to_string(ndim), 8);
  uint64_t pos = 10;
  for (uint16_t i = 0; i < ndim; ++i) {
    if (got < pos + 8) throw FormatError("truncated PTYA file", pos);
    const uint64_t d = le64(b + pos);
    if (d == 0 || d > (uint64_t{1} << 32)) throw FormatError("implausible dimension " + std::to_string(d), pos);
    h.dims.push_back(d);
    pos += 8;
  }
  h.payload_offset = pos;
  return h;
}

void ptya_stream_frames(const std::string& path, int64_t J, int64_t s, void* stream,
                        const std::function<void(int64_t, int64_t, const double*)>& enqueue) {
  const PtyaHeader h = ptya_read_header(path, 1);
  if (h.dims.size() != 3) throw FormatError("expected a 3-D frame stack", 8);
  const uint64_t frame_elems = h.dims[1] * h.dims[2];
  const uint64_t need = h.payload_offset + h.dims[0] * frame_elems * 8;
  // read_frames reads element by element: a short file fails at its end, a
  // long one after the payload (io.cpp:61-64, 127-129)
  if (h.file_bytes < need) throw FormatError("truncated PTYA file", h.file_bytes);
  if (h.file_bytes > need) throw FormatError("trailing bytes after payload", need);
  // FrameStack::validate (scan.cpp:46-56)
  if (static_cast<int64_t>(h.dims[0]) != J || static_cast<int64_t>(h.dims[1]) != s ||
      static_cast<int64_t>(h.dims[2]) != s)
    throw InvalidArgument("FrameStack: frame count != scan position count or frame shape mismatch");
  const auto st = static_cast<cudaStream_t>(stream);
  const int64_t fbytes = static_cast<int64_t>(frame_elems * 8);
  const int64_t per_chunk = std::max<int64_t>(1, static_cast<int64_t>(Ring::kBytes) / fbytes);
  if (per_chunk * fbytes > static_cast<int64_t>(Ring::kBytes))
    throw InvalidArgument("PTYA streaming: frame larger than the chunk buffer");
  const int64_t nchunks = (J + per_chunk - 1) / per_chunk;
  File f(path);
  Ring& ring = Ring::get();
  std::lock_guard<std::mutex> ring_lock(ring.mu);  // one streamed upload at a time per process
  ring.reserve_locked();
  constexpr int S = Ring::kSlots;
  cudaEvent_t ev[S];
  for (auto& e : ev) PDD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // slot state: ready[slot] = chunk index whose bytes are in the slot (-1: none);
  // used[slot] = last chunk enqueued from the slot (its DMA completes at ev[slot])
  int64_t ready[S], used[S];
  for (int i = 0; i < S; ++i) ready[i] = used[i] = -1;
  std::mutex mu;
  std::condition_variable cv;
  std::atomic<int64_t> next{0};
  std::exception_ptr err;
  bool abort = false;
  const int readers = 4;
  std::vector<std::thread> th;
  for (int t = 0; t < readers; ++t)
    th.emplace_back([&] {
      try {
        for (int64_t k = next.fetch_add(1); k < nchunks; k = next.fetch_add(1)) {
          const int slot = static_cast<int>(k % S);
          {
            std::unique_lock<std::mutex> lock(mu);
            cv.wait(lock, [&] { return abort || k < S || used[slot] == k - S; });
            if (abort) return;
          }
          if (k >= S) PDD_CUDA(cudaEventSynchronize(ev[slot]));  // the slot's previous DMA is done
          const int64_t first = k * per_chunk, count = std::min(per_chunk, J - first);
          const uint64_t bytes = static_cast<uint64_t>(count * fbytes);
          if (f.read_at(ring.buf[slot], bytes, h.payload_offset + static_cast<uint64_t>(first * fbytes)) != bytes)
            throw FormatError("truncated PTYA file", h.payload_offset + static_cast<uint64_t>(first * fbytes));
          std::lock_guard<std::mutex> lock(mu);
          ready[slot] = k;
          cv.notify_all();
        }
      } catch (...) {
        std::lock_guard<std::mutex> lock(mu);
        if (!err) err = std::current_exception();
        abort = true;
        cv.notify_all();
      }
    });
  try {
    for (int64_t k = 0; k < nchunks; ++k) {
      const int slot = static_cast<int>(k % S);
      {
        std::unique_lock<std::mutex> lock(mu);
        cv.wait(lock, [&] { return abort || ready[slot] == k; });
        if (abort) break;
      }
      const int64_t first = k * per_chunk, count = std::min(per_chunk, J - first);
      enqueue(first, count, static_cast<const double*>(ring.buf[slot]));
      PDD_CUDA(cudaEventRecord(ev[slot], st));
      std::lock_guard<std::mutex> lock(mu);
      used[slot] = k;
      cv.notify_all();
    }
  } catch (...) {
    std::lock_guard<std::mutex> lock(mu);
    if (!err) err = std::current_exception();
    abort = true;
    cv.notify_all();
  }
  for (auto& t : th) t.join();
  cudaStreamSynchronize(st);  // the ring is reused by the next upload
  for (auto& e : ev) cudaEventDestroy(e);
  if (err) std::rethrow_exception(err);
}

}  // namespace pdd
