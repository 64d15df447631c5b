// PTYA frame stacks streamed from disk straight to the device (SURVEY.md
// sec. 8(f) row 3).
//
// The reference reads a whole frames.ptya into a std::vector<RealField2D>
// (io.cpp:186-202, one heap block per frame), which the solver then copies
// again; for config 4 that is 8.4 GB of float64 intensities held twice in host
// memory before anything reaches a GPU.  Here the file is read in large chunks
// by host threads into a ring of page-locked buffers, each chunk is DMA'd to a
// device staging buffer, and a kernel converts float64 intensity -> T
// amplitude sqrt(f) while scattering the frames to this rank's local order --
// disk, PCIe and conversion overlap, and no frame stack ever exists in host
// memory.  The container format and its validation follow io.cpp:80-112 and
// 186-202 (magic "PTYA", u16 version 1, u16 dtype 1 = f64, u16 ndim 3, u64
// dims, little-endian payload, no trailing bytes); malformed input raises
// FormatError with the byte offset (io.hpp:12-18).
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace pdd {

struct FormatError : std::runtime_error {
  uint64_t offset;
  FormatError(const std::string& msg, uint64_t off)
      : std::runtime_error(msg + " (byte offset " + std::to_string(off) + ")"), offset(off) {}
};

struct PtyaHeader {
  uint16_t version = 0, dtype = 0;
  std::vector<uint64_t> dims;
  uint64_t payload_offset = 0;  // bytes
  uint64_t file_bytes = 0;
};

// Parse and validate a header (io.cpp:95-115); want_dtype 1 = f64, 2 = c128.
PtyaHeader ptya_read_header(const std::string& path, uint16_t want_dtype);

// Stream the payload of a [J][s][s] float64 frame stack (validated against
// J and s as FrameStack::validate would, scan.cpp:46-56) in file order:
// enqueue(first, count, host) is called on the calling thread for every chunk
// of whole frames, with `host` a page-locked buffer holding the raw payload;
// it must enqueue its asynchronous use of `host` (the H2D copy) on `st` and
// return -- the buffer is refilled only after that work completes.  Reading
// runs ahead on host threads.
void ptya_stream_frames(const std::string& path, int64_t J, int64_t s, void* st,
                        const std::function<void(int64_t first, int64_t count, const double* host)>& enqueue);

}  // namespace pdd
