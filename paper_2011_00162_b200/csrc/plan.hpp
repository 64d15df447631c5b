// Scan geometry and overlapping domain-decomposition plans (host, integer).
//
// Restates the reference's setup layer -- make_raster_scan (scan.cpp:18-34),
// scan_coverage (scan.cpp:36-44), plan_stripes (ddplan.cpp:28-94),
// pair_index / local_overlap / pairs_of (ddplan.cpp:7-26) -- and adds
// plan_grid, the 2-D block plan that configs 2 and 3 need (same rules on both
// scan axes).  Everything here is integer and must be
// bit-exact with the reference; tests compare it field by field.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace pdd {

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct OutOfRange : std::out_of_range {
  using std::out_of_range::out_of_range;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Divergence : std::runtime_error {
  int64_t iteration;
  explicit Divergence(int64_t it)
      : std::runtime_error("solver diverged: non-finite iterate at iteration " + std::to_string(it)),
        iteration(it) {}
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Half-open [r0,r1) x [c0,c1) (field.hpp:14-45).
struct Rect {
  int64_t r0 = 0, r1 = 0, c0 = 0, c1 = 0;
  int64_t h() const { return r1 - r0; }
  int64_t w() const { return c1 - c0; }
  int64_t area() const { return h() * w(); }
  bool intersects(const Rect& o) const { return r0 < o.r1 && o.r0 < r1 && c0 < o.c1 && o.c0 < c1; }
  Rect intersection(const Rect& o) const {
    return {std::max(r0, o.r0), std::min(r1, o.r1), std::max(c0, o.c0), std::min(c1, o.c1)};
  }
  bool contains(const Rect& o) const { return o.r0 >= r0 && o.r1 <= r1 && o.c0 >= c0 && o.c1 <= c1; }
  bool operator==(const Rect& o) const { return r0 == o.r0 && r1 == o.r1 && c0 == o.c0 && c1 == o.c1; }
};

struct Geometry {
  int64_t s = 0, step = 0, H = 0, W = 0, grid_rows = 0, grid_cols = 0;
  std::vector<int64_t> pos;  // [J][2] (row, col) window corners
  int64_t J() const { return static_cast<int64_t>(pos.size() / 2); }
  Rect window(int64_t j) const { return {pos[2 * j], pos[2 * j] + s, pos[2 * j + 1], pos[2 * j + 1] + s}; }
  void validate() const;  // scan.cpp:5-16
};

Geometry make_raster_scan(int64_t H, int64_t W, int64_t s, int64_t step);

struct Plan {
  struct Pair {
    int d1 = 0, d2 = 0;
    Rect region;
  };
  int D = 0;
  Geometry g;
  std::vector<Rect> subs;
  std::vector<int32_t> assign;
  std::vector<std::vector<int64_t>> frames_of;
  std::vector<Pair> overlaps;
  std::vector<Geometry> local;
  bool raster_blocks = false;  // built by plan_stripes/plan_grid: every subdomain is tiled by its own windows

  size_t pair_index(int a, int b) const;
  Rect local_overlap(int d, size_t p) const;
  std::vector<size_t> pairs_of(int d) const;
};

enum Axis { kAxisAuto = 0, kAxisColumns = 1, kAxisRows = 2 };

Plan plan_stripes(const Geometry& g, int D, int axis);
Plan plan_grid(const Geometry& g, int Dr, int Dc);
// General plan from explicit arrays (any scan positions); validates and
// derives frames_of / local geometries exactly as the reference does.
Plan plan_from_arrays(const Geometry& g, int D, const int32_t* assign, const int64_t* subs, int npairs,
                      const int32_t* pairs, const int64_t* regions);

// Per-pixel count of covering windows (scan.cpp:36-44), as int32.
std::vector<int32_t> scan_coverage(const Geometry& g);

}  // namespace pdd
