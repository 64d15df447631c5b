#include "plan.hpp"

#include <algorithm>

namespace pdd {

void Geometry::validate() const {
  if (s < 1 || step < 1) throw InvalidArgument("ScanGeometry: frame_side, step >= 1");
  if (step >= s) throw InvalidArgument("ScanGeometry: step must be < frame_side for sufficient overlap");
  if (J() == 0) throw InvalidArgument("ScanGeometry: no scan positions");
  if (J() != grid_rows * grid_cols)
    throw InvalidArgument("ScanGeometry: positions do not form the declared raster grid");
  for (int64_t j = 0; j < J(); ++j) {
    const int64_t r = pos[2 * j], c = pos[2 * j + 1];
    if (r < 0 || c < 0 || r + s > H || c + s > W) throw InvalidArgument("ScanGeometry: window outside image bounds");
  }
}

Geometry make_raster_scan(int64_t H, int64_t W, int64_t s, int64_t step) {
  if (s > H || s > W) throw InvalidArgument("make_raster_scan: frame larger than image");
  if (s < 1 || step < 1) throw InvalidArgument("ScanGeometry: frame_side, step >= 1");
  Geometry g;
  g.s = s;
  g.step = step;
  g.H = H;
  g.W = W;
  g.grid_rows = (H - s) / step + 1;
  g.grid_cols = (W - s) / step + 1;
  g.pos.reserve(static_cast<size_t>(2 * g.grid_rows * g.grid_cols));
  for (int64_t i = 0; i < g.grid_rows; ++i)
    for (int64_t j = 0; j < g.grid_cols; ++j) {
      g.pos.push_back(i * step);
      g.pos.push_back(j * step);
    }
  g.validate();
  return g;
}

size_t Plan::pair_index(int a, int b) const {
  if (a > b) std::swap(a, b);
  for (size_t p = 0; p < overlaps.size(); ++p)
    if (overlaps[p].d1 == a && overlaps[p].d2 == b) return p;
  throw InvalidArgument("DecompositionPlan: subdomains are not neighbors");
}

Rect Plan::local_overlap(int d, size_t p) const {
  const Rect& ov = overlaps[p].region;
  const Rect& sub = subs[d];
  return {ov.r0 - sub.r0, ov.r1 - sub.r0, ov.c0 - sub.c0, ov.c1 - sub.c0};
}

std::vector<size_t> Plan::pairs_of(int d) const {
  std::vector<size_t> out;
  for (size_t p = 0; p < overlaps.size(); ++p)
    if (overlaps[p].d1 == d || overlaps[p].d2 == d) out.push_back(p);
  return out;
}

namespace {

std::vector<int64_t> blocks(int64_t lines, int n) {
  std::vector<int64_t> b(static_cast<size_t>(n) + 1, 0);
  const int64_t base = lines / n, extra = lines % n;
  for (int i = 0; i < n; ++i) b[i + 1] = b[i] + base + (i < extra ? 1 : 0);
  return b;
}

int block_of(const std::vector<int64_t>& b, int64_t line) {
  return static_cast<int>(std::upper_bound(b.begin() + 1, b.end(), line) - b.begin() - 1);
}

// Subdomains = union of windows, overlaps = all intersecting pairs d1<d2,
// local geometries translated (ddplan.cpp:59-92).
void finish(Plan& plan, const std::vector<std::pair<int64_t, int64_t>>& local_grid) {
  const Geometry& g = plan.g;
  plan.subs.clear();
  for (int d = 0; d < plan.D; ++d) {
    if (plan.frames_of[d].empty()) throw InvalidArgument("plan_stripes: empty subdomain");
    Rect sub = g.window(plan.frames_of[d].front());
    for (int64_t j : plan.frames_of[d]) {
      const Rect w = g.window(j);
      sub.r0 = std::min(sub.r0, w.r0);
      sub.r1 = std::max(sub.r1, w.r1);
      sub.c0 = std::min(sub.c0, w.c0);
      sub.c1 = std::max(sub.c1, w.c1);
    }
    plan.subs.push_back(sub);
  }
  plan.overlaps.clear();
  for (int d1 = 0; d1 < plan.D; ++d1)
    for (int d2 = d1 + 1; d2 < plan.D; ++d2)
      if (plan.subs[d1].intersects(plan.subs[d2]))
        plan.overlaps.push_back({d1, d2, plan.subs[d1].intersection(plan.subs[d2])});
  plan.local.clear();
  for (int d = 0; d < plan.D; ++d) {
    const Rect& sub = plan.subs[d];
    Geometry l;
    l.s = g.s;
    l.step = g.step;
    l.H = sub.h();
    l.W = sub.w();
    l.grid_rows = local_grid[d].first;
    l.grid_cols = local_grid[d].second;
    for (int64_t j : plan.frames_of[d]) {
      l.pos.push_back(g.pos[2 * j] - sub.r0);
      l.pos.push_back(g.pos[2 * j + 1] - sub.c0);
    }
    l.validate();
    plan.local.push_back(std::move(l));
  }
}

}  // namespace

Plan plan_stripes(const Geometry& g, int D, int axis) {
  g.validate();
  if (D < 1) throw InvalidArgument("plan_stripes: D must be >= 1");
  if (axis == kAxisAuto) axis = g.grid_cols >= g.grid_rows ? kAxisColumns : kAxisRows;
  const bool by_cols = axis == kAxisColumns;
  const int64_t lines = by_cols ? g.grid_cols : g.grid_rows;
  if (D > lines) throw InvalidArgument("plan_stripes: D exceeds the scan frame-line count");
  const auto b = blocks(lines, D);
  Plan plan;
  plan.D = D;
  plan.g = g;
  plan.assign.resize(static_cast<size_t>(g.J()));
  plan.frames_of.resize(static_cast<size_t>(D));
  for (int64_t j = 0; j < g.J(); ++j) {
    const int64_t line = by_cols ? j % g.grid_cols : j / g.grid_cols;
    const int d = block_of(b, line);
    plan.assign[j] = d;
    plan.frames_of[d].push_back(j);
  }
  std::vector<std::pair<int64_t, int64_t>> lg;
  for (int d = 0; d < D; ++d)
    lg.emplace_back(by_cols ? g.grid_rows : b[d + 1] - b[d], by_cols ? b[d + 1] - b[d] : g.grid_cols);
  finish(plan, lg);
  plan.raster_blocks = true;
  return plan;
}

Plan plan_grid(const Geometry& g, int Dr, int Dc) {
  g.validate();
  if (Dr < 1 || Dc < 1) throw InvalidArgument("plan_grid: Dr, Dc must be >= 1");
  if (Dr > g.grid_rows || Dc > g.grid_cols)
    throw InvalidArgument("plan_grid: block count exceeds the scan frame-line count");
  const auto rb = blocks(g.grid_rows, Dr), cb = blocks(g.grid_cols, Dc);
  Plan plan;
  plan.D = Dr * Dc;
  plan.g = g;
  plan.assign.resize(static_cast<size_t>(g.J()));
  plan.frames_of.resize(static_cast<size_t>(plan.D));
  for (int64_t j = 0; j < g.J(); ++j) {
    const int d = block_of(rb, j / g.grid_cols) * Dc + block_of(cb, j % g.grid_cols);
    plan.assign[j] = d;
    plan.frames_of[d].push_back(j);
  }
  std::vector<std::pair<int64_t, int64_t>> lg;
  for (int d = 0; d < plan.D; ++d)
    lg.emplace_back(rb[d / Dc + 1] - rb[d / Dc], cb[d % Dc + 1] - cb[d % Dc]);
  finish(plan, lg);
  plan.raster_blocks = true;
  return plan;
}

Plan plan_from_arrays(const Geometry& g, int D, const int32_t* assign, const int64_t* subs, int npairs,
                      const int32_t* pairs, const int64_t* regions) {
  if (D < 1) throw InvalidArgument("plan: D must be >= 1");
  if (g.s < 1 || g.step < 1) throw InvalidArgument("ScanGeometry: frame_side, step >= 1");
  Plan plan;
  plan.D = D;
  plan.g = g;
  plan.assign.assign(assign, assign + g.J());
  plan.frames_of.resize(static_cast<size_t>(D));
  for (int64_t j = 0; j < g.J(); ++j) {
    if (assign[j] < 0 || assign[j] >= D) throw InvalidArgument("plan: frame assignment out of range");
    plan.frames_of[assign[j]].push_back(j);
  }
  for (int d = 0; d < D; ++d) {
    const Rect r{subs[4 * d], subs[4 * d + 1], subs[4 * d + 2], subs[4 * d + 3]};
    if (r.r0 < 0 || r.c0 < 0 || r.r0 >= r.r1 || r.c0 >= r.c1 || r.r1 > g.H || r.c1 > g.W)
      throw InvalidArgument("plan: subdomain rectangle outside the image");
    for (int64_t j : plan.frames_of[d])
      if (!r.contains(g.window(j))) throw InvalidArgument("plan: subdomain does not contain its windows");
    plan.subs.push_back(r);
  }
  for (int p = 0; p < npairs; ++p) {
    Plan::Pair pr{pairs[2 * p], pairs[2 * p + 1],
                  Rect{regions[4 * p], regions[4 * p + 1], regions[4 * p + 2], regions[4 * p + 3]}};
    if (pr.d1 < 0 || pr.d2 >= D || pr.d1 >= pr.d2) throw InvalidArgument("plan: overlap pair must satisfy d1 < d2");
    if (!plan.subs[pr.d1].contains(pr.region) || !plan.subs[pr.d2].contains(pr.region))
      throw InvalidArgument("plan: overlap region outside its subdomains");
    plan.overlaps.push_back(pr);
  }
  for (int d = 0; d < D; ++d) {
    const Rect& sub = plan.subs[d];
    Geometry l;
    l.s = g.s;
    l.step = g.step;
    l.H = sub.h();
    l.W = sub.w();
    l.grid_rows = 1;
    l.grid_cols = static_cast<int64_t>(plan.frames_of[d].size());
    for (int64_t j : plan.frames_of[d]) {
      l.pos.push_back(g.pos[2 * j] - sub.r0);
      l.pos.push_back(g.pos[2 * j + 1] - sub.c0);
    }
    plan.local.push_back(std::move(l));
  }
  return plan;
}

std::vector<int32_t> scan_coverage(const Geometry& g) {
  // 2-D difference array: O(J + H*W) instead of O(J*s^2).
  std::vector<int32_t> diff(static_cast<size_t>((g.H + 1) * (g.W + 1)), 0);
  auto at = [&](int64_t r, int64_t c) -> int32_t& { return diff[static_cast<size_t>(r * (g.W + 1) + c)]; };
  for (int64_t j = 0; j < g.J(); ++j) {
    const Rect w = g.window(j);
    at(w.r0, w.c0) += 1;
    at(w.r0, w.c1) -= 1;
    at(w.r1, w.c0) -= 1;
    at(w.r1, w.c1) += 1;
  }
  std::vector<int32_t> cov(static_cast<size_t>(g.H * g.W), 0);
  std::vector<int32_t> run(static_cast<size_t>(g.W + 1), 0);
  for (int64_t r = 0; r < g.H; ++r) {
    int32_t acc = 0;
    for (int64_t c = 0; c < g.W; ++c) {
      run[c] += at(r, c);
      acc += run[c];
      cov[static_cast<size_t>(r * g.W + c)] = acc;
    }
  }
  return cov;
}

}  // namespace pdd
