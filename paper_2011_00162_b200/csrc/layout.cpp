#include <cstdlib>
#include "layout.hpp"

#include <algorithm>

namespace pdd {

Layout Layout::build(const Plan& plan, int rank, int world, bool allow_wide, int piece_len) {
  Layout L;
  L.D = plan.D;
  L.rank = rank;
  L.world = world;
  L.S = static_cast<int>(plan.g.s);
  L.sub_local.assign(plan.D, -1);
  for (int d = 0; d < plan.D; ++d)
    if (owner_of(d, plan.D, world) == rank) {
      L.sub_local[d] = static_cast<int>(L.local_subs.size());
      L.local_subs.push_back(d);
    }

  // images and frames
  L.sub_fr_beg.push_back(0);
  for (int ld = 0; ld < L.nls(); ++ld) {
    const int d = L.local_subs[ld];
    const Rect& sub = plan.subs[d];
    L.sub_img_off.push_back(L.img_elems);
    L.sub_h.push_back(static_cast<int32_t>(sub.h()));
    L.sub_w.push_back(static_cast<int32_t>(sub.w()));
    const Geometry& lg = plan.local[d];
    for (int64_t k = 0; k < lg.J(); ++k) {
      const int64_t r = lg.pos[2 * k], c = lg.pos[2 * k + 1];
      L.fr_global.push_back(plan.frames_of[d][k]);
      L.fr_off.push_back(L.img_elems + r * sub.w() + c);
      L.fr_pitch.push_back(static_cast<int32_t>(sub.w()));
      L.fr_r.push_back(static_cast<int32_t>(r));
      L.fr_c.push_back(static_cast<int32_t>(c));
      L.fr_sub.push_back(ld);
    }
    L.img_elems += sub.area();
    L.sub_fr_beg.push_back(static_cast<int64_t>(L.fr_global.size()));
  }
  L.nfr = static_cast<int64_t>(L.fr_global.size());

  // gather tiles: 32 wide, tile_h high; covering frames in ascending order
  // (mid-sized images: 16 rows measured 3-4 % per iteration better than 8 on configs 1 and 3, 32 worse,
  // and 8 better on config 0's 128^2 image)
  L.tile_h = L.img_elems >= (int64_t(4) << 20) ? 32 : L.img_elems >= (int64_t(64) << 10) ? 16 : 8;
  if (const char* e = std::getenv("PDD_TILE_H")) {  // A/B runs: 8, 16 or 32
    const int v = std::atoi(e);
    if (v == 8 || v == 16 || v == 32) L.tile_h = v;
  }
  // 64-wide tiles (16-byte column pairs) when every window column and S are even
  bool even = (L.S % 2) == 0;
  for (int32_t c : L.fr_c) even = even && (c % 2 == 0);
  L.tile_w = (allow_wide && even && L.tile_h == 32) ? 64 : 32;
  const int th = L.tile_h, tw = L.tile_w;
  L.sub_tile_beg.push_back(0);
  for (int ld = 0; ld < L.nls(); ++ld) {
    const int64_t H = L.sub_h[ld], W = L.sub_w[ld];
    const int64_t ntr = (H + th - 1) / th, ntc = (W + tw - 1) / tw;
    // covering frames per tile, ascending f: counting pass, prefix sums, fill
    // (one flat array; a vector per tile cost ~10 ms of host time on config 4)
    std::vector<int32_t> cnt(static_cast<size_t>(ntr * ntc) + 1, 0);
    auto tiles_of = [&](int64_t f, auto&& fn) {
      const int64_t r0 = L.fr_r[f], c0 = L.fr_c[f];
      const int64_t tr_a = r0 / th, tr_b = std::min(ntr - 1, (r0 + L.S - 1) / th);
      const int64_t tc_a = c0 / tw, tc_b = std::min(ntc - 1, (c0 + L.S - 1) / tw);
      for (int64_t tr = tr_a; tr <= tr_b; ++tr)
        for (int64_t tc = tc_a; tc <= tc_b; ++tc) fn(tr * ntc + tc);
    };
    for (int64_t f = L.sub_fr_beg[ld]; f < L.sub_fr_beg[ld + 1]; ++f)
      tiles_of(f, [&](int64_t tile) { ++cnt[static_cast<size_t>(tile) + 1]; });
    for (size_t k = 1; k < cnt.size(); ++k) cnt[k] += cnt[k - 1];
    const size_t base0 = L.tile_frames.size();
    L.tile_frames.resize(base0 + static_cast<size_t>(cnt.back()));
    for (int64_t tr = 0; tr < ntr; ++tr)
      for (int64_t tc = 0; tc < ntc; ++tc)
        L.tiles.push_back(int4{ld, static_cast<int>(tr * th), static_cast<int>(tc * tw),
                               static_cast<int>(base0 + static_cast<size_t>(cnt[static_cast<size_t>(tr * ntc + tc)]))});
    {
      std::vector<int32_t> cur(cnt.begin(), cnt.end() - 1);
      for (int64_t f = L.sub_fr_beg[ld]; f < L.sub_fr_beg[ld + 1]; ++f)
        tiles_of(f, [&](int64_t tile) {
          L.tile_frames[base0 + static_cast<size_t>(cur[static_cast<size_t>(tile)]++)] = static_cast<int32_t>(f);
        });
    }
    L.sub_tile_beg.push_back(static_cast<int64_t>(L.tiles.size()));
  }
  L.tiles.push_back(int4{0, 0, 0, static_cast<int>(L.tile_frames.size())});

  // back-projection pieces (see layout.hpp)
  const bool chain = piece_len > 1;
  L.chained = chain;
  L.piece_len = std::max(1, std::min(piece_len, kPieceLen));
  L.pc_beg.push_back(0);
  const int64_t S = L.S;
  auto add_piece = [&](const std::vector<int64_t>& fs) {
    const int64_t r0 = L.fr_r[fs[0]], h = L.fr_r[fs.back()] - r0 + S;
    const int64_t base = L.part_elems;
    for (size_t i = 0; i < fs.size(); ++i) {
      const int64_t r = L.fr_r[fs[i]];
      const int lo = i + 1 < fs.size() ? static_cast<int>(L.fr_r[fs[i + 1]] - r) : static_cast<int>(S);
      const int nf = i > 0 ? static_cast<int>(S - (r - L.fr_r[fs[i - 1]])) : 0;
      L.pc_pos.push_back(int4{static_cast<int>(fs[i]), lo, nf, static_cast<int>((r >> 4) & 7)});
      L.pc_ofs.push_back(base + (r - r0) * S);
    }
    L.pc_beg.push_back(static_cast<int32_t>(L.pc_pos.size()));
    L.it_r.push_back(static_cast<int32_t>(r0));
    L.it_c.push_back(L.fr_c[fs[0]]);
    L.it_h.push_back(static_cast<int32_t>(h));
    L.it_base.push_back(base);
    L.part_elems += h * S;
  };
  for (int ld = 0; ld < L.nls(); ++ld) {
    const int64_t fb = L.sub_fr_beg[ld], fe = L.sub_fr_beg[ld + 1];
    if (!chain) {
      for (int64_t f = fb; f < fe; ++f) add_piece({f});
      continue;
    }
    // runs per window column (ascending row), split where the spacing breaks
    // the ring (not a positive multiple of 16 up to S), then cut into
    // ceil(n / piece_len) pieces of near-equal length
    std::vector<int64_t> order;
    for (int64_t f = fb; f < fe; ++f) order.push_back(f);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      return L.fr_c[a] != L.fr_c[b] ? L.fr_c[a] < L.fr_c[b] : L.fr_r[a] < L.fr_r[b];
    });
    std::vector<std::vector<int64_t>> runs;
    for (int64_t f : order) {
      bool join = !runs.empty();
      if (join) {
        const auto& cur = runs.back();
        const int64_t pf = cur.back(), d = L.fr_r[f] - L.fr_r[pf];
        join = L.fr_c[f] == L.fr_c[pf] && d > 0 && d <= S && d % 16 == 0;
      }
      if (join) runs.back().push_back(f);
      else runs.push_back({f});
    }
    {
      std::vector<std::vector<int64_t>> cut;
      for (const auto& r : runs) {
        const int64_t n = static_cast<int64_t>(r.size()), k = (n + L.piece_len - 1) / L.piece_len;
        for (int64_t p = 0, b = 0; p < k; ++p) {
          const int64_t e = (n * (p + 1)) / k;
          cut.emplace_back(r.begin() + b, r.begin() + e);
          b = e;
        }
      }
      runs.swap(cut);
    }
    // sweep order: by first row, then column -- concurrently running CTAs
    // then work on horizontally adjacent pieces and share the image rows in L2
    std::stable_sort(runs.begin(), runs.end(), [&](const auto& a, const auto& b) {
      return L.fr_r[a[0]] != L.fr_r[b[0]] ? L.fr_r[a[0]] < L.fr_r[b[0]] : L.fr_c[a[0]] < L.fr_c[b[0]];
    });
    for (const auto& r : runs) add_piece(r);
  }
  // covering pieces per gather tile, (column, row) order
  {
    const int th = L.tile_h, tw = L.tile_w;
    L.tile_item_beg.push_back(0);
    int k0 = 0;
    for (int ld = 0; ld < L.nls(); ++ld) {
      const int64_t H = L.sub_h[ld], W = L.sub_w[ld];
      const int64_t ntr = (H + th - 1) / th, ntc = (W + tw - 1) / tw;
      int k1 = k0;
      while (k1 < L.npieces() && L.fr_sub[L.pc_pos[L.pc_beg[k1]].x] == ld) ++k1;
      std::vector<int32_t> ids;
      for (int k = k0; k < k1; ++k) ids.push_back(k);
      std::stable_sort(ids.begin(), ids.end(), [&](int32_t a, int32_t b) {
        return L.it_c[a] != L.it_c[b] ? L.it_c[a] < L.it_c[b] : L.it_r[a] < L.it_r[b];
      });
      // counting pass, prefix sums, fill (ids order within each tile)
      auto tiles_of = [&](int32_t k, auto&& fn) {
        const int64_t r0 = L.it_r[k], c0 = L.it_c[k];
        const int64_t tr_a = r0 / th, tr_b = std::min(ntr - 1, (r0 + L.it_h[k] - 1) / th);
        const int64_t tc_a = c0 / tw, tc_b = std::min(ntc - 1, (c0 + S - 1) / tw);
        for (int64_t tr = tr_a; tr <= tr_b; ++tr)
          for (int64_t tc = tc_a; tc <= tc_b; ++tc) fn(tr * ntc + tc);
      };
      std::vector<int32_t> cnt(static_cast<size_t>(ntr * ntc) + 1, 0);
      for (int32_t k : ids) tiles_of(k, [&](int64_t tile) { ++cnt[static_cast<size_t>(tile) + 1]; });
      for (size_t q = 1; q < cnt.size(); ++q) cnt[q] += cnt[q - 1];
      const size_t base0 = L.tile_items.size();
      L.tile_items.resize(base0 + static_cast<size_t>(cnt.back()));
      {
        std::vector<int32_t> cur(cnt.begin(), cnt.end() - 1);
        for (int32_t k : ids)
          tiles_of(k, [&](int64_t tile) { L.tile_items[base0 + static_cast<size_t>(cur[static_cast<size_t>(tile)]++)] = k; });
      }
      for (size_t q = 1; q < cnt.size(); ++q) L.tile_item_beg.push_back(static_cast<int32_t>(base0) + cnt[q]);
      k0 = k1;
    }
  }

  // overlap pairs touching a local subdomain, ascending global p
  std::vector<int> lp_of(plan.overlaps.size(), -1);
  for (size_t p = 0; p < plan.overlaps.size(); ++p) {
    const auto& pr = plan.overlaps[p];
    const int l1 = L.sub_local[pr.d1], l2 = L.sub_local[pr.d2];
    if (l1 < 0 && l2 < 0) continue;
    const int lp = static_cast<int>(L.lpairs.size());
    lp_of[p] = lp;
    L.lpairs.push_back(static_cast<int>(p));
    PairGeom pg{};
    pg.h = static_cast<int32_t>(pr.region.h());
    pg.w = static_cast<int32_t>(pr.region.w());
    const int64_t n = pr.region.area();
    L.max_pair_pix = std::max<int>(L.max_pair_pix, static_cast<int>(n));
    pg.v_off = L.v_elems;
    pg.s_off = L.s_elems;
    const int ds[2] = {pr.d1, pr.d2};
    for (int side = 0; side < 2; ++side) {
      const int ld = L.sub_local[ds[side]];
      pg.lam_off[side] = L.lam_elems + side * n;
      if (ld < 0) {
        pg.u_off[side] = -1;
        pg.u_pitch[side] = 0;
      } else {
        const Rect lo = plan.local_overlap(ds[side], p);
        pg.u_off[side] = L.sub_img_off[ld] + lo.r0 * L.sub_w[ld] + lo.c0;
        pg.u_pitch[side] = L.sub_w[ld];
      }
    }
    if ((l1 < 0) != (l2 < 0)) {
      const int my_side = l1 >= 0 ? 0 : 1;
      L.exch.push_back(Exchange{lp, owner_of(ds[1 - my_side], plan.D, world), my_side});
    }
    L.v_elems += n;
    L.lam_elems += 2 * n;
    L.s_elems += 2 * n;
    L.pgeom.push_back(pg);
  }
  L.sub_pbeg.push_back(0);
  for (int ld = 0; ld < L.nls(); ++ld) {
    const int d = L.local_subs[ld];
    for (size_t p : plan.pairs_of(d)) {
      const int lp = lp_of[p];
      const int side = plan.overlaps[p].d1 == d ? 0 : 1;
      const Rect lo = plan.local_overlap(d, p);
      PairSide ps{};
      ps.r0 = static_cast<int32_t>(lo.r0);
      ps.r1 = static_cast<int32_t>(lo.r1);
      ps.c0 = static_cast<int32_t>(lo.c0);
      ps.c1 = static_cast<int32_t>(lo.c1);
      ps.v_off = L.pgeom[lp].v_off;
      ps.lam_off = L.pgeom[lp].lam_off[side];
      L.psides.push_back(ps);
    }
    L.sub_pbeg.push_back(static_cast<int32_t>(L.psides.size()));
  }
  L.flatten_gather_lists();
  return L;
}

void Layout::flatten_gather_lists() {
  const int64_t SS = static_cast<int64_t>(S) * S;
  fmeta_beg.assign(1, 0);
  imeta_beg.assign(1, 0);
  tps_beg.assign(1, 0);
  fmeta.clear();
  imeta.clear();
  fmeta_base.clear();
  imeta_base.clear();
  tps.clear();
  // chained layouts: the update pass walks the pieces (imeta); the per-frame
  // lists are then only read by the one-off density gather at setup, which
  // takes them from tile_frames directly (no flattened copy: 15 MB on config 4)
  const bool frames_flat = !chained;
  if (frames_flat) {
    fmeta.reserve(tile_frames.size());
    fmeta_base.reserve(tile_frames.size());
    fmeta_beg.reserve(static_cast<size_t>(ntiles()) + 1);
  } else {
    fmeta_beg.clear();
    imeta.reserve(tile_items.size());
    imeta_base.reserve(tile_items.size());
    imeta_beg.reserve(static_cast<size_t>(ntiles()) + 1);
  }
  tps_beg.reserve(static_cast<size_t>(ntiles()) + 1);
  for (int t = 0; t < ntiles(); ++t) {
    if (frames_flat) {
      for (int k = tiles[t].w; k < tiles[t + 1].w; ++k) {
        const int f = tile_frames[k];
        fmeta.push_back(int4{fr_r[f], fr_c[f], S, f});
        fmeta_base.push_back(static_cast<int64_t>(f) * SS);
      }
      fmeta_beg.push_back(static_cast<int32_t>(fmeta.size()));
    }
    if (chained) {
      for (int k = tile_item_beg[t]; k < tile_item_beg[t + 1]; ++k) {
        const int it = tile_items[k];
        imeta.push_back(int4{it_r[it], it_c[it], it_h[it], -1});
        imeta_base.push_back(it_base[it]);
      }
      imeta_beg.push_back(static_cast<int32_t>(imeta.size()));
    }
    // pair sides of the tile's subdomain whose overlap rectangle meets the tile
    const int ld = tiles[t].x, r0 = tiles[t].y, c0 = tiles[t].z;
    for (int q = sub_pbeg[ld]; q < sub_pbeg[ld + 1]; ++q) {
      const PairSide& p = psides[q];
      if (p.r0 < r0 + tile_h && r0 < p.r1 && p.c0 < c0 + tile_w && c0 < p.c1) tps.push_back(q);
    }
    tps_beg.push_back(static_cast<int32_t>(tps.size()));
  }
}

void Layout::schedule(int G) {
  ncta = G;
  cta_beg.assign(1, 0);
  cta_pos.clear();
  cta_ofs.clear();
  for (int b = 0; b < G; ++b) {
    for (int k = b; k < npieces(); k += G)
      for (int q = pc_beg[k]; q < pc_beg[k + 1]; ++q) {
        cta_pos.push_back(pc_pos[q]);
        cta_ofs.push_back(pc_ofs[q]);
      }
    cta_beg.push_back(static_cast<int32_t>(cta_pos.size()));
  }
}

}  // namespace pdd
