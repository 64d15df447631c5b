// Device-side data layout of one rank's share of a decomposition plan.
//
// HBM layout (all contiguous, element = cx<T> unless noted):
//   images  u      : local subdomains back to back, row-major [H_d][W_d]
//   frames  Gamma  : [n_local_frames][S][S], frames ordered (local subdomain,
//                    ascending global j) -- the reference's frames_of order
//                    (ddplan.cpp:50-57) -- amplitudes (T) and the
//                    back-projection scratch use the same order
//   overlap v, Lambda, s : per local pair (ascending global p) [h][w];
//                    Lambda and s hold side 0 (d1) then side 1 (d2)
// plus the integer tables the kernels walk: per-frame window offsets, the
// gather tiles with their ascending covering-frame lists, pair sides.
#pragma once

#include <cstdint>
#include <vector>

#include "kernels.hpp"
#include "plan.hpp"

namespace pdd {

// Subdomain d lives on rank floor(d * world / D).
inline int owner_of(int d, int D, int world) { return static_cast<int>((static_cast<int64_t>(d) * world) / D); }

struct Exchange {
  int lp;        // local pair index
  int peer;      // remote rank
  int my_side;   // 0 or 1
};

struct Layout {
  int D = 0, rank = 0, world = 1, S = 0;
  std::vector<int> local_subs;  // global d, ascending
  std::vector<int> sub_local;   // [D] -> local index or -1

  int64_t nfr = 0;
  std::vector<int64_t> fr_global;   // [nfr]
  std::vector<int64_t> sub_fr_beg;  // [nls+1]
  std::vector<int64_t> sub_img_off; // [nls]
  std::vector<int32_t> sub_h, sub_w;
  int64_t img_elems = 0;

  std::vector<int64_t> fr_off;  // window corner offset into the image buffer
  std::vector<int32_t> fr_pitch, fr_r, fr_c, fr_sub;

  int tile_h = 8;
  int tile_w = 32;
  std::vector<int4> tiles;  // + sentinel
  std::vector<int32_t> tile_frames;
  std::vector<int64_t> sub_tile_beg;  // [nls+1]

  // Back-projection pieces.  A piece is a run of frames of one subdomain
  // that share a window column, in ascending rows spaced by a multiple of 16
  // px (at most S apart, at most kPieceLen frames).  The streamed sweep
  // (S = 128, float) keeps a piece's running overlap-add in tensor memory and
  // writes each image row of the piece once, into a [h][S] partial image; the
  // update gather then sums the pieces covering a pixel in (column, row)
  // order.  With chaining off every frame is its own piece and the partial
  // images are the per-frame tiles [nfr][S][S].  Pieces depend only on the
  // subdomain, so iterates stay identical for every GPU count.
  static constexpr int kPieceLen = 8;  // upper bound of piece_len
  bool chained = false;
  int piece_len = 1;
  std::vector<int32_t> pc_beg;   // [npieces+1] CSR into pc_pos / pc_ofs (sweep order)
  std::vector<int4> pc_pos;      // [nfr] {frame, lo, newfrom, rot}: rows y < lo are final after
                                 // this frame, rows y >= newfrom are first touched by it,
                                 // rot = (window row / 16) mod 8 (tensor-memory ring slot)
  std::vector<int64_t> pc_ofs;   // [nfr] element offset of the frame's window row 0 in the partials
  std::vector<int32_t> it_r, it_c, it_h;  // [npieces] partial image rect (subdomain coords, width S)
  std::vector<int64_t> it_base;           // [npieces] element offset of the partial image
  int64_t part_elems = 0;
  std::vector<int32_t> tile_items;        // per tile: covering pieces, (column, row) order
  std::vector<int32_t> tile_item_beg;     // [ntiles+1]
  int npieces() const { return static_cast<int>(pc_beg.size()) - 1; }
  // Sweep schedule for a persistent grid of G CTAs: pieces k = b, b + G, ...
  // go to CTA b; its positions are cta_pos[cta_beg[b] .. cta_beg[b+1]).
  int ncta = 0;
  std::vector<int32_t> cta_beg;
  std::vector<int4> cta_pos;
  std::vector<int64_t> cta_ofs;
  void schedule(int G);

  // Flattened gather lists (GatherArgs::mbeg/meta/mbase): per tile, its
  // covering frames (fmeta) and, chained, its covering pieces (imeta);
  // meta = {r0, c0, h, frame or -1}.  tps: per tile, the PairSide indices
  // whose overlap rectangle meets it.
  std::vector<int32_t> fmeta_beg, imeta_beg, tps_beg, tps;
  std::vector<int4> fmeta, imeta;
  std::vector<int64_t> fmeta_base, imeta_base;
  void flatten_gather_lists();

  std::vector<int> lpairs;          // global pair index per local pair
  std::vector<PairGeom> pgeom;      // per local pair
  std::vector<int32_t> sub_pbeg;    // [nls+1] CSR into psides
  std::vector<PairSide> psides;
  int64_t v_elems = 0, lam_elems = 0, s_elems = 0;
  int max_pair_pix = 0;
  std::vector<Exchange> exch;

  // piece_len > 1: multi-frame back-projection pieces of at most piece_len
  // frames (else one piece per frame)
  static Layout build(const Plan& plan, int rank, int world, bool allow_wide = false, int piece_len = 1);
  int nls() const { return static_cast<int>(local_subs.size()); }
  int ntiles() const { return static_cast<int>(tiles.size()) - 1; }
};

}  // namespace pdd
