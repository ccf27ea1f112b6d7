#include "attn_sched.hpp"

#include <algorithm>
#include <vector>

namespace glmx {

namespace {
size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
}  // namespace

size_t attn_sched_bytes(int max_items, int n_sm, size_t* off_pieces, size_t* off_cta,
                        size_t* off_combine) {
  size_t o = 0;
  if (off_pieces) *off_pieces = o;
  o = align16(o + static_cast<size_t>(max_items + n_sm) * sizeof(AttnPiece));
  if (off_cta) *off_cta = o;
  o = align16(o + static_cast<size_t>(n_sm + 1) * sizeof(int32_t));
  if (off_combine) *off_combine = o;
  o = align16(o + static_cast<size_t>(n_sm) * sizeof(AttnCombine));
  return o;
}

int attn_item_tiles(int t0, int q_len, int ctx_len, int tokens_per_item, int keys_per_tile) {
  const int max_pos = ctx_len - q_len + std::min(t0 + tokens_per_item, q_len) - 1;
  return max_pos / keys_per_tile + 1;
}

void build_attn_schedule(const int32_t* work_xy, int n_work, int Hkv, const int32_t* q_len,
                         const int32_t* ctx_len, int tokens_per_item, int keys_per_tile, int n_sm,
                         AttnSchedule& s) {
  const int n_items = n_work * Hkv;
  s.n_pieces = s.n_combine = s.n_partials = 0;
  s.total_tiles = 0;
  s.grid = 0;
  if (n_items == 0) return;
  std::vector<int> tiles(n_items);
  for (int w = 0; w < n_items; ++w) {
    const int r = work_xy[2 * (w / Hkv)], t0 = work_xy[2 * (w / Hkv) + 1];
    tiles[w] = attn_item_tiles(t0, q_len[r], ctx_len[r], tokens_per_item, keys_per_tile);
    s.total_tiles += tiles[w];
  }
  std::vector<int> n_pieces_of(n_items, 0);
  if (n_items * 2 > n_sm) {
    // Enough items to occupy the SMs: whole items, longest first, dealt round-robin to
    // min(n_items, n_sm) persistent CTAs (no partials, no combine pass).  Splitting here does not
    // pay: the partial O traffic (128 KB per piece) and the combine pass cost more than the
    // idle-SM tail they remove, and the tensor-heavy kernel runs at the power cap anyway.
    std::vector<int> order(n_items);
    for (int w = 0; w < n_items; ++w) order[w] = w;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tiles[a] > tiles[b]; });
    const int grid = std::min(n_items, n_sm);
    s.grid = grid;
    for (int c = 0; c < grid; ++c) {
      s.cta_off[c] = s.n_pieces;
      for (int i = c; i < n_items; i += grid) {
        AttnPiece& p = s.pieces[s.n_pieces++];
        p.item = order[i];
        p.j0 = 0;
        p.j1 = tiles[order[i]];
        p.part = -1;
        n_pieces_of[order[i]] = 1;
      }
    }
    s.cta_off[grid] = s.n_pieces;
  } else {
    // Few items (e.g. one long-context query): split every item's key range into up to
    // n_sm / n_items near-equal pieces, one piece per CTA; the combine pass merges them.
    const int k = n_sm / n_items;
    int c = 0;
    for (int w = 0; w < n_items; ++w) {
      const int np = std::max(1, std::min(k, tiles[w]));
      for (int q = 0; q < np; ++q) {
        s.cta_off[c++] = s.n_pieces;
        AttnPiece& p = s.pieces[s.n_pieces++];
        p.item = w;
        p.j0 = static_cast<int32_t>(static_cast<int64_t>(tiles[w]) * q / np);
        p.j1 = static_cast<int32_t>(static_cast<int64_t>(tiles[w]) * (q + 1) / np);
        p.part = -1;
      }
      n_pieces_of[w] = np;
    }
    s.grid = c;
    s.cta_off[c] = s.n_pieces;
  }
  // partial slots for split items, consecutive per item in sequence order
  int last_item = -1;
  for (int i = 0; i < s.n_pieces; ++i) {
    AttnPiece& p = s.pieces[i];
    if (n_pieces_of[p.item] < 2) continue;
    if (p.item != last_item) {
      AttnCombine& cb = s.combine[s.n_combine++];
      cb.item = p.item;
      cb.part0 = s.n_partials;
      cb.n_part = n_pieces_of[p.item];
      cb.pad = 0;
      last_item = p.item;
    }
    p.part = s.n_partials++;
  }
}

}  // namespace glmx
