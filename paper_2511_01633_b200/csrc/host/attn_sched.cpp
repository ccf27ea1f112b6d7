#include "attn_sched.hpp"

#include <algorithm>
#include <functional>
#include <queue>
#include <tuple>
#include <vector>

namespace glmx {

namespace {
size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

void stream_k_cut(const int32_t* work_xy, int Hkv, const std::vector<int>& tiles_of, int n_sm,
                  AttnSchedule& s, std::vector<int>& n_pieces_of) {
  const int n_items = static_cast<int>(tiles_of.size());
  std::vector<int> order(n_items);
  for (int w = 0; w < n_items; ++w) order[w] = w;
  auto key = [&](int w) {
    return std::make_tuple(work_xy[2 * (w / Hkv)], w % Hkv, work_xy[2 * (w / Hkv) + 1]);
  };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key(a) < key(b); });
  std::vector<int64_t> start(n_items + 1, 0);
  for (int i = 0; i < n_items; ++i) start[i + 1] = start[i] + tiles_of[order[i]];
  const int64_t W = start[n_items];
  const int grid = static_cast<int>(std::min<int64_t>(n_sm, W));
  const int64_t share = (W + grid - 1) / grid;
  const int64_t snap = std::max<int64_t>(1, share / 8);
  std::vector<int64_t> bnd(grid + 1);
  bnd[0] = 0;
  bnd[grid] = W;
  int i = 0;
  for (int c = 1; c < grid; ++c) {
    int64_t b = W * c / grid;
    while (i < n_items && start[i + 1] <= b) ++i;
    if (i < n_items) {
      if (b - start[i] <= snap) b = start[i];
      else if (start[i + 1] - b <= snap) b = start[i + 1];
    }
    bnd[c] = std::max(b, bnd[c - 1]);
  }
  s.grid = grid;
  i = 0;
  for (int c = 0; c < grid; ++c) {
    s.cta_off[c] = s.n_pieces;
    int64_t t = bnd[c];
    while (t < bnd[c + 1]) {
      while (start[i + 1] <= t) ++i;
      const int64_t e = std::min(bnd[c + 1], start[i + 1]);
      AttnPiece& p = s.pieces[s.n_pieces++];
      p.item = order[i];
      p.j0 = static_cast<int32_t>(t - start[i]);
      p.j1 = static_cast<int32_t>(e - start[i]);
      p.part = -1;
      ++n_pieces_of[order[i]];
      t = e;
    }
  }
  s.cta_off[grid] = s.n_pieces;
}
}  // namespace

size_t attn_sched_bytes(int max_items, int n_sm, size_t* off_pieces, size_t* off_cta,
                        size_t* off_combine, size_t* off_partners) {
  size_t o = 0;
  if (off_pieces) *off_pieces = o;
  o = align16(o + static_cast<size_t>(max_items + n_sm) * sizeof(AttnPiece));
  if (off_partners) *off_partners = o;
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
  bool paired = false;
  const int64_t max_tiles = *std::max_element(tiles.begin(), tiles.end());
  // split only long items: below ~8 key tiles the partial traffic + combine pass costs more
  // than the idle SMs (decode steps over short contexts)
  if (n_items * 2 > n_sm || max_tiles < 8) {
    // Enough items to occupy the SMs: whole items, longest first, each to the least-loaded of
    // min(units, n_sm) persistent CTAs (LPT; equal items reduce to round-robin).  A unit is a
    // two-tile item, or two single-tile items of similar length paired into one piece.
    // Pairs are formed only from short single-tile items (<= kPairMaxTiles key tiles): there the
    // per-tile softmax -> PV -> S chain is latency-bound; a pair of long items streams two K/V
    // sequences per CTA and hits the L2 throughput limit that one shared stream avoids.
    constexpr int kPairMaxTiles = 16;
    std::vector<int> single, twin, lone;
    for (int w = 0; w < n_items; ++w) {
      const int r = work_xy[2 * (w / Hkv)], t0 = work_xy[2 * (w / Hkv) + 1];
      if (!s.partners || q_len[r] - t0 > tokens_per_item / 2) twin.push_back(w);
      else if (tiles[w] <= kPairMaxTiles) single.push_back(w);
      else lone.push_back(w);
    }
    auto longer = [&](int a, int b) { return tiles[a] > tiles[b]; };
    std::stable_sort(single.begin(), single.end(), longer);
    using Unit = std::pair<int, int>;  // (item, partner or -1)
    // Cost model per key tile, in quarter tiles of a two-query-tile step: a lone single-tile item
    // runs its softmax/MMA chain unoverlapped at ~3/4 of a full step; a pair costs a full step.
    std::vector<char> is_single(n_items, 0);
    for (int w : single) is_single[w] = 1;
    for (int w : lone) is_single[w] = 1;
    auto cost = [&](const Unit& u) -> int64_t {
      if (u.second >= 0) return 4 * std::max(tiles[u.first], tiles[u.second]);
      return (is_single[u.first] ? 3 : 4) * static_cast<int64_t>(tiles[u.first]);
    };
    struct Plan {
      std::vector<std::vector<Unit>> mine;
      std::vector<int64_t> load;
      int64_t makespan = 0;
    };
    // the shortest n_pair single-tile items are paired with their length neighbours, the rest
    // run alone (a long lone item may set the makespan, pairing it would only lengthen it)
    auto lpt = [&](size_t n_pair) {
      std::vector<Unit> units;
      for (int w : twin) units.push_back({w, -1});
      for (int w : lone) units.push_back({w, -1});
      const size_t n_alone = single.size() - n_pair;
      for (size_t i = 0; i < n_alone; ++i) units.push_back({single[i], -1});
      for (size_t i = n_alone; i < single.size(); i += 2)
        units.push_back({single[i], i + 1 < single.size() ? single[i + 1] : -1});
      std::stable_sort(units.begin(), units.end(),
                       [&](const Unit& a, const Unit& b) { return cost(a) > cost(b); });
      Plan pl;
      const int grid = std::min(static_cast<int>(units.size()), n_sm);
      pl.mine.resize(grid);
      pl.load.assign(grid, 0);
      using Slot = std::pair<int64_t, int>;  // (load, cta): min-heap, ties to the lower CTA
      std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
      for (int c = 0; c < grid; ++c) heap.push({0, c});
      for (const auto& u : units) {
        auto [l, c] = heap.top();
        heap.pop();
        pl.mine[c].push_back(u);
        pl.load[c] = l + cost(u);
        heap.push({pl.load[c], c});
      }
      pl.makespan = *std::max_element(pl.load.begin(), pl.load.end());
      return pl;
    };
    Plan plan = lpt(0);
    if (single.size() >= 2) {
      for (int f = 1; f <= 4; ++f) {  // 1/4, 1/2, 3/4, all of them paired (even counts)
        Plan pp = lpt(single.size() * f / 4 & ~size_t(1));
        if (pp.makespan < plan.makespan) plan = std::move(pp);  // ties: fewer pairs
      }
    }
    const int grid = static_cast<int>(plan.mine.size());
    auto& mine = plan.mine;
    std::vector<int64_t> load(grid);
    for (int c = 0; c < grid; ++c) load[c] = plan.load[c] / 4;
    const int64_t makespan = *std::max_element(load.begin(), load.end());
    const double ideal = static_cast<double>(s.total_tiles) / n_sm;
    if (makespan > 1.3 * ideal && max_tiles >= 16) {
      // A long tail (e.g. 168 long items on 148 SMs: two waves): cut the flattened tile sequence
      // into n_sm equal ranges instead (stream-K).  Items ordered by (request, kv head, first
      // token) so the query blocks reading the same pages run on neighbouring CTAs at the same
      // time; boundaries within share/8 tiles of an item edge snap to it.
      stream_k_cut(work_xy, Hkv, tiles, n_sm, s, n_pieces_of);
    } else {
      paired = s.partners != nullptr;
      s.grid = grid;
      for (int c = 0; c < grid; ++c) {
        s.cta_off[c] = s.n_pieces;
        for (const auto& u : mine[c]) {
          if (paired) s.partners[s.n_pieces] = AttnPiece{u.second, 0, u.second < 0 ? 0 : tiles[u.second], -1};
          AttnPiece& p = s.pieces[s.n_pieces++];
          p.item = u.first;
          p.j0 = 0;
          p.j1 = tiles[u.first];
          p.part = -1;
          n_pieces_of[u.first] = 1;
          if (u.second >= 0) n_pieces_of[u.second] = 1;
        }
      }
      s.cta_off[grid] = s.n_pieces;
    }
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
  if (s.partners && !paired)
    for (int i = 0; i < s.n_pieces; ++i) s.partners[i] = AttnPiece{-1, 0, 0, -1};
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
