// Persistent-CTA schedule for the K3 attention kernel (pure host C++).
//
// The kernel's unit of work is a piece: a key-tile range [j0, j1) of one item (request, 64-token
// query block, kv head); every CTA walks its own list of pieces.  With at least n_sm / 2 items,
// whole items go longest-first to the least-loaded CTA (LPT), unless that leaves a long tail
// (makespan > 1.3 x total / n_sm, e.g. 168 long items on 148 SMs), in which case the flattened
// tile sequence is cut into n_sm equal ranges (stream-K).  With fewer items (a single
// long-context query has only 8-16), each item's key range is split into up to n_sm / n_items
// pieces (only when the longest item has >= 8 key tiles: shorter ones run whole).  Split pieces
// write an unnormalised partial (O, m, l) and a combine pass merges them.
#pragma once

#include <cstddef>
#include <cstdint>

namespace glmx {

struct AttnPiece {
  int32_t item;  // item index w: work entry w / Hkv, kv head w % Hkv
  int32_t j0;    // first key tile
  int32_t j1;    // one past the last key tile
  int32_t part;  // partial slot, or -1: the piece is the whole item (normalised store)
};

struct AttnCombine {
  int32_t item;
  int32_t part0;   // first partial slot (slots of one item are consecutive)
  int32_t n_part;
  int32_t pad;
};

struct AttnSchedule {
  AttnPiece* pieces;   // capacity: n_items + n_sm
  // partner of piece i for query-tile slot 1 (item = -1: none).  Two single-tile items (<= 32
  // tokens, one 128-row query tile each) are paired into one piece so both softmax warpgroups
  // work: slot 0 runs pieces[i] (its first query tile), slot 1 partners[i].  Pairs are never split.
  AttnPiece* partners;  // capacity: n_items + n_sm
  int32_t* cta_off;    // capacity: n_sm + 1 (pieces of CTA c: [cta_off[c], cta_off[c+1]))
  AttnCombine* combine;  // capacity: n_sm
  int n_pieces = 0, grid = 0, n_combine = 0, n_partials = 0;
  int64_t total_tiles = 0;
};

// Bytes of the packed schedule region for `max_items` items (pieces | cta_off | combine, 16 B
// aligned sections) and the section offsets.
size_t attn_sched_bytes(int max_items, int n_sm, size_t* off_pieces, size_t* off_cta,
                        size_t* off_combine, size_t* off_partners);

// Key tiles of an item: the last query row of the item's 64-token block sees keys
// [0, ctx - qlen + min(t0 + tokens_per_item, qlen)).
int attn_item_tiles(int t0, int q_len, int ctx_len, int tokens_per_item, int keys_per_tile);

// work[i] = (request, first token), items w = i * Hkv + kv head.  An item uses one query tile
// when its block holds <= tokens_per_item / 2 tokens.  max_partials bounds the
// partial workspace (2 * n_sm always suffices).
void build_attn_schedule(const int32_t* work_xy, int n_work, int Hkv, const int32_t* q_len,
                         const int32_t* ctx_len, int tokens_per_item, int keys_per_tile, int n_sm,
                         AttnSchedule& s);

}  // namespace glmx
