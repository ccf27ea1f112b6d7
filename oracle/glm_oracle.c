/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's bookkeeping path.
 * Only tests/ (and bench.py's cpu_baseline leg) may load this; the product never does.
 * Deliberately simple (linear scans, qsort): it is a checker, not an implementation. */
#define _POSIX_C_SOURCE 200809L
#include "glm_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* fnv.hpp:9-16 */
uint64_t glmo_fnv1a(const char* data, size_t len, uint64_t seed) {
  uint64_t h = seed;
  for (size_t i = 0; i < len; ++i) {
    h ^= (unsigned char)data[i];
    h *= 1099511628211ULL;
  }
  return h;
}

/* fnv.hpp:18-25 — the eight little-endian bytes of value */
uint64_t glmo_fnv1a_u64(uint64_t value, uint64_t seed) {
  uint64_t h = seed;
  for (int i = 0; i < 8; ++i) {
    h ^= (value >> (i * 8)) & 0xff;
    h *= 1099511628211ULL;
  }
  return h;
}

/* cache.cpp:13-21 — seed 1469598103934665603 (not the FNV basis), root parent 0xb10c0000c0ffee,
 * separator fnv1a_u64(0x1f) after every token. */
static uint64_t block_hash(int has_parent, uint64_t parent, const char* bytes, const uint64_t* offs,
                           size_t begin, size_t end) {
  uint64_t h = glmo_fnv1a_u64(has_parent ? parent : 0xb10c0000c0ffeeULL, 1469598103934665603ULL);
  for (size_t i = begin; i < end; ++i) {
    h = glmo_fnv1a(bytes + offs[i], offs[i + 1] - offs[i], h);
    h = glmo_fnv1a_u64(0x1f, h);
  }
  return h;
}

/* cache.cpp:31-40 — full blocks only, root first */
size_t glmo_chain_ids(const char* bytes, const uint64_t* offs, size_t n_tok, size_t B,
                      uint64_t* out) {
  size_t n = 0;
  uint64_t parent = 0;
  int has_parent = 0;
  for (size_t b = 0; (b + 1) * B <= n_tok; ++b) {
    uint64_t id = block_hash(has_parent, parent, bytes, offs, b * B, (b + 1) * B);
    out[n++] = id;
    parent = id;
    has_parent = 1;
  }
  return n;
}

/* ------------------------------------------------------------------ KvCacheState (cache.hpp) */
typedef struct {
  uint64_t id;
  int tier;
  uint64_t last_used;
  char* session;
} blk_t;

struct glmo_kv {
  size_t cap, B;
  int policy; /* 0 Priority, 1 PlainLru */
  blk_t* blk;
  size_t n, alloc;
  uint64_t clock;
  int64_t hits, misses, ev[4];
};

glmo_kv* glmo_kv_create(size_t capacity, size_t block_tokens, int policy) {
  if (block_tokens == 0) return NULL; /* cache.cpp:28 ConfigError */
  glmo_kv* kv = (glmo_kv*)calloc(1, sizeof(glmo_kv));
  kv->cap = capacity;
  kv->B = block_tokens;
  kv->policy = policy;
  return kv;
}

void glmo_kv_destroy(glmo_kv* kv) {
  if (!kv) return;
  for (size_t i = 0; i < kv->n; ++i) free(kv->blk[i].session);
  free(kv->blk);
  free(kv);
}

static long find_blk(const glmo_kv* kv, uint64_t id) {
  for (size_t i = 0; i < kv->n; ++i)
    if (kv->blk[i].id == id) return (long)i;
  return -1;
}

static void insert_blk(glmo_kv* kv, uint64_t id, int tier, uint64_t lu, const char* session) {
  if (kv->n == kv->alloc) {
    kv->alloc = kv->alloc ? 2 * kv->alloc : 64;
    kv->blk = (blk_t*)realloc(kv->blk, kv->alloc * sizeof(blk_t));
  }
  blk_t* b = &kv->blk[kv->n++];
  b->id = id;
  b->tier = tier;
  b->last_used = lu;
  b->session = strdup(session);
}

static void erase_blk(glmo_kv* kv, long i) {
  free(kv->blk[i].session);
  kv->blk[i] = kv->blk[kv->n - 1];
  kv->n--;
}

/* cache.cpp:42-52 */
static int strongest_tier_over(const uint64_t* tiers3, size_t n_tiers, size_t begin, size_t end) {
  int best = 3;
  for (size_t i = 0; i < n_tiers; ++i) {
    uint64_t rb = tiers3[3 * i], re = tiers3[3 * i + 1];
    int t = (int)tiers3[3 * i + 2];
    if (re <= begin || rb >= end) continue;
    if (t < best) best = t;
  }
  return best;
}

typedef struct {
  int tier;
  uint64_t last_used;
  uint64_t id;
} cand_t;
static int g_cmp_policy;
static int cand_cmp(const void* pa, const void* pb) {
  const cand_t* a = (const cand_t*)pa;
  const cand_t* b = (const cand_t*)pb;
  if (g_cmp_policy == 0 && a->tier != b->tier) return a->tier > b->tier ? -1 : 1;
  if (a->last_used != b->last_used) return a->last_used < b->last_used ? -1 : 1;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  return 0;
}

/* cache.cpp:109-148 */
int glmo_kv_evict(glmo_kv* kv, size_t n, uint64_t* out, size_t cap, size_t* n_out) {
  *n_out = 0;
  if (n == 0) return 0;
  cand_t* c = (cand_t*)malloc((kv->n + 1) * sizeof(cand_t));
  size_t nc = 0;
  for (size_t i = 0; i < kv->n; ++i) {
    if (kv->policy == 0 && kv->blk[i].tier == 0) continue;
    c[nc].tier = kv->blk[i].tier;
    c[nc].last_used = kv->blk[i].last_used;
    c[nc].id = kv->blk[i].id;
    nc++;
  }
  if (nc < n) {
    free(c);
    return 2;
  }
  g_cmp_policy = kv->policy;
  qsort(c, nc, sizeof(cand_t), cand_cmp);
  for (size_t i = 0; i < n; ++i) {
    if (i < cap) out[i] = c[i].id;
    kv->ev[c[i].tier]++;
    erase_blk(kv, find_blk(kv, c[i].id));
  }
  *n_out = n;
  free(c);
  return 0;
}

/* cache.cpp:54-107 */
int glmo_kv_prefill(glmo_kv* kv, const char* bytes, const uint64_t* offs, size_t n_tok,
                    const uint64_t* tiers3, size_t n_tiers, const char* session, uint64_t* rep3,
                    uint64_t* evicted, size_t ev_cap, size_t* n_ev) {
  size_t expect = 0;
  for (size_t i = 0; i < n_tiers; ++i) {
    if (tiers3[3 * i] != expect || tiers3[3 * i + 1] < tiers3[3 * i]) return 1;
    expect = tiers3[3 * i + 1];
  }
  if (expect != n_tok) return 1;
  size_t B = kv->B;
  size_t full = n_tok / B;
  uint64_t* ids = (uint64_t*)malloc((full + 1) * sizeof(uint64_t));
  glmo_chain_ids(bytes, offs, n_tok, B, ids);
  rep3[0] = rep3[1] = 0;
  rep3[2] = n_tok - full * B;
  *n_ev = 0;
  size_t hit = 0;
  while (hit < full && find_blk(kv, ids[hit]) >= 0) ++hit;
  rep3[0] = hit * B;
  kv->hits += (int64_t)hit;
  for (size_t b = 0; b < hit; ++b) {
    blk_t* blk = &kv->blk[find_blk(kv, ids[b])];
    blk->last_used = ++kv->clock;
    int want = strongest_tier_over(tiers3, n_tiers, b * B, (b + 1) * B);
    if (want < blk->tier) blk->tier = want;
  }
  int status = 0;
  for (size_t b = hit; b < full; ++b) {
    rep3[1] += B;
    kv->misses++;
    int tier = strongest_tier_over(tiers3, n_tiers, b * B, (b + 1) * B);
    long at = find_blk(kv, ids[b]);
    if (at >= 0) { /* orphan: refresh only (cache.cpp:87-93) */
      kv->blk[at].last_used = ++kv->clock;
      if (tier < kv->blk[at].tier) kv->blk[at].tier = tier;
      continue;
    }
    if (kv->n >= kv->cap) {
      size_t need = kv->n - kv->cap + 1;
      uint64_t* tmp = (uint64_t*)malloc(need * sizeof(uint64_t));
      size_t got = 0;
      status = glmo_kv_evict(kv, need, tmp, need, &got);
      for (size_t i = 0; i < got; ++i) {
        if (*n_ev < ev_cap) evicted[*n_ev] = tmp[i];
        (*n_ev)++;
      }
      free(tmp);
      if (status) break; /* partial state stays (cache.cpp:94-97 throws mid-loop) */
    }
    insert_blk(kv, ids[b], tier, ++kv->clock, tier == 0 ? "" : session);
  }
  free(ids);
  if (status) { /* the reference returns no report on throw */
    rep3[0] = rep3[1] = rep3[2] = 0;
    *n_ev = 0;
  }
  return status;
}

/* cache.cpp:150-153 */
void glmo_kv_set_tier(glmo_kv* kv, const char* session, int from, int to) {
  for (size_t i = 0; i < kv->n; ++i)
    if (strcmp(kv->blk[i].session, session) == 0 && kv->blk[i].tier == from) kv->blk[i].tier = to;
}

/* cache.cpp:167-176 */
void glmo_kv_force_insert(glmo_kv* kv, uint64_t id, int tier, uint64_t last_used,
                          const char* session) {
  long at = find_blk(kv, id);
  if (at >= 0) erase_blk(kv, at);
  insert_blk(kv, id, tier, last_used, session);
  if (last_used > kv->clock) kv->clock = last_used;
}

void glmo_kv_counters(const glmo_kv* kv, int64_t* out6) {
  out6[0] = kv->hits;
  out6[1] = kv->misses;
  for (int t = 0; t < 4; ++t) out6[2 + t] = kv->ev[t];
}

static int u64_cmp(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y);
}

/* cache.cpp:160-165 (sorted by id) */
size_t glmo_kv_resident(const glmo_kv* kv, uint64_t* ids, int32_t* tiers, uint64_t* last_used,
                        size_t cap) {
  uint64_t* s = (uint64_t*)malloc((kv->n + 1) * sizeof(uint64_t));
  for (size_t i = 0; i < kv->n; ++i) s[i] = kv->blk[i].id;
  qsort(s, kv->n, sizeof(uint64_t), u64_cmp);
  for (size_t i = 0; i < kv->n && i < cap; ++i) {
    const blk_t* b = &kv->blk[find_blk(kv, s[i])];
    ids[i] = b->id;
    tiers[i] = b->tier;
    last_used[i] = b->last_used;
  }
  free(s);
  return kv->n;
}

/* ------------------------------------------------------------------ node_info + render_chunk */
typedef struct {
  char* buf;
  size_t len, cap;
} sbuf;
static void sput(sbuf* s, const char* t, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    if (s->len < s->cap) s->buf[s->len] = t[i];
    s->len++;
  }
}
static void sputs(sbuf* s, const char* t) { sput(s, t, strlen(t)); }

typedef struct {
  const char* k;
  const char* v;
} pair_t;
static int pair_cmp(const void* pa, const void* pb) {
  const pair_t* a = (const pair_t*)pa;
  const pair_t* b = (const pair_t*)pb;
  int c = strcmp(a->k, b->k); /* std::string < is byte-wise (unsigned) like strcmp */
  if (c) return c;
  return strcmp(a->v, b->v);
}

/* retriever.cpp:34-41 + the "{k:v, ...}" part of render_chunk (retriever.cpp:10-20) */
static void render_entry(const glmo_graph* g, int32_t v, sbuf* s) {
  size_t a0 = g->attr_off[v], a1 = g->attr_off[v + 1];
  size_t n = a1 - a0 + 1;
  pair_t* p = (pair_t*)malloc(n * sizeof(pair_t));
  for (size_t i = a0; i < a1; ++i) {
    p[i - a0].k = g->attr_keys[i];
    p[i - a0].v = g->attr_vals[i];
  }
  p[n - 1].k = "type";
  p[n - 1].v = g->types[v];
  qsort(p, n, sizeof(pair_t), pair_cmp);
  sputs(s, g->ids[v]);
  sputs(s, " {");
  for (size_t i = 0; i < n; ++i) {
    if (i) sputs(s, ", ");
    sputs(s, p[i].k);
    sputs(s, ":");
    sputs(s, p[i].v);
  }
  sputs(s, "}");
  free(p);
}

static int i32_cmp(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return x < y ? -1 : (x > y);
}

typedef struct {
  int32_t node;
  int64_t w;
  size_t pos;
} wnode_t;
static int wnode_cmp(const void* pa, const void* pb) { /* stable: pos breaks remaining ties */
  const wnode_t* a = (const wnode_t*)pa;
  const wnode_t* b = (const wnode_t*)pb;
  if (a->w != b->w) return a->w > b->w ? -1 : 1;
  if (a->node != b->node) return a->node < b->node ? -1 : 1; /* ids ascending == index order */
  return a->pos < b->pos ? -1 : (a->pos > b->pos);
}

/* graph_store.cpp:209-213 (all edges, both directions, multi-edges counted, self-loop twice) */
static int64_t total_degree(const glmo_graph* g, int32_t v) {
  int64_t d = 0;
  for (size_t e = 0; e < g->n_edges; ++e) d += (g->src[e] == v) + (g->dst[e] == v);
  return d;
}

/* graph_store.cpp:215-224 restricted to etype; max over incident types (retriever.cpp:100-105) */
static int64_t by_edge_type(const glmo_graph* g, int32_t v) {
  int64_t best = 0;
  for (size_t e = 0; e < g->n_edges; ++e) {
    if (g->src[e] != v && g->dst[e] != v) continue;
    int32_t t = g->etype[e];
    int64_t d = 0;
    for (size_t f = 0; f < g->n_edges; ++f)
      if (g->etype[f] == t) d += (g->src[f] == v) + (g->dst[f] == v);
    if (d > best) best = d;
  }
  return best;
}

/* retriever.cpp:74-121 then render_chunk retriever.cpp:9-30 */
int64_t glmo_node_info_rendered(const glmo_graph* g, int32_t node, int k, int weight_mode,
                                int directed, char* buf, size_t cap) {
  if (node < 0 || (size_t)node >= g->n_nodes) return -1;
  int32_t* nb = (int32_t*)malloc((2 * g->n_edges + 1) * sizeof(int32_t));
  size_t nn = 0;
  for (size_t e = 0; e < g->n_edges; ++e) {
    if (g->src[e] == node) nb[nn++] = g->dst[e];
    if (!directed && g->dst[e] == node) nb[nn++] = g->src[e];
  }
  qsort(nb, nn, sizeof(int32_t), i32_cmp);
  size_t u = 0;
  for (size_t i = 0; i < nn; ++i)
    if (u == 0 || nb[u - 1] != nb[i]) nb[u++] = nb[i];
  wnode_t* w = (wnode_t*)malloc((u + 1) * sizeof(wnode_t));
  for (size_t i = 0; i < u; ++i) {
    w[i].node = nb[i];
    w[i].w = weight_mode == 0 ? total_degree(g, nb[i]) : by_edge_type(g, nb[i]);
    w[i].pos = i;
  }
  qsort(w, u, sizeof(wnode_t), wnode_cmp);
  size_t take = k < 0 ? 0 : (size_t)k;
  if (take > u) take = u;
  sbuf s = {buf, 0, cap};
  sputs(&s, "[Node:");
  render_entry(g, node, &s);
  sputs(&s, "]\n[neighbours:");
  for (size_t i = 0; i < take; ++i) {
    if (i) sputs(&s, ",");
    sputs(&s, "(");
    render_entry(g, w[i].node, &s);
    sputs(&s, ")");
  }
  sputs(&s, "]");
  free(nb);
  free(w);
  return (int64_t)s.len;
}
