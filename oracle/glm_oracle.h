/* TEST INFRASTRUCTURE ONLY — CPU restatement (plain C) of the reference's hot-path bookkeeping.
 * Used by tests/ as the checker; never linked into the product. Each function cites the
 * reference file:line it restates (paths under /root/reference/proj).
 *
 * Parity pinning: checked against (a) the SURVEY Appendix C / SPEC golden vectors committed in
 * tests/golden/, and (b) the reference itself compiled into oracle/_ref/libglmref.so. */
#ifndef GLM_ORACLE_H
#define GLM_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t glmo_fnv1a(const char* data, size_t len, uint64_t seed);
uint64_t glmo_fnv1a_u64(uint64_t value, uint64_t seed);
size_t glmo_chain_ids(const char* bytes, const uint64_t* offs, size_t n_tok, size_t block_tokens,
                      uint64_t* out);

typedef struct glmo_kv glmo_kv;
glmo_kv* glmo_kv_create(size_t capacity, size_t block_tokens, int policy);
void glmo_kv_destroy(glmo_kv* kv);
/* status: 0 ok, 1 bad tier map (GlmError), 2 CacheExhausted */
int glmo_kv_prefill(glmo_kv* kv, const char* bytes, const uint64_t* offs, size_t n_tok,
                    const uint64_t* tiers3, size_t n_tiers, const char* session, uint64_t* rep3,
                    uint64_t* evicted, size_t ev_cap, size_t* n_ev);
int glmo_kv_evict(glmo_kv* kv, size_t n, uint64_t* out, size_t cap, size_t* n_out);
void glmo_kv_set_tier(glmo_kv* kv, const char* session, int from, int to);
void glmo_kv_force_insert(glmo_kv* kv, uint64_t id, int tier, uint64_t last_used,
                          const char* session);
void glmo_kv_counters(const glmo_kv* kv, int64_t* out6);
size_t glmo_kv_resident(const glmo_kv* kv, uint64_t* ids, int32_t* tiers, uint64_t* last_used,
                        size_t cap);

/* node_info + render_chunk over a flat graph description:
 *   nodes 0..n-1 ascending by id bytes; node_text[i] = "<id>" ; attrs are pre-rendered (key,value)
 *   pairs per node (values rendered per attr.hpp:28-48 by the caller) plus node type;
 *   edges (src, dst, etype) as node indices + etype ids. */
typedef struct {
  size_t n_nodes;
  const char* const* ids;
  const char* const* types;
  const size_t* attr_off; /* n_nodes+1 */
  const char* const* attr_keys;
  const char* const* attr_vals;
  size_t n_edges;
  const int32_t* src;
  const int32_t* dst;
  const int32_t* etype;
} glmo_graph;
/* returns rendered length, or -1 if node out of range; writes up to cap bytes */
int64_t glmo_node_info_rendered(const glmo_graph* g, int32_t node, int k, int weight_mode,
                                int directed, char* buf, size_t cap);

#ifdef __cplusplus
}
#endif
#endif
