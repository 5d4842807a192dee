/* oracle.h — plain, slow, obviously-correct CPU oracle for the eLLM KV-traffic hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so. The product library
 * (libellm.so) shares no code, header, table or constant with this file.
 *
 * Paper: "eLLM: Elastic Memory Management Framework for Efficient LLM Serving",
 * arXiv 2506.15155, /root/reference/PAPER.md (cited as P:<line>).
 *
 * What it models (operations O1-O9):
 *   - a unified pool of physical chunks labelled KV or ACT,
 *   - per-request KV kept CONTIGUOUS by logical position (the logical truth; the
 *     paper's KV eTensor "ensures the logical continuity of the KV cache"),
 *   - a LINEAR page table per request: logical chunk i -> DEV c | HOST h | UNMAPPED,
 *   - physical chunk / host-slot byte images written only through the page table,
 *     with the chunk layout [L][2][Hkv][T][d] bf16 (reading R1),
 *   - textbook softmax attention in fp64 (attention over the accumulated KV;
 *     "without sacrificing precision" -> exact, no approximation).
 *
 * Error codes are the values the boundary spec (include/ellm.h) fixes; they are
 * retyped here from the spec, not included from it.
 */
#ifndef ELLM_ORACLE_H
#define ELLM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum {
  EO_OK = 0, EO_ERR_INVALID_ARG = -1, EO_ERR_OUT_OF_RANGE = -2, EO_ERR_NO_CHUNKS = -3,
  EO_ERR_HOST_FULL = -4, EO_ERR_NOT_RESIDENT = -5, EO_ERR_NOT_MAPPED = -6,
  EO_ERR_ALREADY_MAPPED = -7, EO_ERR_IN_USE = -8
};

typedef struct {
  int32_t n_layers, n_heads_q, n_heads_kv, head_dim, tokens_per_chunk;
  int64_t max_chunks, initial_chunks;
  int32_t max_requests, max_chunks_per_request;
  int64_t host_slots;
} eo_config;

typedef struct eo_state eo_state;

eo_state* eo_create(const eo_config* cfg);           /* O1; NULL on a bad config */
void eo_destroy(eo_state* s);
int eo_reserve(eo_state* s, int32_t n, const int32_t* reqs, const int32_t* n_new);             /* O2 */
int eo_append(eo_state* s, int32_t layer, int32_t n, const int32_t* reqs, const int32_t* n_new,
              const uint16_t* k_new, const uint16_t* v_new);                                   /* O3 */
int eo_attention(eo_state* s, int32_t layer, int32_t n, const int32_t* reqs, const uint16_t* q,
                 double scale, double* out, int32_t through_table);                            /* O4 */
/* O12 (f4): causal attention of the last n_q[i] positions of each listed request (n_q in
 * [1, len], else INVALID_ARG). q [sum n_q][Hq][d] bf16 bits, rows in list order then position
 * order; out [sum n_q][Hq][d] fp64. Query k of request i (position P = len - n_q + k) attends
 * keys 0..P. Residency / range errors as eo_attention. */
int eo_prefill_attention(eo_state* s, int32_t layer, int32_t n, const int32_t* reqs,
                         const int32_t* n_q, const uint16_t* q, double scale, double* out,
                         int32_t through_table);                                              /* O12 */
int eo_deflate(eo_state* s, int32_t n, const int32_t* ids, int32_t* slots_out);               /* O5 */
int eo_inflate(eo_state* s, int32_t n, const int32_t* slots, int32_t* ids_out);               /* O6 */
int eo_migrate(eo_state* s, int32_t n, const int32_t* src, const int32_t* dst);               /* O7 */
int eo_release(eo_state* s, int32_t req);                                                      /* O8 */
int eo_grow(eo_state* s, int64_t n);                                                           /* O9 */
int eo_shrink(eo_state* s, int64_t n);                                                         /* O9 */
/* f3: activation eTensor slots in the unified pool.
 * O10 act_alloc: n consecutive ACT chunks outside any slot, the run with the highest last id;
 *   *first_out = its first chunk. n <= 0 -> INVALID_ARG; no run -> NO_CHUNKS.
 * O11 act_free: end the slot starting at `first` (chunks stay ACT, now reclaimable by grow).
 * grow (O9) skips chunks inside live slots. */
int eo_act_alloc(eo_state* s, int64_t n, int64_t* first_out);                                  /* O10 */
int eo_act_free(eo_state* s, int64_t first);                                                   /* O11 */
int64_t eo_act_used(const eo_state* s);   /* chunks inside live activation slots */
/* out[5] = {kv_free, kv_used, act, host_free, host_used} */
int eo_stats(const eo_state* s, int64_t* out);
/* entries: >=0 device chunk id, -1 unmapped, <=-2 host slot h encoded as -(h+2) */
int eo_get_table(const eo_state* s, int32_t req, int32_t* entries, int32_t cap, int32_t* n_out, int32_t* len_out);
int eo_read_chunk(const eo_state* s, int64_t chunk, uint8_t* dst);     /* chunk_bytes; never-written bytes read 0 */
int eo_read_host_slot(const eo_state* s, int64_t slot, uint8_t* dst);  /* chunk_bytes */
int64_t eo_chunk_bytes(const eo_state* s);
/* 0 if I1-I7 hold, else the number of the first violated invariant */
int eo_check_invariants(const eo_state* s);

/* Stateless textbook attention for one request, one layer, fp64:
 * q [Hq][d] bf16 bits, k/v [len][Hkv][d] bf16 bits (token-major, contiguous),
 * out [Hq][d] fp64.  q-head h reads kv-head h / (Hq/Hkv). Uses OpenMP over heads
 * when built with -fopenmp. */
int eo_attention_contig(int32_t n_heads_q, int32_t n_heads_kv, int32_t head_dim, int32_t len,
                        const uint16_t* q, const uint16_t* k, const uint16_t* v, double scale,
                        double* out);
int eo_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
