// oracle.cpp — plain CPU oracle for the eLLM KV-traffic hot path (see oracle.h).
//
// TEST INFRASTRUCTURE ONLY: never linked into, loaded by, or called from the product
// path (paper_2506_15155_b200/). fp64 for all floating point; no blocking, no fusion.
//
// Parity pins (tests/test_oracle_*.py):
//   - attention: numpy brute-force textbook softmax (oracle/brute.py) + special cases
//     (len=1, equal keys, constant V, needle, MHA, head permutation);
//   - tables: closed forms for C1 (SURVEY §8(c) "What pins each part");
//   - state machine: invariants I1-I6 after every op of long random op sequences;
//   - chunk layout: hand-written golden offsets (tests/golden/layout_c1.json).
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <set>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr int32_t UNMAPPED = -1;
inline bool is_dev(int32_t e) { return e >= 0; }
inline bool is_host(int32_t e) { return e <= -2; }
inline int32_t host_of(int32_t e) { return -e - 2; }
inline int32_t enc_host(int32_t h) { return -(h + 2); }

// bf16 bits -> double: a bf16 is the high half of an fp32, so this is exact.
inline double bf16_to_double(uint16_t b) {
  uint32_t u = uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return double(f);
}

enum Owner : uint8_t { KV = 0, ACT = 1 };

struct Request {
  int64_t len = 0;                 // logical tokens (KV grows with generation)
  int32_t pending = 0;             // n_new of the latest reserve (the positions append writes)
  std::vector<int32_t> pt;         // linear page table (size max_chunks_per_request)
  std::vector<uint16_t> kv;        // contiguous logical KV [len][L][2][Hkv][d] bf16 bits
  std::vector<uint8_t> written;    // [len][L]: position appended for that layer (I4 domain)
};

}  // namespace

struct eo_state {
  eo_config c;
  int64_t chunk_elems = 0;   // T*L*2*Hkv*d
  int64_t row_elems = 0;     // L*2*Hkv*d (one token, all layers)
  std::vector<uint8_t> owner;     // per chunk: KV / ACT
  std::vector<uint8_t> used;      // per chunk: USED (1) / FREE (0), KV-owned only
  // O10/O11: activation eTensor slots — runs of consecutive ACT chunks
  // holding activations. act_len[c] = slot length if a slot starts at c, else 0;
  // in_act[c] = chunk c belongs to a live activation slot.
  std::vector<int64_t> act_len;
  std::vector<uint8_t> in_act;
  std::vector<uint8_t> hused;     // per host slot
  std::map<int64_t, std::vector<uint16_t>> phys;   // chunk id -> byte image (lazy)
  std::map<int64_t, std::vector<uint16_t>> host;   // host slot -> byte image (lazy)
  std::vector<Request> req;

  std::vector<uint16_t>& phys_img(int64_t c) {
    auto& v = phys[c];
    if (v.empty()) v.assign(size_t(chunk_elems), 0);
    return v;
  }
  std::vector<uint16_t>& host_img(int64_t h) {
    auto& v = host[h];
    if (v.empty()) v.assign(size_t(chunk_elems), 0);
    return v;
  }
  int64_t T() const { return c.tokens_per_chunk; }
  int64_t nchunks_of(int64_t len) const { return (len + T() - 1) / T(); }
  // element offset of (layer, kv, head, row-in-chunk) inside a chunk: layout [L][2][Hkv][T][d]
  int64_t chunk_off(int64_t l, int64_t kv, int64_t h, int64_t t) const {
    return (((l * 2 + kv) * c.n_heads_kv + h) * T() + t) * c.head_dim;
  }
  // element offset inside kv[r]: layout [pos][L][2][Hkv][d]
  int64_t contig_off(int64_t p, int64_t l, int64_t kv, int64_t h) const {
    return (((p * c.n_layers + l) * 2 + kv) * c.n_heads_kv + h) * c.head_dim;
  }
  int64_t count_free_kv() const {
    int64_t n = 0;
    for (size_t i = 0; i < owner.size(); ++i) n += (owner[i] == KV && !used[i]);
    return n;
  }
  int64_t lowest_free_kv() const {
    for (size_t i = 0; i < owner.size(); ++i)
      if (owner[i] == KV && !used[i]) return int64_t(i);
    return -1;
  }
  int64_t lowest_free_host() const {
    for (size_t i = 0; i < hused.size(); ++i)
      if (!hused[i]) return int64_t(i);
    return -1;
  }
  // (request, logical chunk) holding table entry value e, or {-1,-1}
  std::pair<int32_t, int32_t> find_entry(int32_t e) const {
    for (size_t r = 0; r < req.size(); ++r)
      for (size_t i = 0; i < req[r].pt.size(); ++i)
        if (req[r].pt[i] == e) return {int32_t(r), int32_t(i)};
    return {-1, -1};
  }
};

static bool has_dup(int32_t n, const int32_t* a) {
  std::set<int32_t> s(a, a + n);
  return int32_t(s.size()) != n;
}

extern "C" {

int eo_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

eo_state* eo_create(const eo_config* cfg) {
  if (!cfg) return nullptr;
  const eo_config& c = *cfg;
  if (c.n_layers <= 0 || c.n_heads_q <= 0 || c.n_heads_kv <= 0 || c.head_dim <= 0 ||
      c.tokens_per_chunk <= 0 || c.max_chunks <= 0 || c.initial_chunks < 0 ||
      c.initial_chunks > c.max_chunks || c.max_requests <= 0 || c.max_chunks_per_request <= 0 ||
      c.host_slots < 0 || c.n_heads_q % c.n_heads_kv != 0)
    return nullptr;
  eo_state* s = new eo_state();
  s->c = c;
  s->row_elems = int64_t(c.n_layers) * 2 * c.n_heads_kv * c.head_dim;
  s->chunk_elems = s->row_elems * c.tokens_per_chunk;
  // O1: ids 0..C_kv-1 are KV/FREE, the rest ACT.
  s->owner.assign(size_t(c.max_chunks), ACT);
  s->act_len.assign(size_t(c.max_chunks), 0);
  s->in_act.assign(size_t(c.max_chunks), 0);
  s->used.assign(size_t(c.max_chunks), 0);
  for (int64_t i = 0; i < c.initial_chunks; ++i) s->owner[size_t(i)] = KV;
  s->hused.assign(size_t(c.host_slots), 0);
  s->req.resize(size_t(c.max_requests));
  for (auto& r : s->req) r.pt.assign(size_t(c.max_chunks_per_request), UNMAPPED);
  return s;
}

void eo_destroy(eo_state* s) { delete s; }

int64_t eo_chunk_bytes(const eo_state* s) { return s->chunk_elems * 2; }

// O2 — on-demand chunk mapping at write time, prefix-contiguous logical KV,
// all-or-nothing for the whole call: no hold-and-wait.
int eo_reserve(eo_state* s, int32_t n, const int32_t* reqs, const int32_t* n_new) {
  if (n < 0) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (reqs[i] < 0 || reqs[i] >= s->c.max_requests) return EO_ERR_OUT_OF_RANGE;
  if (has_dup(n, reqs)) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (n_new[i] < 0) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i) {
    const Request& R = s->req[size_t(reqs[i])];
    if (s->nchunks_of(R.len + n_new[i]) > s->c.max_chunks_per_request) return EO_ERR_OUT_OF_RANGE;
  }
  for (int32_t i = 0; i < n; ++i) {
    const Request& R = s->req[size_t(reqs[i])];
    if (n_new[i] > 0 && R.len % s->T() != 0 && is_host(R.pt[size_t(R.len / s->T())]))
      return EO_ERR_NOT_RESIDENT;
  }
  int64_t need = 0;
  for (int32_t i = 0; i < n; ++i) {
    const Request& R = s->req[size_t(reqs[i])];
    need += s->nchunks_of(R.len + n_new[i]) - s->nchunks_of(R.len);
  }
  if (need > s->count_free_kv()) return EO_ERR_NO_CHUNKS;
  for (int32_t i = 0; i < n; ++i) {
    Request& R = s->req[size_t(reqs[i])];
    for (int64_t ci = s->nchunks_of(R.len); ci < s->nchunks_of(R.len + n_new[i]); ++ci) {
      int64_t c = s->lowest_free_kv();
      R.pt[size_t(ci)] = int32_t(c);
      s->used[size_t(c)] = 1;
    }
    R.len += n_new[i];
    R.pending = n_new[i];
    R.kv.resize(size_t(R.len * s->row_elems), 0);
    R.written.resize(size_t(R.len * s->c.n_layers), 0);
  }
  return EO_OK;
}

// O3 — the KV cache grows by the generated K/V. Row order of k_new/v_new:
// requests in the given order, positions ascending, then kv-head; each row d bf16.
int eo_append(eo_state* s, int32_t layer, int32_t n, const int32_t* reqs, const int32_t* n_new,
              const uint16_t* k_new, const uint16_t* v_new) {
  if (layer < 0 || layer >= s->c.n_layers) return EO_ERR_OUT_OF_RANGE;
  if (n < 0) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (reqs[i] < 0 || reqs[i] >= s->c.max_requests) return EO_ERR_OUT_OF_RANGE;
  if (has_dup(n, reqs)) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (n_new[i] != s->req[size_t(reqs[i])].pending) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i) {
    const Request& R = s->req[size_t(reqs[i])];
    for (int64_t p = R.len - n_new[i]; p < R.len; ++p)
      if (!is_dev(R.pt[size_t(p / s->T())])) return EO_ERR_NOT_RESIDENT;
  }
  const int64_t Hkv = s->c.n_heads_kv, d = s->c.head_dim;
  int64_t row = 0;
  for (int32_t i = 0; i < n; ++i) {
    Request& R = s->req[size_t(reqs[i])];
    for (int64_t p = R.len - n_new[i]; p < R.len; ++p, ++row) {
      std::vector<uint16_t>& img = s->phys_img(R.pt[size_t(p / s->T())]);
      for (int64_t h = 0; h < Hkv; ++h)
        for (int64_t e = 0; e < d; ++e) {
          uint16_t kb = k_new[(row * Hkv + h) * d + e];
          uint16_t vb = v_new[(row * Hkv + h) * d + e];
          R.kv[size_t(s->contig_off(p, layer, 0, h) + e)] = kb;
          R.kv[size_t(s->contig_off(p, layer, 1, h) + e)] = vb;
          img[size_t(s->chunk_off(layer, 0, h, p % s->T()) + e)] = kb;
          img[size_t(s->chunk_off(layer, 1, h, p % s->T()) + e)] = vb;
        }
      R.written[size_t(p * s->c.n_layers + layer)] = 1;
    }
  }
  return EO_OK;
}

// Textbook softmax attention, fp64: s_j = scale * q.k_j ; o = sum softmax(s)_j v_j.
int eo_attention_contig(int32_t Hq, int32_t Hkv, int32_t d, int32_t len, const uint16_t* q,
                        const uint16_t* k, const uint16_t* v, double scale, double* out) {
  if (Hq <= 0 || Hkv <= 0 || d <= 0 || len <= 0 || Hq % Hkv != 0) return EO_ERR_INVALID_ARG;
  const int32_t group = Hq / Hkv;
#pragma omp parallel for schedule(static)
  for (int32_t h = 0; h < Hq; ++h) {
    const int32_t g = h / group;  // GQA: contiguous q-head groups share one kv-head (DESIGN R6)
    std::vector<double> sc(static_cast<size_t>(len));
    double m = -std::numeric_limits<double>::infinity();
    for (int32_t j = 0; j < len; ++j) {
      double acc = 0.0;
      for (int32_t e = 0; e < d; ++e)
        acc += bf16_to_double(q[int64_t(h) * d + e]) *
               bf16_to_double(k[(int64_t(j) * Hkv + g) * d + e]);
      sc[size_t(j)] = scale * acc;
      m = std::max(m, sc[size_t(j)]);
    }
    double denom = 0.0;
    for (int32_t j = 0; j < len; ++j) {
      sc[size_t(j)] = std::exp(sc[size_t(j)] - m);
      denom += sc[size_t(j)];
    }
    std::vector<double> acc(static_cast<size_t>(d), 0.0);
    for (int32_t j = 0; j < len; ++j)
      for (int32_t e = 0; e < d; ++e)
        acc[size_t(e)] += sc[size_t(j)] * bf16_to_double(v[(int64_t(j) * Hkv + g) * d + e]);
    for (int32_t e = 0; e < d; ++e) out[int64_t(h) * d + e] = acc[size_t(e)] / denom;
  }
  return EO_OK;
}

// O4 — attention over the accumulated KV of each listed request at one layer. With
// through_table=1 K/V are read through the page table from the physical chunk images;
// with 0 from the contiguous logical copy. Both must agree exactly (translation check).
int eo_attention(eo_state* s, int32_t layer, int32_t n, const int32_t* reqs, const uint16_t* q,
                 double scale, double* out, int32_t through_table) {
  if (layer < 0 || layer >= s->c.n_layers) return EO_ERR_OUT_OF_RANGE;
  if (n < 0) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (reqs[i] < 0 || reqs[i] >= s->c.max_requests) return EO_ERR_OUT_OF_RANGE;
  for (int32_t i = 0; i < n; ++i)
    if (s->req[size_t(reqs[i])].len == 0) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i) {
    const Request& R = s->req[size_t(reqs[i])];
    for (int64_t ci = 0; ci < s->nchunks_of(R.len); ++ci)
      if (!is_dev(R.pt[size_t(ci)])) return EO_ERR_NOT_RESIDENT;
  }
  const int64_t Hq = s->c.n_heads_q, Hkv = s->c.n_heads_kv, d = s->c.head_dim;
  for (int32_t i = 0; i < n; ++i) {
    Request& R = s->req[size_t(reqs[i])];
    std::vector<uint16_t> k(size_t(R.len * Hkv * d)), v(size_t(R.len * Hkv * d));
    for (int64_t p = 0; p < R.len; ++p)
      for (int64_t h = 0; h < Hkv; ++h)
        for (int64_t e = 0; e < d; ++e) {
          size_t o = size_t((p * Hkv + h) * d + e);
          if (through_table) {
            const std::vector<uint16_t>& img = s->phys_img(R.pt[size_t(p / s->T())]);
            k[o] = img[size_t(s->chunk_off(layer, 0, h, p % s->T()) + e)];
            v[o] = img[size_t(s->chunk_off(layer, 1, h, p % s->T()) + e)];
          } else {
            k[o] = R.kv[size_t(s->contig_off(p, layer, 0, h) + e)];
            v[o] = R.kv[size_t(s->contig_off(p, layer, 1, h) + e)];
          }
        }
    eo_attention_contig(int32_t(Hq), int32_t(Hkv), int32_t(d), int32_t(R.len), q + i * Hq * d,
                        k.data(), v.data(), scale, out + i * Hq * d);
  }
  return EO_OK;
}

// O12 (P:871 chunked prefill over the KV cache) — causal attention of the
// last n_q[i] positions of each listed request: query k (q row cum + k) sits at position
// P = len - n_q + k and attends keys 0..P (each token attends to the tokens before
// it and itself). Written as that definition: the decode routine applied to the first P+1
// keys, read through the page table (or from the contiguous copy with through_table = 0).
int eo_prefill_attention(eo_state* s, int32_t layer, int32_t n, const int32_t* reqs,
                         const int32_t* n_q, const uint16_t* q, double scale, double* out,
                         int32_t through_table) {
  if (layer < 0 || layer >= s->c.n_layers) return EO_ERR_OUT_OF_RANGE;
  if (n < 0) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (reqs[i] < 0 || reqs[i] >= s->c.max_requests) return EO_ERR_OUT_OF_RANGE;
  for (int32_t i = 0; i < n; ++i) {
    const int64_t len = s->req[size_t(reqs[i])].len;
    if (len == 0 || n_q[i] < 1 || n_q[i] > len) return EO_ERR_INVALID_ARG;
  }
  for (int32_t i = 0; i < n; ++i) {
    const Request& R = s->req[size_t(reqs[i])];
    for (int64_t ci = 0; ci < s->nchunks_of(R.len); ++ci)
      if (!is_dev(R.pt[size_t(ci)])) return EO_ERR_NOT_RESIDENT;
  }
  const int64_t Hq = s->c.n_heads_q, Hkv = s->c.n_heads_kv, d = s->c.head_dim;
  int64_t row = 0;
  for (int32_t i = 0; i < n; ++i) {
    Request& R = s->req[size_t(reqs[i])];
    std::vector<uint16_t> k(size_t(R.len * Hkv * d)), v(size_t(R.len * Hkv * d));
    for (int64_t p = 0; p < R.len; ++p)
      for (int64_t h = 0; h < Hkv; ++h)
        for (int64_t e = 0; e < d; ++e) {
          size_t o = size_t((p * Hkv + h) * d + e);
          if (through_table) {
            const std::vector<uint16_t>& img = s->phys_img(R.pt[size_t(p / s->T())]);
            k[o] = img[size_t(s->chunk_off(layer, 0, h, p % s->T()) + e)];
            v[o] = img[size_t(s->chunk_off(layer, 1, h, p % s->T()) + e)];
          } else {
            k[o] = R.kv[size_t(s->contig_off(p, layer, 0, h) + e)];
            v[o] = R.kv[size_t(s->contig_off(p, layer, 1, h) + e)];
          }
        }
    for (int64_t kq = 0; kq < n_q[i]; ++kq, ++row) {
      const int64_t P = R.len - n_q[i] + kq;  // keys 0..P (K/V are token-major: a prefix)
      eo_attention_contig(int32_t(Hq), int32_t(Hkv), int32_t(d), int32_t(P + 1), q + row * Hq * d,
                          k.data(), v.data(), scale, out + row * Hq * d);
    }
  }
  return EO_OK;
}

// O5 — offload KV chunks to CPU DRAM; deflation is the reverse of
// inflation. Lowest free host slot first, in list order (DESIGN R7).
int eo_deflate(eo_state* s, int32_t n, const int32_t* ids, int32_t* slots_out) {
  if (n < 0) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= s->c.max_chunks) return EO_ERR_OUT_OF_RANGE;
  if (has_dup(n, ids)) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (s->owner[size_t(ids[i])] != KV || !s->used[size_t(ids[i])]) return EO_ERR_NOT_MAPPED;
  int64_t free_h = 0;
  for (uint8_t u : s->hused) free_h += !u;
  if (n > free_h) return EO_ERR_HOST_FULL;
  for (int32_t i = 0; i < n; ++i) {
    int64_t c = ids[i];
    int64_t h = s->lowest_free_host();
    s->host_img(h) = s->phys_img(c);
    auto where = s->find_entry(int32_t(c));
    s->req[size_t(where.first)].pt[size_t(where.second)] = enc_host(int32_t(h));
    s->hused[size_t(h)] = 1;
    s->used[size_t(c)] = 0;
    slots_out[i] = int32_t(h);
  }
  return EO_OK;
}

// O6 — fetch when the request's decoding is scheduled; the chunk is
// remapped into the KV space. Lowest free KV chunk first, in list order.
int eo_inflate(eo_state* s, int32_t n, const int32_t* slots, int32_t* ids_out) {
  if (n < 0) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (slots[i] < 0 || slots[i] >= s->c.host_slots) return EO_ERR_OUT_OF_RANGE;
  if (has_dup(n, slots)) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (!s->hused[size_t(slots[i])]) return EO_ERR_NOT_MAPPED;
  if (n > s->count_free_kv()) return EO_ERR_NO_CHUNKS;
  for (int32_t i = 0; i < n; ++i) {
    int64_t h = slots[i];
    int64_t c = s->lowest_free_kv();
    s->phys_img(c) = s->host_img(h);
    auto where = s->find_entry(enc_host(int32_t(h)));
    s->req[size_t(where.first)].pt[size_t(where.second)] = int32_t(c);
    s->used[size_t(c)] = 1;
    s->hused[size_t(h)] = 0;
    ids_out[i] = int32_t(c);
  }
  return EO_OK;
}

// O7 — device-to-device chunk migration (BASELINE.json north_star; the paper's own
// migration is ownership-only). phys[dst] = phys[src]; table repointed; src FREE.
int eo_migrate(eo_state* s, int32_t n, const int32_t* src, const int32_t* dst) {
  if (n < 0) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (src[i] < 0 || src[i] >= s->c.max_chunks) return EO_ERR_OUT_OF_RANGE;
  for (int32_t i = 0; i < n; ++i)
    if (dst[i] < 0 || dst[i] >= s->c.max_chunks) return EO_ERR_OUT_OF_RANGE;
  std::vector<int32_t> all(src, src + n);
  all.insert(all.end(), dst, dst + n);
  if (has_dup(int32_t(all.size()), all.data())) return EO_ERR_INVALID_ARG;
  for (int32_t i = 0; i < n; ++i)
    if (s->owner[size_t(src[i])] != KV || !s->used[size_t(src[i])]) return EO_ERR_NOT_MAPPED;
  for (int32_t i = 0; i < n; ++i) {
    if (s->owner[size_t(dst[i])] != KV) return EO_ERR_NOT_MAPPED;
    if (s->used[size_t(dst[i])]) return EO_ERR_ALREADY_MAPPED;
  }
  for (int32_t i = 0; i < n; ++i) {
    s->phys_img(dst[i]) = s->phys_img(src[i]);
    auto where = s->find_entry(src[i]);
    s->req[size_t(where.first)].pt[size_t(where.second)] = dst[i];
    s->used[size_t(dst[i])] = 1;
    s->used[size_t(src[i])] = 0;
  }
  return EO_OK;
}

// O8 — released slots return to the pool.
int eo_release(eo_state* s, int32_t r) {
  if (r < 0 || r >= s->c.max_requests) return EO_ERR_OUT_OF_RANGE;
  Request& R = s->req[size_t(r)];
  for (auto& e : R.pt) {
    if (is_dev(e)) s->used[size_t(e)] = 0;
    if (is_host(e)) s->hused[size_t(host_of(e))] = 0;
    e = UNMAPPED;
  }
  R.len = 0;
  R.pending = 0;
  R.kv.clear();
  R.written.clear();
  return EO_OK;
}

// O9 — inflation (1)-(4): ownership transfer ACT -> KV and remap. Only chunks of
// "inactive" activation memory can be reclaimed (step 2): chunks inside a live
// activation slot (O10) are skipped.
int eo_grow(eo_state* s, int64_t n) {
  if (n < 0) return EO_ERR_INVALID_ARG;
  int64_t act = 0;
  for (size_t i = 0; i < s->owner.size(); ++i) act += (s->owner[i] == ACT && !s->in_act[i]);
  if (n > act) return EO_ERR_NO_CHUNKS;
  for (size_t i = 0; i < s->owner.size() && n > 0; ++i)
    if (s->owner[i] == ACT && !s->in_act[i]) {
      s->owner[i] = KV;
      s->used[i] = 0;
      --n;
    }
  return EO_OK;
}

// O9 — deflation, "the reverse process": the n highest-id FREE KV chunks -> ACT.
int eo_shrink(eo_state* s, int64_t n) {
  if (n < 0) return EO_ERR_INVALID_ARG;
  if (n > s->count_free_kv()) return EO_ERR_IN_USE;
  for (int64_t i = int64_t(s->owner.size()) - 1; i >= 0 && n > 0; --i)
    if (s->owner[size_t(i)] == KV && !s->used[size_t(i)]) {
      s->owner[size_t(i)] = ACT;
      s->phys.erase(i);  // physical memory given back: contents undefined (read as 0)
      --n;
    }
  return EO_OK;
}

// O10 — activation eTensor allocation (f3; activation tensor slots are
// non-uniformly sized VA segments aligned to the chunk granularity, backed by ACT-owned chunks
// of the unified pool). A slot of n chunks is the run of n consecutive ACT chunks
// not already in a slot whose LAST chunk has the highest id (activations fill the pool from the
// top, KV inflation takes the lowest ACT ids). NO_CHUNKS if no such run exists.
int eo_act_alloc(eo_state* s, int64_t n, int64_t* first_out) {
  if (n <= 0) return EO_ERR_INVALID_ARG;
  const int64_t C = s->c.max_chunks;
  for (int64_t last = C - 1; last - n + 1 >= 0; --last) {
    bool ok = true;
    for (int64_t c = last - n + 1; c <= last && ok; ++c)
      ok = s->owner[size_t(c)] == ACT && !s->in_act[size_t(c)];
    if (!ok) continue;
    const int64_t first = last - n + 1;
    for (int64_t c = first; c <= last; ++c) s->in_act[size_t(c)] = 1;
    s->act_len[size_t(first)] = n;
    *first_out = first;
    return EO_OK;
  }
  return EO_ERR_NO_CHUNKS;
}

// O11 — activation eTensor release: the slot starting at `first` ends; its chunks stay ACT,
// now inactive (reclaimable by O9). Not a slot start -> NOT_MAPPED; id range -> OUT_OF_RANGE.
int eo_act_free(eo_state* s, int64_t first) {
  if (first < 0 || first >= s->c.max_chunks) return EO_ERR_OUT_OF_RANGE;
  const int64_t n = s->act_len[size_t(first)];
  if (n == 0) return EO_ERR_NOT_MAPPED;
  for (int64_t c = first; c < first + n; ++c) s->in_act[size_t(c)] = 0;
  s->act_len[size_t(first)] = 0;
  return EO_OK;
}

int64_t eo_act_used(const eo_state* s) {
  int64_t n = 0;
  for (uint8_t a : s->in_act) n += a;
  return n;
}

int eo_stats(const eo_state* s, int64_t* out) {
  int64_t kv_free = 0, kv_used = 0, act = 0, hf = 0, hu = 0;
  for (size_t i = 0; i < s->owner.size(); ++i) {
    if (s->owner[i] == ACT) ++act;
    else if (s->used[i]) ++kv_used;
    else ++kv_free;
  }
  for (uint8_t u : s->hused) (u ? hu : hf)++;
  out[0] = kv_free; out[1] = kv_used; out[2] = act; out[3] = hf; out[4] = hu;
  return EO_OK;
}

int eo_get_table(const eo_state* s, int32_t r, int32_t* entries, int32_t cap, int32_t* n_out,
                 int32_t* len_out) {
  if (r < 0 || r >= s->c.max_requests) return EO_ERR_OUT_OF_RANGE;
  const Request& R = s->req[size_t(r)];
  int64_t nc = s->nchunks_of(R.len);
  if (n_out) *n_out = int32_t(nc);
  if (len_out) *len_out = int32_t(R.len);
  for (int64_t i = 0; i < nc && i < cap; ++i) entries[i] = R.pt[size_t(i)];
  return EO_OK;
}

int eo_read_chunk(const eo_state* s, int64_t c, uint8_t* dst) {
  if (c < 0 || c >= s->c.max_chunks) return EO_ERR_OUT_OF_RANGE;
  auto it = s->phys.find(c);
  if (it == s->phys.end()) std::memset(dst, 0, size_t(s->chunk_elems * 2));
  else std::memcpy(dst, it->second.data(), size_t(s->chunk_elems * 2));
  return EO_OK;
}

int eo_read_host_slot(const eo_state* s, int64_t h, uint8_t* dst) {
  if (h < 0 || h >= s->c.host_slots) return EO_ERR_OUT_OF_RANGE;
  auto it = s->host.find(h);
  if (it == s->host.end()) std::memset(dst, 0, size_t(s->chunk_elems * 2));
  else std::memcpy(dst, it->second.data(), size_t(s->chunk_elems * 2));
  return EO_OK;
}

// Invariants I1-I6 and I7 (activation slots, f3).
int eo_check_invariants(const eo_state* s) {
  const int64_t C = s->c.max_chunks, H = s->c.host_slots;
  std::vector<int> dev_refs(size_t(C), 0), host_refs(size_t(H), 0);
  for (const Request& R : s->req) {
    int64_t nc = s->nchunks_of(R.len);
    for (int64_t i = 0; i < int64_t(R.pt.size()); ++i) {
      int32_t e = R.pt[size_t(i)];
      if (i < nc && e == UNMAPPED) return 1;   // I1: every live token maps somewhere
      if (i >= nc && e != UNMAPPED) return 1;  // I1: prefix-contiguous
      if (is_dev(e)) {
        if (e >= C || s->owner[size_t(e)] != KV) return 2;
        if (++dev_refs[size_t(e)] > 1) return 2;  // I2: no double mapping
      }
      if (is_host(e)) {
        if (host_of(e) >= H) return 2;
        if (++host_refs[size_t(host_of(e))] > 1) return 2;
      }
    }
  }
  int64_t st[5];
  eo_stats(s, st);
  if (st[0] + st[1] + st[2] != C || st[3] + st[4] != H) return 3;  // I3: conservation
  for (size_t r = 0; r < s->req.size(); ++r) {  // I4: bytes through pt == logical KV
    const Request& R = s->req[r];
    for (int64_t p = 0; p < R.len; ++p) {
      int32_t e = R.pt[size_t(p / s->T())];
      const std::map<int64_t, std::vector<uint16_t>>& imgs = is_dev(e) ? s->phys : s->host;
      int64_t key = is_dev(e) ? e : host_of(e);
      auto it = imgs.find(key);
      for (int64_t l = 0; l < s->c.n_layers; ++l) {
        if (!R.written[size_t(p * s->c.n_layers + l)]) continue;
        if (it == imgs.end()) return 4;
        for (int64_t kv = 0; kv < 2; ++kv)
          for (int64_t h = 0; h < s->c.n_heads_kv; ++h)
            for (int64_t e2 = 0; e2 < s->c.head_dim; ++e2)
              if (it->second[size_t(s->chunk_off(l, kv, h, p % s->T()) + e2)] !=
                  R.kv[size_t(s->contig_off(p, l, kv, h) + e2)])
                return 4;
      }
    }
  }
  for (int64_t c = 0; c < C; ++c)  // I6: USED <=> referenced exactly once
    if (bool(s->used[size_t(c)]) != (dev_refs[size_t(c)] == 1)) return 6;
  for (int64_t h = 0; h < H; ++h)
    if (bool(s->hused[size_t(h)]) != (host_refs[size_t(h)] == 1)) return 6;
  // I7 (f3): activation slots are disjoint runs of ACT chunks that exactly cover in_act
  std::vector<uint8_t> cover(size_t(C), 0);
  for (int64_t c = 0; c < C; ++c)
    for (int64_t k = 0; k < s->act_len[size_t(c)]; ++k) {
      if (c + k >= C || s->owner[size_t(c + k)] != ACT || cover[size_t(c + k)]) return 7;
      cover[size_t(c + k)] = 1;
    }
  for (int64_t c = 0; c < C; ++c)
    if (cover[size_t(c)] != s->in_act[size_t(c)]) return 7;
  return 0;
}

}  // extern "C"
