// internal.h — private declarations of libellm.so (not part of the ABI; see include/ellm.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/ellm.h"

struct ellm_vtensor;

namespace ellm {

// ---- driver API through the runtime's entry-point table (no -lcuda link dependency) ----
struct Driver {
  bool ok = false;
  CUresult (*memAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*memAddressFree)(CUdeviceptr, size_t);
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                        unsigned long long);
  CUresult (*memRelease)(CUmemGenericAllocationHandle);
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*memUnmap)(CUdeviceptr, size_t);
  CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*memGetAllocationGranularity)(size_t*, const CUmemAllocationProp*,
                                          CUmemAllocationGranularity_flags);
  CUresult (*tensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
};
const Driver& driver();  // loads once; .ok false if unavailable
// Context entry points for the swap engine's side context (swap mode 3): cuCtxCreate_v2 etc.
struct CtxDriver {
  bool ok = false;
  CUresult (*deviceGet)(CUdevice*, int);
  CUresult (*ctxCreate)(CUcontext*, unsigned int, CUdevice);
  CUresult (*ctxDestroy)(CUcontext);
  CUresult (*ctxPushCurrent)(CUcontext);
  CUresult (*ctxPopCurrent)(CUcontext*);
};
const CtxDriver& ctx_driver();

int64_t now_ns();
int vt_unmap_slot_nosync(ellm_vtensor* vt, int64_t slot);
int vt_map_from(ellm_vtensor* vt, int64_t dst, int64_t src);

// ---- staging ring: host-snapshot -> device small-array uploads, stream-ordered ----------
// Pinned host + device buffers split into segments; a segment is reused only after the
// events recorded for work that consumed it have completed.
class StagingRing {
 public:
  int init(size_t seg_bytes, int n_segs);
  void destroy();
  // Reserve `bytes` (<= seg_bytes) and return host / device views of it.
  int alloc(size_t bytes, void** host, void** dev, uint64_t* generation);
  // Copy the host view of [dev, dev+bytes) to the device on `stream` (async).
  int upload(void* dev, size_t bytes, cudaStream_t stream);
  // Mark the segment holding `dev` as used by the work about to be enqueued.
  void touch(const void* dev);
  // Record that work enqueued on `stream` so far consumes every touched segment.
  int commit(cudaStream_t stream);
  // Same, but the event is recorded later on `stream` (next commit, or before reuse).
  int commit_lazy(cudaStream_t stream);
  bool still_valid(const void* dev, uint64_t generation) const;
  size_t seg_bytes() const { return seg_bytes_; }

 private:
  struct Seg {
    uint64_t generation = 0;
    std::vector<cudaEvent_t> events;
    std::vector<cudaStream_t> streams;
  };
  int retire_and_advance();
  int commit_seg(int seg, cudaStream_t stream);
  int flush_pending(int only_seg);  // -1: all
  std::vector<std::pair<int, cudaStream_t>> pending_;
  std::vector<int> touched_;
  uint8_t* h_ = nullptr;
  uint8_t* d_ = nullptr;
  size_t seg_bytes_ = 0;
  int n_segs_ = 0;
  int cur_ = 0;
  size_t off_ = 0;
  std::vector<Seg> segs_;
  std::vector<cudaEvent_t> free_events_;
};

// ---- kernel launchers (kernels.cu / attention.cu) ---------------------------------------
struct TableUpdate {
  int32_t index;
  int32_t value;
};
cudaError_t launch_table_scatter(int32_t* d_table, const TableUpdate* d_updates, int32_t n,
                                 cudaStream_t s);

// a10: wait on `s` until *flag (this rank's gather flag word) >= target (wrapping compare).
cudaError_t launch_gather_wait(const uint32_t* flag, uint32_t target, uint64_t timeout_ns, cudaStream_t s);

// Rotated slabs: on the device, layer l's [2][Hkv][T][d] slab of chunk c sits in
// slab slot (l + c / kRotGroup) mod L of the chunk (rot = L), so one layer's slabs of
// consecutive chunk groups are not all at the same offset a chunk stride apart — with chunk
// strides of 5 / 10 MiB (70B shape) that pattern loses ~20% of HBM read bandwidth
// (tools/slab_read.cu). Within an aligned group of kRotGroup chunks the slot is constant, so
// the prefill kernel's multi-chunk TMA boxes (<= 8 chunks) keep a plain chunk stride and
// split only at group boundaries (1 tile in 4 at T = 16; 8-chunk groups cost prefill 8%).
// rot = 0: slot l. Host slots, read_chunk and the oracle keep the canonical image.
constexpr int32_t kRotGroup = 32;
__host__ __device__ inline int32_t slab_slot(int64_t c, int32_t l, int32_t rot) {
  return rot ? int32_t((uint32_t(l) + uint32_t(c) / kRotGroup) % uint32_t(rot)) : l;  // c < 2^31
}
__host__ __device__ inline int32_t slab_shift(int64_t c, int32_t rot) {  // slot of layer 0
  return rot ? int32_t((uint32_t(c) / kRotGroup) % uint32_t(rot)) : 0;
}

struct AppendDesc {  // device-resident arrays, n entries (+1 for cum)
  const int32_t* req;
  const int32_t* pos0;
  const int32_t* cum_rows;
};
cudaError_t launch_kv_append(const AppendDesc& d, int32_t n, int64_t total_rows, const int32_t* table,
                             int32_t table_stride, uint8_t* pool, int64_t chunk_bytes, int32_t T,
                             int32_t layer, int32_t Hkv, int32_t D, const void* k_new,
                             const void* v_new, int num_sms, cudaStream_t s, int32_t rot);

// Chunk copy: dst_base + dst_idx[i]*bytes <- src_base + src_idx[i]*bytes, i < n.
// (seg_off, seg_bytes): copy only that byte range of each chunk (seg_bytes < 0: whole chunk).
// `work`: a device word that is 0 when the kernel starts, the work-claim counter (callers upload
// it with the index lists, so every call has its own).
cudaError_t launch_chunk_copy(uint8_t* dst_base, const int32_t* dst_idx, const uint8_t* src_base,
                              const int32_t* src_idx, int32_t n, int64_t chunk_bytes, int grid,
                              uint32_t* work, cudaStream_t s, int64_t seg_off = 0, int64_t seg_bytes = -1,
                              int32_t rot = 0, int64_t slab = 0, bool src_dev = false, bool dst_dev = false);
// (rot, slab, src_dev, dst_dev): offsets are canonical; a side marked _dev is a pool chunk whose
// slabs are rotated (slab_slot), the other side (host slot) is canonical.
inline uint32_t* work_word(const int32_t* uploaded, int64_t index) {
  return reinterpret_cast<uint32_t*>(const_cast<int32_t*>(uploaded + index));
}

constexpr int kMaxPeers = 8;            // ranks of a fused head gather (one 8-GPU box)

struct AttnDesc {  // device-resident
  const int32_t* req;      // [n]
  const int32_t* len;      // [n]
  const int32_t* cum_s;    // [n_vr + 1] prefix of static tiles (first stat(vr) tiles of vr)
  const int32_t* cum_d;    // [n_vr + 1] prefix of dynamic tiles (last dyn(vr) tiles of vr)
  const int32_t* b_first;  // [n_vr] static owner CTAs of vr (empty if last < first)
  const int32_t* b_last;   // [n_vr]
  const int32_t* u_first;  // [n_vr] dynamic owner units of vr (empty if last < first)
  const int32_t* u_last;   // [n_vr]
};
// Schedule of one attention launch: the W_s static tiles (the first stat(vr) tiles of every
// request) are split evenly over G CTAs; the W_d dynamic tiles (the last dyn(vr) = tiles(vr) /
// dyn_div of every request) go in n_dyn units of U tiles claimed with a ticket counter.
struct AttnPlan {
  int64_t W_s = 0, W_d = 0, U = 1, n_dyn = 0;
  int32_t G = 0;
  unsigned long long* ticket = nullptr;
  unsigned long long ticket_base = 0;
  const int32_t* dyn_info = nullptr;  // device: [n_dyn][8] (int4 pairs, see attention.cu Params)
  const int32_t* dyn_ent = nullptr;   // device: [n_dyn][U * npieces]
  const int32_t* cta_first = nullptr; // device: [G][8] first static segment of each CTA
  // fused decode append (ellm_decode_append_attention): one new token per request, or nullptr
  const void* k_new = nullptr;
  const void* v_new = nullptr;
  uint8_t* pool = nullptr;
  int64_t chunk_bytes = 0;
  // a10 fused head gather (ellm_attention_gather): per rank, where this call's rows and its
  // merged-request count go; n_peer = 0 writes `out` as a local [n, Hq, D] tensor instead.
  void* gout[kMaxPeers] = {};
  uint32_t* gflag[kMaxPeers] = {};
  int32_t n_peer = 0, Hq_out = 0, q_off = 0;
  uint32_t* gdone = nullptr;   // CTAs of gather launches that finished (device counter)
  unsigned long long* trace = nullptr;  // ellm_set_attn_trace slot of this launch
  uint32_t range_shift = 0;    // ELLM_ATTN_RANGE_ROT=1: rotate static ranges over CTAs per launch
  uint32_t gdone_target = 0;   // value the counter reaches when this launch's last CTA arrives
  // a10 folded gather wait (ellm_gather_wait_next): before staging Q or writing anything, the
  // producer spins (acquire, system scope) until *wait_flag reaches wait_target; nullptr = none
  const uint32_t* wait_flag = nullptr;
  uint32_t wait_target = 0;
  uint64_t wait_timeout_ns = 0;
  // programmatic dependent launch: this launch may start while the previous kernel on the
  // stream finishes (attention.cu: K/V streamed before griddepcontrol.wait, all else after)
  bool pdl = false;
};
struct AttnShape {
  int32_t D, HB, HG, Hkv, Hq, group, T, L, TT, nsub;
  int32_t rot;      // slab rotation (slab_slot): L, or 0 for the canonical layout
  int64_t slab;     // bytes of one layer's [2][Hkv][T][d] slab
};
constexpr int64_t kMaxDynUnits = 4096;   // cap on dynamic units per attention launch
int attn_heads_per_block(int32_t Hkv);  // HB
int attn_stage_tokens(int32_t HB);      // TT
cudaError_t attn_configure(int32_t D, int32_t HB);   // smem attributes, once
cudaError_t encode_kv_tensor_map(CUtensorMap* map, void* pool_base, int64_t max_chunks,
                                 const AttnShape& sh);
cudaError_t launch_paged_attention(const CUtensorMap& tmap, const AttnShape& sh, const AttnDesc& d,
                                   int32_t n, int32_t n_vr, const AttnPlan& plan,
                                   const int32_t* table, int32_t table_stride, int32_t layer,
                                   const void* q, void* out, float* part, float* part_ml,
                                   int32_t* arrivals, float scale, cudaStream_t s, int* launches);

// chunked-prefill attention (prefill.cu). work: [n_work][8] int32 items
// {req, len, q_row0, p0, n_valid, kvh, n_tiles, 0}. kv / run[] depend only on the pool (cached);
// q is encoded per call.
struct alignas(64) PrefillMaps {
  CUtensorMap kv;       // 128-token boxes inside one chunk (T >= 128)
  CUtensorMap run[4];   // boxes of 1/2/4/8 consecutive whole chunks (T < 128)
  CUtensorMap q;
  int32_t runs;         // 1: run maps usable, 0: none (one box per chunk)
};
cudaError_t encode_prefill_kv_maps(PrefillMaps* m, void* pool_base, int64_t max_chunks, const AttnShape& sh,
                                   int64_t chunk_bytes);
cudaError_t encode_prefill_q_map(PrefillMaps* m, const AttnShape& sh, const void* q, int64_t q_rows);
cudaError_t launch_prefill_attention(const PrefillMaps& maps, const AttnShape& sh, const int32_t* work,
                                     int32_t n_work, const int32_t* table, int32_t table_stride, int32_t layer,
                                     void* out, float scale, cudaStream_t s, void* trace = nullptr);

}  // namespace ellm

// ---- the pool ---------------------------------------------------------------------------
struct ellm_vtensor {
  int32_t device = -1;
  size_t slot_bytes = 0;
  int64_t n_slots = 0;
  CUdeviceptr base = 0;
  std::vector<CUmemGenericAllocationHandle> handles;
  std::vector<uint8_t> mapped;
  std::vector<uint8_t> owned;  // slot owns (releases) its handle; 0 after vt_map_from moved it
  int64_t n_map = 0, n_unmap = 0, map_ns = 0, unmap_ns = 0;
};

struct ellm_pool {
  ellm_pool_config cfg{};
  bool has_dev = false;
  int64_t chunk_bytes = 0;
  int32_t T = 0, group = 0;

  // ownership / state: owner 0 = KV, 1 = ACT
  std::vector<uint8_t> owner, used;
  int64_t n_free_kv = 0, n_used_kv = 0, n_act = 0;
  int64_t free_hint = 0;  // no FREE KV chunk below this id
  std::vector<int32_t> chunk_req, chunk_idx;  // back-pointers of USED chunks
  std::vector<uint8_t> hused;
  int64_t n_host_used = 0, host_hint = 0;
  std::vector<int32_t> slot_req, slot_idx;

  // per request
  std::vector<int32_t> table;  // [max_requests][max_chunks_per_request] host authoritative
  std::vector<int64_t> len;
  std::vector<int32_t> pending, nonres;

  // device side
  ellm_vtensor* vt = nullptr;        // one slot per map unit
  int64_t unit_bytes = 0;            // bytes per physical map unit
  int64_t chunks_per_unit = 1;       // >1 when chunk_bytes < granularity
  std::vector<int32_t> unit_kv;      // KV-owned chunks in each unit
  int32_t* d_table = nullptr;
  uint8_t* host_slots = nullptr;     // pinned, mapped
  float* d_part = nullptr;
  float* d_part_ml = nullptr;
  int32_t* d_arrivals = nullptr;     // per virtual request, for the fused split-K merge
  int64_t part_records = 0;
  int64_t attn_cap = 0;              // list entries the split-K state above is sized for
  CUtensorMap tmap{};
  ellm::AttnShape ash{};
  int num_sms = 0;
  ellm::StagingRing ring;
  int swap_mode = 0;                 // 0 SM copy kernel, 1 copy engines, 2 staged inflate, 3 side-context inflate
  CUcontext side_ctx = nullptr;      // swap mode 3 / ellm_upload: second context on the pool's device
  uint8_t* side_stage = nullptr;       // ... owning this staging buffer (256 MiB)
  int64_t side_stage_bytes = 0;
  cudaEvent_t side_ev = nullptr;       // last use of the staging buffer
  cudaStream_t side_ev_stream = nullptr;  // ... recorded on this stream
  bool side_ev_used = false;
  uint8_t* d_stage = nullptr;        // swap_mode 2: device staging buffer for inflate (256 MiB)
  cudaEvent_t stage_ev = nullptr;    // last use of the staging buffer
  cudaStream_t stage_stream = nullptr;
  std::vector<ellm::TableUpdate> pending_updates;

  // attention descriptor cache
  std::vector<int32_t> cache_key;     // req ids then lens
  uint64_t table_epoch = 0;           // bumped by every table entry change
  int64_t cache_info_off = 0, cache_ent_off = 0;  // dynamic-unit arrays inside the descriptor
  int64_t cache_cta_off = 0;        // per-CTA first-segment info in the cached descriptor
  uint64_t cache_epoch = ~uint64_t(0);
  const int32_t* cache_dev = nullptr;
  uint64_t cache_gen = 0;
  int32_t cache_n_vr = 0;
  ellm::AttnPlan cache_plan;
  unsigned long long* d_ticket = nullptr;  // dynamic-unit ticket counter (device)
  uint64_t ticket_base = 0;                // tickets consumed by earlier launches
  uint32_t gdone_base = 0;                 // gather-launch CTAs counted by earlier launches
  unsigned long long* trace_buf = nullptr; // ellm_set_attn_trace: caller's device buffer
  int32_t trace_slots = 0;
  std::vector<float> dbg_weights;          // ellm_debug_attn_weights: static split weights per CTA
  int64_t trace_launch = 0;
  int64_t dyn_div = 0;                     // dynamic tail = tiles/dyn_div per request (0: static only)
  int64_t dyn_unit = 8;                    // minimum tiles per dynamic unit

  // stream-ordered reuse: a chunk / host slot freed by work on stream S carries the event
  // recorded after that work; a later call on another stream that allocates it first makes
  // its stream wait on the event (allocation order itself stays deterministic).
  struct FreeEvent {
    cudaEvent_t ev = nullptr;
    cudaStream_t stream = nullptr;
    int32_t refs = 0;
  };
  std::vector<FreeEvent> free_events;
  std::vector<int32_t> free_event_pool;          // indices of unreferenced events
  std::vector<int32_t> chunk_ev, slot_ev;        // per chunk / host slot: event index or -1
  // layer-wise offload in progress (ellm_offload_*): reserved slot and layers copied, per chunk
  std::vector<int32_t> off_slot;
  std::vector<uint64_t> off_layers;  // per chunk: bitset of layers copied by offload_layer (off_words words)
  int64_t off_words = 1;

  // f1: VMM work off the caller's critical path. A worker thread keeps
  // the `premap_units` lowest all-ACT units mapped ahead of pool_grow (speculative pre-mapping)
  // and unmaps units pool_shrink left all-ACT (asynchronous unmapping). pool_grow that needs an
  // unmapped unit while another awaits its async unmap takes that unit's physical handle
  // (multi-mapping); the donor's VA stays mapped ("doomed") until the worker unmaps it.
  std::mutex vmm_mu;                 // guards vt, unit_kv, doomed and the fields below
  std::condition_variable vmm_cv;
  std::thread vmm_thread;
  bool vmm_started = false, vmm_stop = false, vmm_dirty = false, vmm_busy = false;
  int64_t premap_units = 0;
  bool async_unmap = false;
  int64_t vmm_delay_us = 0;          // test knob (ELLM_VMM_WORKER_DELAY_US): worker start delay
  std::vector<uint8_t> doomed;       // per unit: handle moved away, VA mapping awaits unmap
  std::vector<uint64_t> unit_gen;    // per unit: bumped when its first chunk becomes KV
  int vmm_error = 0;                 // sticky worker failure, reported by ellm_vmm_sync
  int64_t crit_vmm_ns = 0;           // VMM + device-sync time inside pool_grow / pool_shrink
  int64_t n_steal = 0, premap_hits = 0;

  // f3: activation eTensor slots in the same pool. A slot is a run of
  // consecutive ACT chunks; units holding live slots stay mapped, and a unit activations used
  // stays mapped after they end ("mapped, available" pooling) until pool_grow takes
  // its chunks (ownership transfer with no driver call) or ellm_act_trim releases it.
  std::vector<int64_t> act_len;      // per chunk: slot length if a slot starts here, else 0
  std::vector<uint8_t> in_act;       // per chunk: inside a live slot
  int64_t n_act_used = 0;
  std::vector<int32_t> unit_act;     // per unit: chunks inside live slots (under vmm_mu)
  std::vector<uint8_t> act_cached;   // per unit: kept mapped for activations (under vmm_mu)

  ellm::PrefillMaps pf_maps{};       // f4 tensor maps over the pool (encoded on first use)
  bool pf_ready = false;

  // a10 fused head gather (ellm_gather_attach): every rank's gather window (flag words at +0,
  // rows at +ELLM_GATHER_DATA_OFFSET), and per flag word the value this rank's own flag reaches
  // once every rank has finished the calls issued so far
  int32_t g_world = 0, g_rank = 0, g_hq_out = 0;
  std::vector<uint8_t*> g_win;
  int64_t g_win_bytes = 0;
  std::vector<uint32_t> g_expect;
  uint64_t g_timeout_ns = 20000000000ull;
  const uint32_t* g_wait_flag = nullptr;  // folded wait (ellm_gather_wait_next) for the next launch
  uint32_t g_wait_target = 0;

  // programmatic dependent launch of attention (attention.cu; ellm_set_launch_overlap, ELLM_PDL)
  bool pdl = false;
  bool pdl_env = false;              // ELLM_PDL set: the environment wins over the setter
  int32_t last_fused_layer = -1;     // layer the previous attention launch appended into, or -1
  int32_t prev_fused_layer = -1;     // the same for the launch before it

  std::map<int32_t, std::pair<CUdeviceptr, size_t>> alias;
  int last_cuda_error = 0;
  int64_t launches = 0;
};
