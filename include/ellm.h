/* ellm.h — C ABI of libellm.so: the B200-native KV-traffic hot path of eLLM
 * (arXiv 2506.15155, "eLLM: Elastic Memory Management Framework for Efficient LLM
 * Serving"; paper text at /root/reference/PAPER.md, cited P:<line>).
 *
 * Layering:
 *   vtensor   — a virtual address range whose chunk-aligned slots are backed on demand by
 *               physical chunks (the paper's eTensor: "an array pointer structure
 *               that references a contiguous segment within the GPU's virtual address
 *               space").
 *   pool      — one vtensor of `max_chunks` KV chunks + per-chunk ownership KV/ACT
 *               + per-request chunk tables + pinned host slots (the CPU elastic buffer,
 *               P:390-399) + the kernels that move KV through them.
 *
 * Conventions for every call
 *   - Return int: ELLM_OK (0) or a negative ELLM_ERR_*. No exception crosses the ABI.
 *   - All-or-nothing: every precondition is validated BEFORE any state changes, so an
 *     error leaves the pool exactly as it was (no hold-and-wait).
 *   - Validation order (R12): argument ranges (OUT_OF_RANGE) -> duplicates /
 *     malformed counts (INVALID_ARG) -> per-request capacity (OUT_OF_RANGE) -> residency
 *     (NOT_RESIDENT) / ownership (NOT_MAPPED, ALREADY_MAPPED) -> pool capacity (NO_CHUNKS,
 *     HOST_FULL, IN_USE). Within a class, list order decides which element reports.
 *   - Host metadata (request ids, counts, chunk / slot lists, outputs such as slot ids) are
 *     HOST pointers, read/written before the call returns. Tensors (q, k_new, v_new, out)
 *     are DEVICE pointers owned by the caller; they must stay valid until the stream
 *     reaches the enqueued work. `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Device work is enqueued on `stream`. Reuse is stream-ordered by the library: a chunk or
 *     host slot freed by work on stream A (deflate, inflate, migrate, release) carries the event
 *     recorded after that work, and a later call on stream B that is handed it makes B wait on
 *     that event first (allocation order itself stays deterministic). Work on the same request
 *     from two streams must still be ordered by the caller. Attention calls on one pool share
 *     its split-K workspace and must be ordered among themselves. Kernel faults surface as
 *     ELLM_ERR_CUDA at a later call (ellm_last_cuda_error gives the cudaError_t).
 *   - One pool per device; calls on one pool are externally serialised.
 *   - Allocation policy (R7): lowest free chunk id / host slot first, requests in
 *     the given order, positions ascending. Tables are therefore deterministic and identical
 *     on every KV-head shard.
 *
 * Chunk geometry (R1): one chunk = T tokens x L layers x {K,V} x Hkv local
 * kv-heads x d, bf16, layout [L][2][Hkv][T][d]; chunk_bytes = 4*T*L*Hkv*d.
 * Chunk c lives at pool_base + c*chunk_bytes. On the device, layer l's [2][Hkv][T][d] slab sits
 * in slab slot (l + floor(c/32)) mod L of the chunk ("rotated slabs": consecutive chunks'
 * slabs of one layer are not at a fixed offset, which costs HBM bandwidth for chunk strides that
 * are not a power of two); it is used when chunk_bytes is not a power of two, and never when a
 * chunk is its own map unit (map_unit_bytes == chunk_bytes, the ellm_alias_request
 * configuration) or for L = 1; ELLM_ROTATE=1 / 0 forces it on / off. Host slots,
 * ellm_read_chunk and ellm_read_host_slot always hold the canonical image above.
 * Table entries: >=0 device chunk id,
 * -1 unmapped, <=-2 host slot h encoded as -(h+2).
 */
#ifndef ELLM_H
#define ELLM_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum {
  ELLM_OK = 0,
  ELLM_ERR_INVALID_ARG = -1,    /* malformed argument, duplicate id, zero-length attention */
  ELLM_ERR_OUT_OF_RANGE = -2,   /* id / layer / capacity out of range */
  ELLM_ERR_NO_CHUNKS = -3,      /* not enough FREE KV chunks (or ACT chunks for grow) */
  ELLM_ERR_HOST_FULL = -4,      /* not enough free host slots */
  ELLM_ERR_NOT_RESIDENT = -5,   /* a needed chunk is in a host slot */
  ELLM_ERR_NOT_MAPPED = -6,     /* chunk FREE/ACT (or host slot free) where USED is required */
  ELLM_ERR_ALREADY_MAPPED = -7, /* destination chunk USED */
  ELLM_ERR_IN_USE = -8,         /* shrink needs more FREE chunks than exist */
  ELLM_ERR_CUDA = -9,           /* CUDA runtime / driver failure */
  ELLM_ERR_PEER = -10,          /* a peer rank's gather window could not be opened (ellm_ipc_open) */
  ELLM_ERR_NO_DEVICE = -11,     /* call needs a device but the pool is host-metadata-only */
  ELLM_ERR_UNSUPPORTED = -12    /* shape outside what the kernels implement (see pool_create) */
};

/* device = ELLM_DEVICE_NONE creates a host-metadata-only pool (tables, ownership, host
 * slot bookkeeping; no VMM, no kernels). Calls that move bytes update metadata only in
 * that mode and the attention / append / read calls return ELLM_ERR_NO_DEVICE. It exists
 * so the allocation logic can be tested on a machine without a GPU. */
#define ELLM_DEVICE_NONE (-1)

typedef struct ellm_pool ellm_pool;
typedef struct ellm_vtensor ellm_vtensor;

typedef struct {
  int32_t device;                  /* CUDA ordinal or ELLM_DEVICE_NONE */
  int32_t n_layers;                /* L */
  int32_t n_heads_q;               /* q-heads on this shard (Hq_local) */
  int32_t n_heads_kv;              /* kv-heads on this shard (Hkv_local); Hq % Hkv == 0 */
  int32_t head_dim;                /* d: 64 or 128 */
  int32_t tokens_per_chunk;        /* T: multiple of 16 */
  int64_t max_chunks;              /* VA capacity in chunks (KV + ACT) */
  int64_t initial_chunks;          /* chunks KV-owned (mapped) at create: ids [0, initial) */
  int32_t max_requests;            /* request ids are [0, max_requests) */
  int32_t max_chunks_per_request;  /* table row length (the KV eTensor span) */
  int64_t host_slots;              /* pinned host slots, chunk_bytes each (CPU buffer P_B) */
  int64_t map_unit_bytes;          /* physical allocation unit backing consecutive chunks: 0 = auto
                                      (>= 64 MiB; VMM cost is per handle), else a multiple of
                                      lcm(chunk_bytes, granularity). ellm_alias_request needs
                                      map_unit_bytes == chunk_bytes. */
} ellm_pool_config;

typedef struct {
  int64_t kv_free, kv_used, act;   /* chunk counts; kv_free + kv_used + act == max_chunks */
  int64_t host_free, host_used;    /* host slot counts */
  int64_t n_map, n_unmap;          /* VMM map / unmap operations so far */
  int64_t map_ns, unmap_ns;        /* host wall time spent in them */
  int64_t chunk_bytes;             /* bytes per chunk */
  int64_t mapped_bytes;            /* physical device bytes currently mapped */
  /* f1 (ellm_set_vmm_overlap) */
  int64_t premapped_bytes;         /* all-ACT units mapped ahead of pool_grow (premap window) */
  int64_t pending_unmap;           /* all-ACT units still mapped, waiting for the async unmap */
  int64_t crit_vmm_ns;             /* VMM + device-sync wall time inside pool_grow / pool_shrink
                                      (the caller's critical path; worker time is excluded) */
  int64_t n_steal;                 /* units pool_grow backed with a pending-unmap unit's handle */
  int64_t premap_hits;             /* units pool_grow found already mapped while all-ACT */
  /* f3 (ellm_act_*) */
  int64_t act_used;                /* ACT chunks inside live activation slots */
  int64_t act_cached_bytes;        /* units kept mapped only for (ended) activation slots */
} ellm_stats;

/* ---- vtensor (VMM) ------------------------------------------------------------------
 * A VA reservation of n_slots * slot_bytes (cuMemAddressReserve), each slot backed on
 * demand by its own physical allocation (cuMemCreate + cuMemMap + cuMemSetAccess RW for
 * `device`). slot_bytes must be a multiple of the allocation granularity
 * (ellm_vmm_granularity), else INVALID_ARG. map of a mapped slot -> ALREADY_MAPPED;
 * unmap of an unmapped slot -> NOT_MAPPED (whole range validated first). unmap is
 * synchronous w.r.t. the device (cuMemUnmap, cuda.h \note_sync): it synchronises the
 * device first. The library owns the reservation and handles; destroy releases both. */
int ellm_vmm_granularity(int32_t device, size_t* out);
int ellm_vtensor_create(int32_t device, size_t slot_bytes, int64_t n_slots, ellm_vtensor** out);
int ellm_vtensor_map(ellm_vtensor* vt, int64_t first_slot, int64_t n);
int ellm_vtensor_unmap(ellm_vtensor* vt, int64_t first_slot, int64_t n);
int ellm_vtensor_is_mapped(const ellm_vtensor* vt, int64_t slot); /* 1 / 0, <0 on error */
void* ellm_vtensor_base(const ellm_vtensor* vt);
int ellm_vtensor_destroy(ellm_vtensor* vt);

/* ---- pool ---------------------------------------------------------------------------
 * create: validates the config (head_dim in {64,128}, T % 16 == 0,
 * group Hq/Hkv in [1,8], chunk_bytes a multiple or a divisor of the granularity, else
 * UNSUPPORTED / INVALID_ARG), reserves VA for max_chunks, maps the initial KV chunks,
 * allocates host_slots pinned+mapped host slots and the device tables / workspaces. */
int ellm_pool_create(const ellm_pool_config* cfg, ellm_pool** out);
int ellm_pool_destroy(ellm_pool* pool);
int ellm_pool_stats(const ellm_pool* pool, ellm_stats* out);
void* ellm_pool_base(const ellm_pool* pool);        /* device VA of chunk 0 (NULL if no device) */
void* ellm_pool_host_base(const ellm_pool* pool);   /* host VA of slot 0 (pinned) */

/* kv_reserve (a2; "Physical chunks are allocated on-demand during actual writes"):
 * for each listed request r (distinct), extend its logical length by n_new[i] >= 0,
 * mapping logical chunks ceil(len/T) .. ceil((len+n_new)/T)-1 to the lowest FREE KV ids
 * (requests in list order, chunks ascending). Records n_new[i] as the positions the next
 * kv_append of r writes. Errors: id range / table capacity -> OUT_OF_RANGE; duplicate or
 * negative -> INVALID_ARG; partially-filled last chunk in a host slot (and n_new>0) ->
 * NOT_RESIDENT; total new chunks > FREE KV -> NO_CHUNKS. Enqueues the device-table update
 * on `stream`. No implicit growth: call ellm_pool_grow first. */
int ellm_kv_reserve(ellm_pool* pool, int32_t n, const int32_t* req_ids, const int32_t* n_new,
                    void* stream);

/* kv_append (a3): write K/V of layer `layer` for positions [len-n_new, len) of each listed
 * request (n_new[i] must equal the latest reservation, else INVALID_ARG; R13).
 * k_new, v_new: device [sum(n_new), Hkv, d] bf16, rows in list order then position order.
 * Every target chunk must be on the device (else NOT_RESIDENT). Bit-exact copy. */
int ellm_kv_append(ellm_pool* pool, int32_t layer, int32_t n, const int32_t* req_ids,
                   const int32_t* n_new, const void* k_new, const void* v_new, void* stream);

/* paged_decode_attention (a4+a5, exact softmax attention over the accumulated
 * KV read through the chunk table): for each listed request i (duplicates allowed) and
 * q-head h, out[i][h] = sum_j softmax_j(scale * q[i][h].k_j) v_j over j < len, with kv-head
 * h / (Hq/Hkv). q: device [n, Hq, d] bf16; out: device [n, Hq, d] bf16 (fp32 accumulate,
 * RNE). A list longer than max_requests (repeated ids) grows the split-K state once, which
 * synchronises the device. len == 0 -> INVALID_ARG; any chunk of the request in a host slot ->
 * NOT_RESIDENT. */
int ellm_paged_decode_attention(ellm_pool* pool, int32_t layer, int32_t n, const int32_t* req_ids,
                                const void* q, void* out, float softmax_scale, void* stream);

/* decode_append_attention (a3 + a4 + a5 fused for decode): exactly kv_append(layer, n, req_ids,
 * n_new = 1 each, k_new, v_new) followed by paged_decode_attention(layer, n, req_ids, q, out,
 * softmax_scale), in one kernel launch: the CTA that streams a request's last tile first writes
 * the new token's K/V rows into the chunk, then reads the tile. Requires distinct requests whose
 * latest reservation is exactly 1 token (else INVALID_ARG); errors as the two calls. */
int ellm_decode_append_attention(ellm_pool* pool, int32_t layer, int32_t n, const int32_t* req_ids,
                                 const void* k_new, const void* v_new, const void* q, void* out,
                                 float softmax_scale, void* stream);

/* prefill_attention (P:871 chunked prefill, P:109-112 causal attention):
 * for each listed request i, the LAST n_q[i] positions (the chunk just reserved and appended)
 * attend causally to the request's KV read through its chunk table: query k of request i sits
 * at position P = len - n_q[i] + k and out row = sum_{j <= P} softmax_j(scale * q.k_j) v_j per
 * q-head (kv-head h / (Hq/Hkv)). q: device [sum n_q, Hq, d] bf16, rows in list order then
 * position order; out: device [sum n_q, Hq, d] bf16 (fp32 accumulate, RNE). Runs on the
 * tcgen05 tensor cores (S and O in tensor memory). Errors: layer / id range -> OUT_OF_RANGE;
 * n_q[i] < 1 or > len -> INVALID_ARG; a chunk in a host slot -> NOT_RESIDENT; Hq/Hkv not
 * dividing 128 or more than 32768 work items (request x kv-head x 128/group positions) ->
 * UNSUPPORTED. */
int ellm_prefill_attention(ellm_pool* pool, int32_t layer, int32_t n, const int32_t* req_ids,
                           const int32_t* n_q, const void* q, void* out, float softmax_scale, void* stream);

/* release: all device chunks and host slots of req become FREE; len = 0. */
int ellm_release(ellm_pool* pool, int32_t req_id, void* stream);

/* deflate = swap-out / offload (a6): copy each listed USED chunk to the lowest
 * free host slot (list order), repoint its table entry to the slot, mark the chunk FREE.
 * host_slots_out[i] receives the slot. Errors: id range -> OUT_OF_RANGE; duplicates ->
 * INVALID_ARG; chunk not USED KV -> NOT_MAPPED; n > free slots -> HOST_FULL. */
int ellm_deflate(ellm_pool* pool, int32_t n, const int32_t* chunk_ids, int32_t* host_slots_out,
                 void* stream);
/* inflate = swap-in / fetch (a7): copy each listed USED host slot into the
 * lowest FREE KV chunk (list order), repoint the table entry, free the slot.
 * chunk_ids_out[i] receives the chunk. Errors: slot range -> OUT_OF_RANGE; duplicates ->
 * INVALID_ARG; slot not used -> NOT_MAPPED; n > FREE KV chunks -> NO_CHUNKS. */
int ellm_inflate(ellm_pool* pool, int32_t n, const int32_t* host_slots, int32_t* chunk_ids_out,
                 void* stream);
/* Layer-wise pipelined offload ("offloading KV cache ... during the
 * prefill stage", "layer-wise pipelining", "O(N) ... overhead can be completely hidden").
 * offload_begin: reserve the lowest free host slots for the listed USED chunks (list order);
 *   no data moves and tables still point at the chunks. Errors as deflate, plus a chunk
 *   already being offloaded -> ALREADY_MAPPED.
 * offload_layer: copy layer `layer`'s K/V slabs (2*Hkv*T*d*2 contiguous bytes per chunk) of the
 *   listed chunks to their reserved slots on `stream` — call it right after that layer's
 *   kv_append so the copy overlaps the following layers. The copy runs on the SM copy kernel,
 *   or on the DMA copy engines when ellm_set_swap_mode(1) (no SMs taken from the compute it
 *   overlaps): one cudaMemcpy2DAsync per run of chunks whose ids and slots are both evenly
 *   spaced, else one cudaMemcpyAsync per slab. Chunk not being offloaded -> NOT_MAPPED. Appends
 *   into an offloading chunk after its layer was copied are not carried. A layer counts as
 *   copied only once its copy was enqueued without error.
 * offload_commit: every layer 0..L-1 of every listed chunk copied (a per-chunk layer bitset;
 *   repeating one layer does not count for another; else INVALID_ARG): repoint the
 *   table entries to the slots and free the chunks — the same end state (tables, slots, bytes)
 *   as ellm_deflate of the same list. */
int ellm_offload_begin(ellm_pool* pool, int32_t n, const int32_t* chunk_ids, int32_t* host_slots_out);
int ellm_offload_layer(ellm_pool* pool, int32_t layer, int32_t n, const int32_t* chunk_ids, void* stream);
int ellm_offload_commit(ellm_pool* pool, int32_t n, const int32_t* chunk_ids, void* stream);

/* migrate (a8; BJ; D2D compaction): copy chunk src[i] -> dst[i], repoint the table entry,
 * src becomes FREE, dst USED. Errors: range -> OUT_OF_RANGE; any repeated id among the 2n
 * -> INVALID_ARG; src not USED KV -> NOT_MAPPED; dst ACT -> NOT_MAPPED; dst USED ->
 * ALREADY_MAPPED. */
int ellm_migrate(ellm_pool* pool, int32_t n, const int32_t* src, const int32_t* dst, void* stream);

/* pool_grow (a9; inflation steps 3-4): the n lowest-id ACT chunks become FREE KV
 * and their physical memory is created and mapped. n > #ACT -> NO_CHUNKS.
 * pool_shrink (a9; deflation): the n highest-id FREE KV chunks become ACT; physical
 * memory whose chunks are all ACT is unmapped and released (device-synchronising).
 * n > #FREE KV -> IN_USE. */
int ellm_pool_grow(ellm_pool* pool, int64_t n);
int ellm_pool_shrink(ellm_pool* pool, int64_t n);

/* VMM-overhead hiding. Off by default; the first call starts one
 * background worker thread per pool. Ownership, tables and every other result are unchanged —
 * only WHEN physical memory is mapped / unmapped moves off the caller's thread.
 *   premap_bytes ("decoding speculative pre-mapping"): keep the lowest all-ACT map
 *     units covering premap_bytes (rounded up to whole units) physically mapped, so pool_grow of
 *     the next ACT ids makes no driver call; the worker refills the window after each grow.
 *     The paper's budget is < 50 MB; a map unit is >= 64 MiB by default (config).
 *   async_unmap = 1 ("asynchronous unmapping"): pool_shrink only changes ownership;
 *     the worker device-synchronises and unmaps + releases units left all-ACT. A pool_grow that
 *     needs fresh memory while such a unit is still mapped maps that unit's physical handle at
 *     the new address instead (one handle, two mappings until the old one is unmapped —
 *     invariant I2 relaxed as S:205 allows); pending work on the memory is ordered through the
 *     donor chunks' free events. pool_grow of a unit still awaiting unmap reuses it as is.
 * Device-synchronising calls from the worker thread: do not run it during stream capture.
 * ellm_vmm_sync waits until the worker is idle and returns its sticky error (ELLM_ERR_CUDA)
 * or ELLM_OK. NO_DEVICE on a host-only pool; INVALID_ARG for premap_bytes < 0 or
 * async_unmap not in {0,1}. */
int ellm_set_vmm_overlap(ellm_pool* pool, int64_t premap_bytes, int32_t async_unmap);
int ellm_vmm_sync(ellm_pool* pool);

/* Launch overlap between consecutive attention calls of this pool on one stream (programmatic
 * dependent launch): with enable = 1 a full-grid attention launch may start on
 * SMs the previous attention launch has left, streaming its layer's K/V before it waits for
 * that launch; everything else (Q, appends, outputs, split-K workspace) follows the wait. For
 * callers that issue a model's layers back to back; a caller that records events or issues
 * other work between attention calls gains nothing from it (and was measured slower in the C5
 * churn loop), hence off by default. ELLM_PDL=0/1 in the environment overrides. INVALID_ARG
 * for enable not in {0,1}; NO_DEVICE on a host-only pool. */
int ellm_set_launch_overlap(ellm_pool* pool, int32_t enable);

/* ---- activation eTensors in the unified pool --------------
 * act_alloc: an activation tensor slot of ceil(bytes / chunk_bytes) consecutive ACT chunks
 *   that are not inside another slot — the run with the highest last chunk id (activations
 *   fill the pool from the top, KV inflation takes the lowest ACT ids: DESIGN.md R16). Its
 *   units are mapped if needed (on this thread); memory an earlier slot or KV chunk freed on
 *   another stream is waited for on `stream`. *first_out = first chunk; *ptr_out (optional)
 *   = device address pool_base + first*chunk_bytes (NULL on a host-only pool). bytes <= 0 ->
 *   INVALID_ARG; no such run -> NO_CHUNKS. Chunks stay ACT-owned.
 * act_free: end the slot starting at chunk `first` (work on `stream` so far is its last use).
 *   Its chunks stay ACT and mapped ("mapped, available"): pool_grow can take them
 *   as KV with no driver call (the paper's zero-overhead ownership transfer).
 *   Not a slot start -> NOT_MAPPED; range -> OUT_OF_RANGE.
 * act_trim: release units kept mapped only for ended slots (unmapped now, or by the f1
 *   worker with async unmapping).
 * pool_grow never takes chunks inside live slots (NO_CHUNKS counts only idle ACT chunks). */
int ellm_act_alloc(ellm_pool* pool, int64_t bytes, void* stream, int64_t* first_out, void** ptr_out);
int ellm_act_free(ellm_pool* pool, int64_t first, void* stream);
int ellm_act_trim(ellm_pool* pool);
/* torch.cuda.memory.CUDAPluggableAllocator hooks: allocations of a torch MemPool built on
 * them become activation slots of the pool registered with ellm_torch_set_pool (NULL
 * detaches). alloc returns NULL (torch raises OOM) when the pool has no fitting run. */
int ellm_torch_set_pool(ellm_pool* pool);
void* ellm_torch_alloc(size_t size, int device, void* stream);
void ellm_torch_free(void* ptr, size_t size, int device, void* stream);

/* ---- a10: head-sharded output gather fused into attention ------
 * Boundary deviation from SURVEY §8(b): §8(b) sketches ellm_comm_init(pool, rank, world, NCCL
 * unique id) for an NCCL communicator inside the library. The exchange here is fused into the
 * attention kernel as peer-memory stores (no collective launch per layer), so the
 * library needs peer windows, not a communicator: ellm_gather_window_create / ellm_ipc_open /
 * ellm_gather_attach replace ellm_comm_init, and the 64-byte IPC handles travel over the
 * caller's process group (torch.distributed, shard.PeerGather). NCCL stays on the caller's side
 * only as the comparison path (bench.py --gather nccl).
 * KV-head sharding over N GPUs of one box: rank i owns kv-heads [i*Hkv/N, (i+1)*Hkv/N) and
 * q-heads [i*Hq/N, (i+1)*Hq/N) (its pool is created with the local counts). After attention
 * every rank needs all N ranks' head outputs. Instead of attention followed by an all-gather,
 * the attention kernel's split-K merge stores each finished output row directly into EVERY
 * rank's gather window over peer memory (NVLink P2P stores); the CTAs count their completion at
 * GPU scope and the last one adds the call's request count to every rank's flag word for that
 * layer (one system-scope release per call).
 * A gather window is one device allocation per rank, identical size on all ranks:
 *   [0, ELLM_GATHER_DATA_OFFSET)     uint32 flag words, one per layer (monotone counters)
 *   [ELLM_GATHER_DATA_OFFSET, bytes) rows: a call with out_offset writes [n, Hq_total, d] bf16
 *                                     at data + out_offset (global q-head order).
 * window_create: cudaMalloc + zero on `device` (makes it the calling thread's current device);
 *   ipc_handle_out (optional, 64 B) receives its cudaIpcMemHandle_t for the other ranks.
 * ipc_open / ipc_close: map / unmap another process's window (cudaIpcOpenMemHandle, lazy peer
 *   access; a handle that cannot be opened -> ELLM_ERR_PEER). The caller owns windows and
 *   opened mappings; they must outlive the attachment.
 * gather_attach: windows[i] = rank i's window as seen from this process (own window at
 *   windows[rank]); heads_q_total must equal world * the pool's Hq (INVALID_ARG), world in
 *   [1, 8] and rank < world (OUT_OF_RANGE), windows 256-B aligned and non-NULL. Reads this
 *   rank's current flag values: all ranks must be idle (attach everywhere, then a barrier).
 * attention_gather: paged_decode_attention (k_new == v_new == NULL) or decode_append_attention
 *   (both given; same preconditions and errors as those calls) whose output goes to every
 *   rank's window at out_offset (16-B aligned; past the window -> OUT_OF_RANGE; not attached ->
 *   INVALID_ARG). Every rank must issue the same sequence of calls with the same requests.
 * gather_wait: makes `stream` wait until this rank's flag word of `layer` shows every rank's
 *   rows of all attention_gather calls issued so far for that layer (one 1-thread kernel;
 *   after ELLM_GATHER_TIMEOUT_MS, default 20000, it traps: a missing peer fails the stream
 *   with ELLM_ERR_CUDA instead of hanging it). Window rows of one layer may be rewritten by the
 *   next call for that layer only after every rank has consumed them (the caller's order). */
#define ELLM_GATHER_DATA_OFFSET 4096
int ellm_gather_window_create(int32_t device, int64_t bytes, void** window_out, void* ipc_handle_out);
int ellm_gather_window_destroy(void* window);
int ellm_ipc_open(const void* ipc_handle, void** window_out);
int ellm_ipc_close(void* window);
int ellm_gather_attach(ellm_pool* pool, int32_t world, int32_t rank, int32_t heads_q_total,
                       void* const* windows, int64_t window_bytes);
int ellm_gather_detach(ellm_pool* pool);
int ellm_attention_gather(ellm_pool* pool, int32_t layer, int32_t n, const int32_t* req_ids,
                          const void* k_new, const void* v_new, const void* q, int64_t out_offset,
                          float softmax_scale, void* stream);
int ellm_gather_wait(ellm_pool* pool, int32_t layer, void* stream);
/* gather_wait_next: the same ordering as gather_wait(layer), folded into the NEXT attention
 * launch of this pool (paged_decode_attention, decode_append_attention or attention_gather, on
 * the stream the caller would have passed to gather_wait): that launch's producer warp streams
 * its first K/V tiles, then spins (acquire, system scope, bounded like gather_wait) until the
 * flag of `layer` reaches the target fixed by this call, and only then stages Q or writes. This
 * models Q(l+1) depending on the gathered rows of layer l without a wait kernel between two
 * attention launches, so they still overlap (launch overlap / PDL). Without a following attention
 * launch nothing waits: call gather_wait instead. Requires that the peers' launches progress
 * independently of this launch (one GPU per rank, or ranks sharing one stream): a spinning CTA
 * holds its SM. One wait is pending at a time: a second call before the next attention launch
 * replaces the first (fold the wait the next launch actually needs). Errors as gather_wait; no
 * stream argument. */
int ellm_gather_wait_next(ellm_pool* pool, int32_t layer);
/* cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, stream): host <-> window copies. */
int ellm_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* Swap engine selection: 0 = SM copy kernels (default), 1 = DMA copy engines (one
 * cudaMemcpyAsync per maximal contiguous run of the chunk list, one cudaMemcpy2DAsync per maximal
 * evenly strided run), 2 = as 1 for deflate / offload, and a staged inflate: the
 * host link writes 256 MiB batches into a device staging buffer outside the KV pool, then an SM
 * copy moves them into the chunks, 3 = as 1 for deflate / offload, and inflate staged through
 * memory owned by a second CUDA context on the pool's device (created by this call, once per
 * pool): 256 MiB batches host -> that context's staging buffer -> device-to-device into the
 * chunks, all on the caller's stream (host-link writes into memory of the decode's own context
 * slow a concurrent decode ~2x; into another context's memory ~1.1x: DESIGN.md §5 C3). All are
 * exact byte copies. INVALID_ARG outside 0..3; mode 3 returns CUDA (ellm_last_cuda_error = 10000 +
 * CUresult for a driver failure) or UNSUPPORTED if the side context cannot be created. */
int ellm_set_swap_mode(ellm_pool* pool, int32_t mode);
/* Host -> device copy of `bytes` from host `src` (pinned) to device `dst` on `stream`, staged in
 * 256 MiB pieces through the same side-context buffer as swap mode 3 (created on first use), so
 * that uploading the next step's inputs beside a running decode costs it ~1.1x instead of ~2x
 * (DESIGN.md §6 e2e). Exact copy; stream-ordered like cudaMemcpyAsync (a use of the staging
 * buffer on another stream waits for the previous one). INVALID_ARG (null pointer with bytes > 0,
 * bytes < 0), NO_DEVICE, CUDA / UNSUPPORTED as ellm_set_swap_mode(3). */
int ellm_upload(ellm_pool* pool, void* dst, const void* src, int64_t bytes, void* stream);

/* ---- introspection (parity tests) --------------------------------------------------- */
/* table of req: entries[0 .. n_out) for the ceil(len/T) live logical chunks. */
int ellm_get_table(const ellm_pool* pool, int32_t req_id, int32_t* entries, int32_t cap,
                   int32_t* n_out, int32_t* len_out);
/* states of chunks [first, first+n): out[i] = ELLM_CHUNK_FREE (KV-owned, mapped, unused),
 * ELLM_CHUNK_USED (referenced by a table), ELLM_CHUNK_ACT (activation-owned, idle) or
 * ELLM_CHUNK_ACT_SLOT (activation-owned, inside a live activation slot). */
enum { ELLM_CHUNK_FREE = 0, ELLM_CHUNK_USED = 1, ELLM_CHUNK_ACT = 2, ELLM_CHUNK_ACT_SLOT = 3 };
int ellm_chunk_states(const ellm_pool* pool, int64_t first, int64_t n, uint8_t* out);
/* copy the canonical [L][2][Hkv][T][d] image (chunk_bytes) of device chunk `chunk_id` to
 * host_dst, un-rotating its slabs (synchronises `stream`). */
int ellm_read_chunk(ellm_pool* pool, int64_t chunk_id, void* host_dst, void* stream);
/* copy chunk_bytes of host slot `slot` to host_dst (synchronises the device). */
int ellm_read_host_slot(ellm_pool* pool, int64_t slot, void* host_dst);
/* Map req's physical chunks, in logical order, contiguously into a fresh VA span
 * (multi-mapping) and return its device pointer: the paper's literal KV eTensor
 * view. Needs chunk_bytes % granularity == 0 and all chunks on the device. */
int ellm_alias_request(ellm_pool* pool, int32_t req_id, void** contig_dev_ptr);
int ellm_unalias_request(ellm_pool* pool, int32_t req_id);

const char* ellm_status_string(int status);
int ellm_last_cuda_error(const ellm_pool* pool);
/* Number of kernels this pool has launched so far (bench accounting). */
int64_t ellm_kernel_launches(const ellm_pool* pool);
/* Timeline instrumentation of the attention kernel (profiling; tools/attn_timeline.py). With a
 * caller-owned device buffer of launches * #SM * 8 uint64, attention launch k of this pool
 * (counted from this call) writes, per CTA b, into slot (k % launches): [b*8 + 0] start,
 * [1] producer past griddepcontrol.wait, [2] first stage data seen, [3] streaming done,
 * [4] merges done, [5] end, all %globaltimer ns (0 = not reached), [6] requests merged, [7] SM id.
 * NULL disables. launches < 0 or (buffer with launches == 0) -> INVALID_ARG. While set, every
 * prefill launch also writes, for its first CTA and key tiles t < 16, clock64 stamps of the
 * TMA / MMA / softmax hand-offs into words [t*16 + 0..13] of the buffer (tools/pf_timeline.py). */
int ellm_set_attn_trace(ellm_pool* pool, void* device_buf, int32_t launches);
/* Measurement knob: split the attention kernel's static work over CTA b in proportion to w[b]
 * (n >= the launch's CTA count; n = 0 restores equal shares). Outputs stay within R8. */
int ellm_debug_attn_weights(ellm_pool* pool, const float* w, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* ELLM_H */
