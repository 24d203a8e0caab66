/*
 * gh.h — C ABI of the B200-native Glinthawk two-tier decode path.
 *
 * The reference (`tierplan`, /root/reference/proj) has no decode code; its only coupling to
 * the kernels is (a) the model-shape contract, (b) per-prompt KV sizing, (c) the inter-tier
 * message byte counts and (d) the per-stage kernel-latency CSV.  Every entry point below cites
 * the reference symbol it implements or the paper operation it executes (P = PAPER.md).
 *
 * Conventions
 *  - Plain C types only: no torch, no C++ types.  `stream` arguments are `cudaStream_t`
 *    passed as `void*` (NULL = legacy default stream).  All device pointers are raw.
 *  - Status codes, never exceptions.  0..3 mirror the reference CLI exit codes
 *    (proj/include/tierplan/commands.hpp:14-17): OK / internal / validation / feasibility.
 *    gh_last_error() returns a thread-local message for the last failing call.
 *  - Ownership: the library owns weights and the KV arena; the caller owns token / position /
 *    slot arrays, activations and message buffers.  Hot calls never allocate device memory.
 *  - Threading: a handle is used by one host thread at a time; device work is asynchronous on
 *    the given stream.  Accounting calls are pure functions (reference S:105-106).
 *  - Storage dtype = spec.dtype_bytes (4 = fp32, 2 = bf16); compute is fp32 (P:514:
 *    "Kernel computations run at FP32, while kernel results are stored in the model's native
 *    data type").
 *
 * Message layouts (row-major, token-major, storage dtype; byte counts = PayloadModel,
 * proj/src/netmodel.cpp:18-24):
 *    fwd  (Tier-1 -> Tier-2) per token: [ x (D) | q (D) | k (D_kv) | v (D_kv) ]
 *    bwd  (Tier-2 -> Tier-1) per token: [ x (D) | attn (D) ]
 *    pp   (Tier-1 -> Tier-1) per token: [ x (D) ]
 */
#ifndef GH_GH_H
#define GH_GH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GH_ABI_VERSION 1

typedef enum {
  GH_OK = 0,
  GH_EINTERNAL = 1,     /* commands.hpp:14-17 exit 1 */
  GH_EINVAL = 2,        /* ValidationError, errors.hpp:18-22, exit 2 */
  GH_EINFEASIBLE = 3,   /* FeasibilityError, errors.hpp:24-32, exit 3 (e.g. KV slots exhausted) */
  GH_ECUDA = 4,         /* CUDA runtime / driver error (or no device) */
  GH_ENCCL = 5,         /* NCCL error or NCCL library unavailable */
  GH_EUNSUPPORTED = 6   /* shape/dtype the kernels do not implement */
} gh_status;

/* First nine fields = TransformerSpec (proj/include/tierplan/model.hpp:14-28), vocab_size 0 =
 * absent.  rope_theta / norm_eps are the sidecar hyper-parameters the reference JSON rejects
 * (model.cpp:92-100) and that the paper leaves to the Llama-2 defaults. */
typedef struct gh_model_spec {
  uint64_t n_layers;     /* N    */
  uint64_t d_model;      /* D    */
  uint64_t d_kv;         /* D_kv */
  uint64_t d_hidden;     /* D_h  */
  uint64_t n_heads;      /* H    */
  uint64_t n_kv_heads;   /* H_kv */
  uint64_t max_seq_len;  /* S    */
  uint64_t dtype_bytes;  /* 4 = fp32, 2 = bf16 */
  uint64_t vocab_size;   /* V    */
  float rope_theta;
  float norm_eps;
} gh_model_spec;

/* StageKind (proj/include/tierplan/profiles.hpp:13) */
typedef enum { GH_STAGE_NONATTENTION = 0, GH_STAGE_ATTENTION = 1, GH_STAGE_CLASSIFIER = 2 } gh_stage;

typedef struct gh_tier1 gh_tier1;
typedef struct gh_tier2 gh_tier2;
typedef struct gh_engine gh_engine;
typedef struct gh_comm gh_comm;

/* ------------------------------------------------------------------ misc */
int gh_abi_version(void);
const char* gh_last_error(void);
const char* gh_status_name(gh_status s);
/* Number of CUDA devices visible (0 on a GPU-less host; never fails). */
int gh_device_count(void);

/* ------------------------------------------------------------------ accounting (host only)
 * Bit-identical restatements of the reference's contract functions; tests compare each one
 * against the reference library compiled from /root/reference (oracle/_ref). */
gh_status gh_spec_validate(const gh_model_spec* spec);                     /* model.cpp:12-38 */
gh_status gh_kv_bytes_per_prompt(const gh_model_spec* spec, uint64_t seq_len,
                                 uint64_t* out);                           /* model.cpp:40-46 */
gh_status gh_nonattention_footprint(const gh_model_spec* spec, uint64_t batch,
                                    uint64_t* mem_accesses, uint64_t* flops); /* model.cpp:48-56 */
gh_status gh_attention_footprint(const gh_model_spec* spec, uint64_t batch, uint64_t seq_len,
                                 uint64_t* mem_accesses, uint64_t* flops); /* model.cpp:58-67 */
gh_status gh_weights_bytes(const gh_model_spec* spec, uint64_t* out);    /* model.cpp:69-77 */
/* out[0] = tier1_to_tier2_per_token, out[1] = tier2_to_tier1_per_token,
 * out[2] = intra_tier1_per_token (netmodel.cpp:18-24) */
gh_status gh_payload_bytes(const gh_model_spec* spec, uint64_t out[3]);
gh_status gh_layer_spans(uint64_t n_layers, uint64_t nodes, uint64_t* spans_out); /* optimizer.cpp:116-123 */
gh_status gh_node_weight_bytes(const gh_model_spec* spec, uint64_t tier1_nodes,
                               uint64_t* bytes_out);                       /* optimizer.cpp:125-136 */
gh_status gh_two_tier_context_slots(const gh_model_spec* spec, uint64_t tier1_nodes,
                                    uint64_t tier2_per_tier1, uint64_t tier2_memory_per_node,
                                    uint64_t seq_len, uint64_t* out);      /* optimizer.cpp:175-192 */
/* Rounded sqrt(2) grid (profiles.cpp:232-245).  Writes at most `cap` entries, *n = full count. */
gh_status gh_batch_grid(uint64_t max_batch, uint64_t* out, uint64_t cap, uint64_t* n);
/* Tier split of a Tier-1 batch over K' Tier-2 ranks: balanced shards differing by at most one
 * prompt (analytic.cpp:119), lower ranks first; off/cnt arrays of length kp. */
gh_status gh_shard_plan(uint64_t batch, uint64_t kp, uint64_t* off, uint64_t* cnt);
/* Rank layout of the engine's tier split (host only; gh_engine_create uses exactly this):
 * world = T + n1 * K' ranks.  Tier-1 ranks come first -- n1 = tier1_ranks pipeline spans
 * (layer_spans, optimizer.cpp:116-123) or T = tier1_tp tensor-parallel ranks sharing every layer
 * -- then K' Tier-2 ranks per span, rank T + s*K' + j holding prompt shard j
 * (gh_shard_plan, analytic.cpp:119) of span s's layers.  world 1 = colocated. */
typedef struct gh_rank_layout {
  int role;                 /* 0 colocated, 1 Tier-1, 2 Tier-2 */
  int span;                 /* Tier-1 pipeline span served */
  int tp_rank;              /* Tier-1 tensor-parallel slice (0 without TP) */
  int shard;                /* Tier-2: shard index within its span; -1 otherwise */
  uint32_t kp;              /* Tier-2 ranks per span (K'); 0 colocated */
  uint32_t layer_begin, layer_end;
  uint32_t row_off, row_cnt;  /* rows of each in-flight batch whose KV this rank holds (Tier-2) */
} gh_rank_layout;
gh_status gh_engine_layout(uint32_t world, uint32_t rank, uint32_t tier1_ranks, uint32_t tier1_tp,
                           uint64_t n_layers, uint32_t batch, gh_rank_layout* out);
/* Throughput identity B_total*IF/mean(TBT) (des.cpp:298-310); gen_ts in ns. */
gh_status gh_throughput_from(const int64_t* gen_ts_ns, uint64_t n, uint64_t batch_total,
                             uint64_t inflight, double* tokens_per_s);

/* ------------------------------------------------------------------ kernel-latency boundary
 * Writes rows of `device,stage,seq_len,batch_size,latency_us` (profiles.hpp:66-69,
 * parse_profile profiles.cpp:168-224).  mode "w" writes the header first, "a" appends rows.
 * Rejects non-positive latency and a stage name outside {nonattention,attention,classifier}. */
gh_status gh_profile_write_csv(const char* path, const char* mode, const char* device,
                               gh_stage stage, uint64_t seq_len, const uint64_t* batches,
                               const double* latency_us, uint64_t n);

/* ------------------------------------------------------------------ Tier-1 (weights; F1, F3, classifier)
 * Owns layers [layer_begin, layer_end) (a layer_spans block), the embedding when
 * layer_begin == 0 and the final norm + classifier when layer_end == n_layers.  Weights are
 * generated on the device from `weight_seed`.
 * max_batch bounds B for every call (scratch is sized at create time). */
gh_status gh_tier1_create(const gh_model_spec* spec, int device, uint32_t layer_begin,
                          uint32_t layer_end, uint64_t weight_seed, uint32_t max_batch,
                          gh_tier1** out);
gh_status gh_tier1_destroy(gh_tier1* t1);
/* x[b,:] = E[tok[b],:]   (tok: device int32 [B]; x: device [B, D]) */
gh_status gh_tier1_embed(gh_tier1* t1, uint32_t B, const int32_t* tok, void* x, void* stream);
/* F1: RMSNorm -> x*[Wq|Wk|Wv] -> RoPE(pos) -> msg_fwd [x|q|k|v]  (pos: device int32 [B]) */
gh_status gh_tier1_pre(gh_tier1* t1, uint32_t layer, uint32_t B, const void* x,
                       const int32_t* pos, void* msg_fwd, void* stream);
/* F3: h = attn*Wo + x; x_next = h + W2(silu(W1 rms(h)) * W3 rms(h)).  msg_bwd [x|attn]. */
gh_status gh_tier1_post(gh_tier1* t1, uint32_t layer, uint32_t B, const void* msg_bwd,
                        void* x_next, void* stream);
/* Classifier: RMSNorm -> x*Wcls^T -> greedy argmax (lowest index on ties).
 * logits (optional, device fp32 [B, V]); next_tok device int32 [B]. */
gh_status gh_tier1_classify(gh_tier1* t1, uint32_t B, const void* x, float* logits,
                            int32_t* next_tok, void* stream);
/* Classifier with temperature sampling: inv_temperature [B] device fp32 (1/T, 0 = greedy row),
 * seed [B] device uint32, pos [B] device int32 (the position of the token being decoded);
 * logits (required, device fp32 [B, V]) receive the logits the sampler reads. */
gh_status gh_tier1_classify_sample(gh_tier1* t1, uint32_t B, const void* x, const int32_t* pos,
                                   const float* inv_temperature, const uint32_t* seed, float* logits,
                                   int32_t* next_tok, void* stream);

/* ------------------------------------------------------------------ Tier-2 (KV context; F2)
 * KV arena for layers [layer_begin, layer_end) and n_slots prompts at max_seq_len:
 * n_slots * 2 * dtype * S * D_kv * span bytes (<= two_tier_context_slots). */
gh_status gh_tier2_create(const gh_model_spec* spec, int device, uint32_t layer_begin,
                          uint32_t layer_end, uint32_t n_slots, gh_tier2** out);
gh_status gh_tier2_destroy(gh_tier2* t2);
/* F2: append (k,v) of msg_fwd at pos[b] into slot[b], attend over positions
 * 0..pos[b] with the new key included, write msg_bwd [x|attn].
 * slot: device uint32 [B]; pos: device int32 [B].  Returns GH_EINFEASIBLE (checked on the
 * host only when check_host != 0 via gh_tier2_check) for slot >= n_slots or pos >= S. */
gh_status gh_tier2_attend(gh_tier2* t2, uint32_t layer, uint32_t B, const uint32_t* slot,
                          const int32_t* pos, const void* msg_fwd, void* msg_bwd, void* stream);
/* KV append of every row of msg_fwd at (slot[b], pos[b]) without attention: run before
 * gh_tier2_attend when rows of one step share a slot (chunked prefill), so that every row sees
 * the keys of the rows before it.  gh_tier2_attend's own append rewrites the same values. */
gh_status gh_tier2_append(gh_tier2* t2, uint32_t layer, uint32_t B, const uint32_t* slot,
                          const int32_t* pos, const void* msg_fwd, void* stream);
/* Host-side admission check of a batch (slot < n_slots, 0 <= pos < S). */
gh_status gh_tier2_check(const gh_tier2* t2, uint32_t B, const uint32_t* slot_host,
                         const int32_t* pos_host);
/* Fill positions [0, n_positions) of slots [0, n_slots_to_fill) (all layers) with synthetic
 * N(0,1)-like values from `seed` (benchmark pre-fill; content does not change the cost).  Paged
 * arena: each slot is filled up to min(n_positions, its mapped positions). */
gh_status gh_tier2_fill_synthetic(gh_tier2* t2, uint64_t seed, uint32_t n_slots_to_fill,
                                  uint32_t n_positions, void* stream);
/* Paged KV arena (the page-granular form of the slot arena): n_slots logical slots
 * share a pool of n_pages pages of GH_KV_PAGE_POSITIONS positions (all layers of the span, K and V,
 * every KV head: n_pages * 2 * dtype * 64 * D_kv * span bytes).  A slot's positions must be mapped
 * before a step attends them; pages return to the pool on unmap, so prompts of different lengths
 * share the arena instead of each reserving max_seq_len.  Attention results are bit-identical to
 * the contiguous arena. */
#define GH_KV_PAGE_POSITIONS 64
gh_status gh_tier2_create_paged(const gh_model_spec* spec, int device, uint32_t layer_begin,
                                uint32_t layer_end, uint32_t n_slots, uint32_t n_pages, gh_tier2** out);
/* Ensure positions [0, n_positions) of `slot` are backed by pages (grows the slot's mapping; no
 * partial allocation: GH_EINFEASIBLE when the pool is short).  Synchronises `stream` first, so
 * the table is updated between steps.  No-op (n_positions <= S checked) on a contiguous arena. */
gh_status gh_tier2_map(gh_tier2* t2, uint32_t slot, uint32_t n_positions, void* stream);
/* Return the slot's pages to the pool (after the last step that reads it has been queued on the
 * stream the next gh_tier2_map synchronises). */
gh_status gh_tier2_unmap(gh_tier2* t2, uint32_t slot);
uint32_t gh_tier2_pages_free(const gh_tier2* t2);
/* Copy one (layer, slot, kv, head) block of positions [0, n) to host (tests). */
gh_status gh_tier2_read_kv(gh_tier2* t2, uint32_t layer, uint32_t slot, uint32_t kv,
                           uint32_t head, uint32_t n, void* host_out);
uint64_t gh_tier2_arena_bytes(const gh_tier2* t2);
/* Swap a slot's context out to / back from host memory (preemption by swap instead of
 * recompute, P:471-479 batch state).  The host buffer holds positions [0, n) of every owned
 * layer in a library-defined layout of gh_tier2_kv_swap_bytes(t2, n) bytes; restore may target
 * a different slot (and different pages) mapped for n positions.  Synchronous on `stream`. */
uint64_t gh_tier2_kv_swap_bytes(const gh_tier2* t2, uint32_t n_positions);
gh_status gh_tier2_kv_swap(gh_tier2* t2, uint32_t slot, uint32_t n_positions, void* host,
                           int to_host, void* stream);

/* ------------------------------------------------------------------ NCCL transport
 * One communicator per process (one process per GPU).  `unique_id` is the 128-byte
 * ncclUniqueId produced by gh_comm_unique_id on rank 0 and distributed by the caller. */
gh_status gh_comm_unique_id(uint8_t out[128]);
gh_status gh_comm_create(const uint8_t unique_id[128], int nranks, int rank, int device,
                         gh_comm** out);
/* n_comms communicators at once (ids: n_comms * 128 bytes); the engine's tier split uses one
 * communicator per in-flight batch so that batches never wait on each other's transfers. */
gh_status gh_comm_create_n(const uint8_t* unique_ids, int n_comms, int nranks, int rank,
                           int device, gh_comm** out);
gh_status gh_comm_destroy(gh_comm* c);

/* ------------------------------------------------------------------ Engine: one decode step
 * Role of this process:
 *   - colocated (world 1): Tier-1 for all layers + Tier-2 for all layers on one GPU;
 *   - tier split (world n >= 2): rank 0 = Tier-1 (all layers, embedding, classifier),
 *     ranks 1..n-1 = Tier-2 each holding the KV of its prompt shard for all layers.
 * A step decodes one token for each of the B prompts of every in-flight batch. */
typedef struct gh_engine_config {
  gh_model_spec spec;
  int device;
  uint64_t weight_seed;
  uint32_t batch;          /* prompts per in-flight batch (whole Tier-1 batch B*K') */
  uint32_t inflight;       /* IF in-flight batches (>=1); each has its own slots */
  uint32_t n_slots;        /* Tier-2 slots on this GPU (0 = exactly what the shard needs) */
  int use_graph;           /* capture the step in a CUDA graph (colocated only) */
  int transport;           /* tier split, pipelined step (gh_engine_step_all*): GH_TRANSPORT_* */
  uint32_t tier1_ranks;    /* tier split: Tier-1 pipeline stages (0/1 = one Tier-1 rank). With T > 1
                              ranks 0..T-1 hold contiguous layer spans (layer_spans,
                              optimizer.cpp:116-123; embedding on the first, classifier on the
                              last) and ranks T + s*K' + j are the K' Tier-2 ranks dedicated to
                              span s; world = T * (1 + K').  Peer transport only. */
  int prefill;             /* rows of one step may share a slot at consecutive positions
                              (chunked prefill mixed with decode rows); every row's key / value is
                              appended before attention (gh_tier2_append) */
  uint32_t kv_pages;       /* 0: contiguous slots of max_seq_len positions; > 0: paged KV arena of
                              kv_pages pages of GH_KV_PAGE_POSITIONS positions shared by the slots
                              (gh_tier2_create_paged; map with gh_engine_kv_map before a step) */
  uint32_t tier1_tp;       /* tier split: Tier-1 tensor parallelism (0/1 = none; SURVEY 8f-3,
                              if_tp analytic.cpp:22-29).  Ranks 0..T-1 each hold a head slice of
                              W_q/W_k/W_v and the matching input columns of W_o, and a hidden-unit
                              slice of W_1/W_3 and the matching input columns of W_2, for every
                              layer; W_o and W_2 are all-reduced inside their GEMM epilogue over
                              NVLink peer stores with per-slice flags (no NCCL).  Ranks T.. are the
                              K' = world - T Tier-2 ranks; the inter-tier messages are the
                              PayloadModel rows cut into T head blocks ([x_r|q_r|k_r|v_r] from
                              rank r, [x_r|attn_r] back to it).  bf16, head dim 128, peer
                              transport, gh_engine_step_all / step_all_host only; every Tier-1 rank
                              decodes the same tokens (feed them the same host tokens). */
} gh_engine_config;

/* Inter-tier message transport of the pipelined tier-split step.
 *  AUTO: PEER when every rank can map every peer buffer (CUDA IPC over NVLink), else NCCL.
 *  NCCL: grouped ncclSend/ncclRecv on the compute stream.
 *  PEER: copy-engine writes into the receiving GPU's message buffers + sequence-number flags
 *        (cuStreamWriteValue32 / cuStreamWaitValue32); no SM time is spent on transfers.
 * The per-batch entry points (gh_engine_step_device / step_host) always use NCCL. */
enum { GH_TRANSPORT_AUTO = 0, GH_TRANSPORT_NCCL = 1, GH_TRANSPORT_PEER = 2 };
/* Transport in use (split roles), -1 when colocated. */
int gh_engine_transport(const gh_engine* e);

gh_status gh_engine_create(const gh_engine_config* cfg, gh_comm* comm, gh_engine** out);
gh_status gh_engine_destroy(gh_engine* e);
/* Rank role: 0 = colocated, 1 = tier1, 2 = tier2 */
int gh_engine_role(const gh_engine* e);
/* Device-resident step for in-flight batch `ib`: tokens/pos/slots are device arrays owned by
 * the engine (see gh_engine_io).  next_tok is written on device. */
gh_status gh_engine_step_device(gh_engine* e, uint32_t ib, void* stream);
/* End-to-end step through host buffers: copies tok_host/pos_host (pinned or pageable) to the
 * device, runs the step, copies next tokens (and optionally logits [B,V] fp32) back.
 * Synchronous on `stream` when it returns.  Tier-2 ranks pass NULLs. */
gh_status gh_engine_step_host(gh_engine* e, uint32_t ib, const int32_t* tok_host,
                              const int32_t* pos_host, int32_t* next_host, float* logits_host,
                              void* stream);
/* Full step over all in-flight batches, pipelined across batches (tier split) or sequential
 * (colocated).  Device-resident inputs (engine io buffers). */
gh_status gh_engine_step_all(gh_engine* e, void* stream);
/* End-to-end variant of gh_engine_step_all: copies every in-flight batch's tokens and positions
 * from host ([inflight][batch] int32 each, row per batch), runs the pipelined step and copies
 * the next tokens back ([inflight][batch]).  Synchronous.  Tier-2 ranks pass NULLs. */
gh_status gh_engine_step_all_host(gh_engine* e, const int32_t* tok_host, const int32_t* pos_host,
                                  int32_t* next_host, void* stream);
/* Device pointers of in-flight batch ib: tok [B] int32, pos [B] int32, slot [B] uint32,
 * next [B] int32.  Any may be NULL. */
gh_status gh_engine_io(gh_engine* e, uint32_t ib, int32_t** tok, int32_t** pos,
                       uint32_t** slot, int32_t** next);
/* Device-side batch-state update for batch ib: tok <- next, pos += pos_increment (pos_increment
 * 0 keeps the context length fixed, the steady-state benchmark mode). Tier-1 / colocated only.
 * On the first of several Tier-1 pipeline spans it is applied when the batch's next step starts
 * (its tokens come back from the last span); host inputs of gh_engine_step_all_host replace it. */
gh_status gh_engine_advance(gh_engine* e, uint32_t ib, int pos_increment, void* stream);
/* Copy the next tokens of in-flight batch ib to host (synchronous; Tier-1 / colocated only). */
gh_status gh_engine_read_next(gh_engine* e, uint32_t ib, int32_t* next_host);
/* keep != 0: every classifier run of the engine also writes the fp32 logits [B, V] of its batch
 * (off by default: the argmax epilogue then stores no logits); gh_engine_read_logits copies the
 * last ones of batch ib to host (synchronous; Tier-1 ranks that own the classifier). */
gh_status gh_engine_keep_logits(gh_engine* e, int keep);
gh_status gh_engine_read_logits(gh_engine* e, uint32_t ib, float* logits_host);
gh_tier1* gh_engine_tier1(gh_engine* e);
gh_tier2* gh_engine_tier2(gh_engine* e);
/* Paged KV (kv_pages > 0): gh_tier2_map / gh_tier2_unmap of this rank's Tier-2 (slot = ib * batch
 * + row on a colocated engine, the local slot on a Tier-2 rank); no-ops for contiguous slots. */
gh_status gh_engine_kv_map(gh_engine* e, uint32_t slot, uint32_t n_positions);
gh_status gh_engine_kv_unmap(gh_engine* e, uint32_t slot);
/* gh_tier2_kv_swap on the engine's Tier-2 context (after the engine's queued steps finish). */
gh_status gh_engine_kv_swap(gh_engine* e, uint32_t slot, uint32_t n_positions, void* host, int to_host);
uint64_t gh_engine_kv_swap_bytes(const gh_engine* e, uint32_t n_positions);
/* Per-row context slots of in-flight batch ib (default ib * rows + row).  Colocated: one slot per
 * row of the batch; Tier-2 rank: the local slots of its shard's rows (gh_engine_shard); Tier-1:
 * no-op.  With prefill != 0 several rows may name the same slot (consecutive positions of one
 * prompt).  Synchronises the device. */
gh_status gh_engine_set_slots(gh_engine* e, uint32_t ib, const uint32_t* slot_host);
/* Per-row sampling of in-flight batch ib (batch state "temperature"): temperature 0 =
 * greedy (the default), > 0 = sample from softmax(logits / T) by the Gumbel-max rule with noise
 * from (seed, position, token id) -- deterministic and reproducible on the host
 * (oracle/sampling.py).  Synchronises the device; Tier-2 ranks ignore it. */
gh_status gh_engine_set_sampling(gh_engine* e, uint32_t ib, const float* temperature_host,
                                 const uint32_t* seed_host);
/* This rank's rows of every in-flight batch: a Tier-2 rank holds the KV of rows [off, off + cnt)
 * (shard `index` of kp, gh_shard_plan) in its local slots ib * cnt + (row - off); other roles
 * report index -1 and the whole batch.  kp = Tier-2 ranks per Tier-1 span (0 colocated). */
gh_status gh_engine_shard(const gh_engine* e, int* index, uint32_t* off, uint32_t* cnt, uint32_t* kp);
/* Launch count of this library's kernels since the last reset (device work accounting). */
uint64_t gh_kernel_launches(int reset);

/* ------------------------------------------------------------------ batch-state dispatcher
 * Glinthawk's dispatcher: batch-state objects for the IF in-flight batches, refilled
 * from the request queue as prompts finish.  Lanes = IF x B rows, each bound to its context slot;
 * per-Tier-2-shard page accounting on a paged arena (admission maps a request's positions, or,
 * with on_demand, its prompt and then a page at a time, preempting the shard's most recently
 * admitted request by recompute or by swap when a pool runs dry -- the oversubscription the
 * planner assumes, optimizer.cpp:42-45, 194-207).  Decisions depend only on lengths, max_new and
 * page counts, so in a tier split every rank runs the same dispatcher over the same requests
 * (SPMD; Tier-2 ranks apply the KV actions of their shard, Tier-1 ranks feed tokens).  The
 * engine step is gh_engine_step_all (pipelined IF >= 2 split, or the colocated CUDA graphs);
 * lane inputs, page tables and sampling state are updated stream-ordered (no host
 * synchronisation per change), and a step's tokens are read one step later.
 * Chunked prefill (prefill_chunk > 1; needs gh_engine_config.prefill): the idle lanes of
 * an in-flight batch's shard carry further prompt tokens of that shard's lanes still reading
 * their prompts (up to prefill_chunk tokens of one request per step, at consecutive positions of
 * the request's own slot). */
typedef struct gh_dispatcher gh_dispatcher;
typedef struct gh_dispatch_config {
  uint32_t max_new;      /* tokens generated per request */
  int on_demand;         /* paged arena: map the prompt, grow a page at a time, preempt when dry */
  int preempt_swap;      /* preempt by swapping the context to host memory (else recompute) */
  int order_shortest;    /* admit the shortest prompt first (else FIFO) */
  uint32_t prefill_chunk; /* prompt tokens of one request per step (0 / 1: one; > 1: chunked prefill) */
} gh_dispatch_config;
typedef struct gh_dispatch_stats {
  uint64_t steps, admitted, finished, tokens, preemptions, swaps;
  uint32_t peak_pages;   /* most pages of one shard's pool in use at once */
  uint64_t lane_steps;   /* busy lanes summed over steps: tokens processed (prompt, generated, recomputed) */
  uint64_t context_sum;  /* positions attended summed over busy lane-steps (mean context = / lane_steps) */
} gh_dispatch_stats;
/* Not for engines with Tier-1 pipeline spans (tier1_ranks > 1). */
gh_status gh_dispatcher_create(gh_engine* e, const gh_dispatch_config* cfg, gh_dispatcher** out);
gh_status gh_dispatcher_destroy(gh_dispatcher* d);
/* Queue a request generating max_new tokens (0 = the configured max_new); GH_EINFEASIBLE when it
 * can never fit a slot / a shard's page pool. */
gh_status gh_dispatcher_submit(gh_dispatcher* d, const int32_t* prompt, uint32_t len, float temperature,
                               uint32_t seed, uint32_t max_new, uint64_t* id);
/* One engine step over every in-flight batch; *busy = 0 once every request has finished. */
gh_status gh_dispatcher_step(gh_dispatcher* d, int* busy);
/* Steps until every submitted request has finished and its tokens are on the host. */
gh_status gh_dispatcher_run(gh_dispatcher* d, uint64_t* steps);
/* Generated tokens of a finished request (max_new; zeros on Tier-2 ranks). */
gh_status gh_dispatcher_result(const gh_dispatcher* d, uint64_t id, int32_t* tokens, uint32_t cap, uint32_t* n);
gh_status gh_dispatcher_stats(const gh_dispatcher* d, gh_dispatch_stats* out);

/* The dispatcher's decision logic alone (host only, no GPU): plan -> the caller runs the step ->
 * commit -> resolve (the tokens of the oldest committed step, any lag).  Lane inputs: src 0 idle
 * (a dummy token at position 0), 1 host token, 2 the token the lane's previous step generated.
 * KV actions (op 0 map [0, n), 1 unmap, 2 swap out [0, n) to buffer `buf`, 3 swap in) apply to
 * the lane's slot before the step. */
typedef struct gh_sched gh_sched;
typedef struct gh_sched_config {
  uint32_t batch, inflight, kp, pages, max_seq, max_new;
  int on_demand, preempt_swap, order_shortest;
  uint32_t prefill_chunk;
} gh_sched_config;
/* src 0 idle (dummy token at position 0), 1 host token `tok`, 2 the token the lane's previous step
 * generated; home = the lane whose slot the row appends to and attends over (itself, or with
 * chunked prefill the lane whose prompt token it carries). */
typedef struct gh_lane_input { int32_t src, tok, pos; uint32_t home; } gh_lane_input;
typedef struct gh_kv_action { int32_t op; uint32_t lane; uint32_t n; uint64_t buf; } gh_kv_action;
gh_status gh_sched_create(const gh_sched_config* cfg, gh_sched** out);
gh_status gh_sched_destroy(gh_sched* s);
gh_status gh_sched_submit(gh_sched* s, const int32_t* prompt, uint32_t len, float temperature, uint32_t seed,
                          uint32_t max_new, uint64_t* id);
gh_status gh_sched_plan(gh_sched* s, gh_lane_input* inputs, gh_kv_action* actions, uint32_t cap, uint32_t* n_actions);
gh_status gh_sched_commit(gh_sched* s);
gh_status gh_sched_resolve(gh_sched* s, const int32_t* next_tokens);
int gh_sched_done(const gh_sched* s);
uint32_t gh_sched_unresolved(const gh_sched* s);
gh_status gh_sched_result(const gh_sched* s, uint64_t id, int32_t* tokens, uint32_t cap, uint32_t* n);
gh_status gh_sched_stats(const gh_sched* s, gh_dispatch_stats* out);

/* ------------------------------------------------------------------ diagnostics
 * Microbenchmark of the Tier-1 tcgen05 GEMM on device 0: Y[B,N] = X[B,K] W[N,K]^T (bf16) with
 * the plain-store epilogue.  flags = GEMM_DBG_* bits (1 no MMA, 2 no activation loads, 4 no L2
 * cache hints, 8 no epilogue); stages / cluster 0 = the production choice (cluster = CTAs per
 * thread-block cluster = K splits per tile, 1/2/4/8).  Returns the mean device
 * time per launch over `reps` launches (CUDA events) in *us. */
gh_status gh_debug_gemm_bench(int N, int K, int B, int flags, int stages, int cluster, int reps, float* us);
/* Same, rotating over `copies` weight buffers (copies * N*K*2 bytes > L2 defeats L2 reuse) and,
 * when trace != NULL, recording 16 globaltimer stamps per CTA of the last launch into trace
 * (ns; 0 start, 1 weights prefetched, 2 after griddepcontrol.wait, 3 first stage landed,
 * 4 last MMA issued, 5 epilogue done, 6 exit, 7.. epilogue phases of the last tile). */
gh_status gh_debug_gemm_trace(int N, int K, int B, int copies, int reps, float* us,
                              unsigned long long* trace, int trace_cap);
/* on == 1: bracket every Tier-1 GEMM launch of this process with CUDA events (serialising it:
 * no PDL overlap); _dump writes one line per (N, K, B, all-reduce) shape with the mean time and
 * weight-stream rate, then clears the records.  on == 2: timeline mode -- no events; every GEMM
 * launch (up to 2048) records per-CTA globaltimer stamps and _dump writes one line per launch
 * (first CTA start, median griddepcontrol.wait return, last CTA exit, in us). */
gh_status gh_debug_gemm_profile(int on);
gh_status gh_debug_gemm_profile_dump(char* buf, uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* GH_GH_H */
