/*
 * sinkr_cuda.h — C-ABI of the B200-native (sm_100a) SinkRouter decode engine.
 *
 * This is the drop-in boundary for the reference's C++ operator API
 * (/root/reference/proj/include/sinkr/ *.hpp).  Every entry point below names
 * the reference interface it replaces.  Plain pointers and sizes only; no
 * torch or C++ types cross the boundary.  A C++ shim with the reference's own
 * signatures and exception types sits on top: include/sinkr/cuda/router.hpp.
 *
 * Hot path per call: ONE persistent cooperative sm_100a kernel (step.cuh),
 * replayed from a CUDA graph on the engine stream, in three phases:
 *   routing — cosine proxy vs. the cached token-0 key (exact fp64, sequential
 *             sums), group mean, tau(L) compare -> route bitmap + Active list
 *   stream  — Split-K flash-decode over the Active groups only (TMA -> smem
 *             ring -> mma.sync hi/lo-split bf16, fp32 online softmax)
 *   merge   — log-sum-exp merge of the Split-K partials; Sink groups get
 *             bitwise-zero rows.
 * The three-kernel form (probe -> decode -> combine) is kept for A/B
 * profiling (SINKR_FUSED=0), score collection and the multi-rank merge.
 *
 * Threading: an engine is bound to one device and one stream; like the
 * reference's ThreadPool (parallel.hpp:15-18) it must not be driven by two host
 * threads at once.  Errors are reported as sinkr_status codes that mirror the
 * reference's exception classes; the message of the last failing call on the
 * calling thread is available from sinkr_last_error().
 */
#ifndef SINKR_CUDA_H_
#define SINKR_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Exception classes of the reference (router.cpp:37-38,51-53,60,86-90;
 * kv_cache.cpp:56-57,67-74,93,101,110-113; attention.cpp:15-22,187-190). */
typedef enum sinkr_status {
    SINKR_OK = 0,
    SINKR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    SINKR_OUT_OF_RANGE = 2,     /* std::out_of_range     */
    SINKR_RUNTIME_ERROR = 3,    /* std::runtime_error    */
    SINKR_LOGIC_ERROR = 4,      /* std::logic_error      */
    SINKR_CUDA_ERROR = 5,       /* CUDA runtime / driver failure */
    SINKR_NO_DEVICE = 6         /* no sm_100 device: the engine never falls back to the CPU */
} sinkr_status;

typedef struct sinkr_engine sinkr_engine;

/* CacheConfig (kv_cache.hpp:13-24).  num_seqs > 1 batches B independent caches
 * (the reference realises batch as independent KvCache instances)
 * so one launch serves all of them; 0 means 1. */
typedef struct sinkr_cache_config {
    size_t num_layers;
    size_t num_q_heads;  /* H_q */
    size_t num_kv_heads; /* H_kv */
    size_t head_dim;     /* D: 32, 64 or 128 */
    size_t capacity;     /* L_max tokens per (layer, seq, kv_head) slot */
    size_t num_seqs;     /* B */
} sinkr_cache_config;

/* The part of ThresholdProfile (calibration.hpp:21-34) that routing reads. */
typedef struct sinkr_threshold_profile {
    double coeffs[4]; /* a, b, c, d */
    double length_normalizer;
    double clamp_lo;
    double clamp_hi;
} sinkr_threshold_profile;

/* RoutingConfig (router.hpp:16-26). */
typedef struct sinkr_routing_config {
    double gamma; /* carried for parity; routing does not read it */
    sinkr_threshold_profile profile;
    const size_t* excluded_layers; /* reference default {0, 1} */
    size_t num_excluded_layers;
    int sink_on_tie; /* fault-injection hook: S >= tau instead of S > tau */
} sinkr_routing_config;

/* EngineOptions (router.hpp:69-76).  num_splits and block_size are validated
 * and accepted for API parity; the GPU partitions work over its SMs itself
 * (outputs agree within tolerance, loaded-token counts exactly).
 * global_context_len: tau(L) uses this length when the sequence is sharded
 * across GPUs (0 = this engine's token_count, router.cpp:89,113). */
typedef struct sinkr_engine_options {
    size_t num_splits;
    size_t block_size;
    int observe_only;
    size_t global_context_len;
} sinkr_engine_options;

/* LoadCounters (counters.hpp:9-28).  kv_floats_loaded counts K/V ELEMENTS as
 * the reference does (2 * rows * D per Active group), measured by the decode
 * kernel itself; the *_seconds fields come from CUDA events. */
typedef struct sinkr_load_counters {
    uint64_t kv_floats_loaded;
    uint64_t anchor_floats_loaded;
    uint64_t groups_active;
    uint64_t groups_skipped;
    double routing_seconds;
    double attention_seconds;
    double merge_seconds;
} sinkr_load_counters;

/* GroupStepInfo + RouteDecision (router.hpp:28-39,56-61).  Head scores are
 * returned in a separate H_q array (query-head order, router.cpp:118). */
typedef struct sinkr_group_info {
    size_t layer;
    size_t kv_head;
    double group_score;
    double threshold;
    int32_t sink;
    int32_t degenerate;
    uint64_t kv_floats_loaded;
    uint64_t tokens_loaded; /* rows streamed by the decode kernel (the skipped-block record) */
} sinkr_group_info;

const char* sinkr_last_error(void);
const char* sinkr_version(void);

/* ---- engine / KvCache (kv_cache.hpp:42-80) --------------------------------- */
/* KvCache::KvCache — allocates bf16 K/V [layer][seq][kv_head][capacity][D] in
 * HBM plus the f32 anchor table; throws like CacheConfig::validate
 * (kv_cache.cpp:32-39). */
sinkr_status sinkr_engine_create(const sinkr_cache_config* config, int device,
                                 sinkr_engine** out);
sinkr_status sinkr_engine_destroy(sinkr_engine* engine);
/* The engine's configuration (num_seqs filled in). */
sinkr_status sinkr_engine_config(sinkr_engine* e, sinkr_cache_config* out);
/* The engine's CUDA stream (cudaStream_t) — all work is ordered on it. */
void* sinkr_engine_stream(sinkr_engine* engine);

/* KvCache::append (kv_cache.cpp:61-84), for `rows` consecutive f32 host rows.
 * Rows are stored as bf16 (RNE).  On a slot's first row the anchor is captured
 * from the stored (bf16-rounded) key with the reference's rule: k0_norm =
 * (float)sqrt(sum (double)k^2), degenerate (< 1e-12) -> RUNTIME_ERROR. */
sinkr_status sinkr_kv_append(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                             const float* k, const float* v, size_t rows);
/* Same, for bf16 rows already on the device (device prefill path). */
sinkr_status sinkr_kv_append_device_bf16(sinkr_engine* e, size_t seq, size_t layer,
                                         size_t kv_head, const void* k, const void* v,
                                         size_t rows);
/* Appends `rows` synthetic rows generated on the device (see
 * oracle/sinkr_oracle.c:orc_fill_rows for the bit-identical CPU restatement):
 * value(row, j) = bf16(scale * gauss12(key, row * D + j)) for global rows
 * row = global_row0 .. global_row0 + rows - 1 (a sequence shard passes the
 * global index of its first row so every shard sees the same tokens). */
sinkr_status sinkr_kv_append_synthetic(sinkr_engine* e, size_t seq, size_t layer,
                                       size_t kv_head, uint64_t key_k, uint64_t key_v,
                                       float k_scale, float v_scale, size_t global_row0,
                                       size_t rows);
/* KvCache::length / token_count (kv_cache.cpp:86-96); token_count throws
 * LOGIC_ERROR when the sequence's slots are ragged. */
sinkr_status sinkr_kv_length(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                             size_t* out);
sinkr_status sinkr_kv_token_count(sinkr_engine* e, size_t seq, size_t* out);
/* KvCache::anchor (kv_cache.cpp:98-104): k0[D] and k0_norm. */
sinkr_status sinkr_kv_anchor(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                             float* k0, float* k0_norm);
/* Installs a replicated anchor on a sequence-shard engine whose slice does not
 * hold global token 0 (multi-GPU sequence sharding). */
sinkr_status sinkr_kv_set_anchor(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                                 const float* k0, float k0_norm);
/* KvCache::historical (kv_cache.cpp:106-121) as a copy: rows [from, to) as f32
 * (exact upcast of the stored bf16), for checkers and snapshots. */
sinkr_status sinkr_kv_read(sinkr_engine* e, size_t seq, size_t layer, size_t kv_head,
                           size_t from, size_t to, float* k, float* v);

/* ---- routing helpers (router.hpp:47-54,78; attention.hpp:82-85) ------------
 * Host scalar control logic of the reference, reproduced with the reference's
 * exact expression order (tau is computed on the host and handed to the probe
 * kernel so no device FMA contraction can perturb it). */
sinkr_status sinkr_threshold_for_length(size_t context_len,
                                        const sinkr_threshold_profile* profile, double* out);
sinkr_status sinkr_route(size_t layer, double score, size_t context_len,
                         const sinkr_routing_config* config, int* sink, double* threshold);
size_t sinkr_auto_num_splits(size_t context_len);
sinkr_status sinkr_split_ranges(size_t len, size_t num_splits, size_t* from_to);

/* ---- the hot path ---------------------------------------------------------- */
/* routed_decode_step (router.hpp:84-86, router.cpp:82-188) for sequence 0, or
 * for all B sequences with the _batch variant.  Host buffers:
 *   queries  [B][H_q][D] f32 (read)      outputs [B][H_q][D] f32 (written)
 *   groups   [B][H_kv]                   head_scores [B][H_q] f64
 *   counters summed over the batch (may be NULL).
 * One graph per call: an H2D copy of the queries + step parameters, then the
 * fused step kernel, which writes outputs and the routing record straight into
 * mapped pinned host memory (blocking until they are there). */
sinkr_status sinkr_routed_decode_step(sinkr_engine* e, const float* queries, size_t layer,
                                      const sinkr_routing_config* config,
                                      const sinkr_engine_options* options, float* outputs,
                                      sinkr_group_info* groups, double* head_scores,
                                      sinkr_load_counters* counters);
sinkr_status sinkr_routed_decode_batch(sinkr_engine* e, const float* queries, size_t layer,
                                       const sinkr_routing_config* config,
                                       const sinkr_engine_options* options, float* outputs,
                                       sinkr_group_info* groups, double* head_scores,
                                       sinkr_load_counters* counters);

/* The decode loop's append (KvCache::append, kv_cache.cpp:61-84):
 * ONE new token's K/V row to every (seq, kv_head) slot of `layer`.
 *   _async: d_k_new / d_v_new are device f32 [B][H_kv][D]; one kernel enqueued
 *           on the engine stream, no host sync (a slot's FIRST row takes the
 *           synchronous host path: anchor capture + degenerate check).
 *   sinkr_decode_append_step: host rows k_new / v_new, then the routed step of
 *           that layer over the grown cache -- one graph per call (H2D of
 *           params + queries + rows, append kernel, step kernel, results
 *           zero-copy), blocking like sinkr_routed_decode_batch.
 * Overflow -> RUNTIME_ERROR ("kv cache overflow"); as token_count requires
 * (kv_cache.cpp:90-96), a sequence's slots must be uniform after the append
 * for the step (LOGIC_ERROR otherwise, nothing appended). */
sinkr_status sinkr_kv_append_token_async(sinkr_engine* e, size_t layer, const float* d_k_new,
                                         const float* d_v_new);
sinkr_status sinkr_decode_append_step(sinkr_engine* e, const float* queries, const float* k_new,
                                      const float* v_new, size_t layer,
                                      const sinkr_routing_config* config,
                                      const sinkr_engine_options* options, float* outputs,
                                      sinkr_group_info* groups, double* head_scores,
                                      sinkr_load_counters* counters);

/* Device-resident variant: d_queries / d_outputs are device pointers; the
 * call only enqueues work on the engine stream (no host sync).  Routing
 * results stay on the device until sinkr_fetch_step_info (which syncs). */
sinkr_status sinkr_routed_decode_async(sinkr_engine* e, const float* d_queries, size_t layer,
                                       const sinkr_routing_config* config,
                                       const sinkr_engine_options* options, float* d_outputs);
sinkr_status sinkr_fetch_step_info(sinkr_engine* e, sinkr_group_info* groups,
                                   double* head_scores, sinkr_load_counters* counters);

/* Sequence-sharded multi-GPU split.  A rank's engine holds the
 * token slice it owns; sinkr_decode_rank_partial_async writes one
 * un-normalised LSE partial per (seq, kv_head, head): d_partial is
 * [B*H_kv][r][D+2] f32 laid out per unit as m[r] (log2 domain), l[r], acc[r][D].
 * After the caller all-gathers N such buffers (NCCL over NVLink),
 * sinkr_merge_rank_partials_async LSE-merges them into d_outputs; Sink units
 * (same bitmap on every rank) come out as bitwise zeros. */
size_t sinkr_rank_partial_floats(sinkr_engine* e);
sinkr_status sinkr_decode_rank_partial_async(sinkr_engine* e, const float* d_queries,
                                             size_t layer, const sinkr_routing_config* config,
                                             const sinkr_engine_options* options,
                                             float* d_partial);
sinkr_status sinkr_merge_rank_partials_async(sinkr_engine* e, const float* d_gathered,
                                             size_t num_ranks, float* d_outputs);

/* The same split with the collective fused into the step kernel: every rank's
 * kernel writes its LSE partials straight into every rank's exchange block
 * over NVLink (peer memory) as LL words {value, step tag} (one 8-byte store:
 * a reader that sees this step's tag sees the value, no fence, no arrival
 * counter); the CTAs that own output elements poll the words they need from
 * every rank and merge them into d_outputs -- one kernel per rank per step,
 * no NCCL call.
 *   sinkr_peer_setup       allocate this rank's exchange block (world <= 8)
 *   sinkr_peer_ipc_handle  64-byte cudaIpcMemHandle of the block (all-gather it)
 *   sinkr_peer_open        map every rank's block from the gathered handles
 *   sinkr_peer_set_blocks  same, from device pointers (ranks in one process)
 * All ranks must issue the same number of peer steps (the step tags count
 * them); a rank that never delivers turns into a step-kernel error after
 * 2 s (NaN outputs), never a hang, and the exchange refuses further steps
 * until every rank calls sinkr_peer_setup again (which resets it: a fresh
 * block, step tags from zero) and connects again. */
sinkr_status sinkr_peer_setup(sinkr_engine* e, uint32_t world, uint32_t rank, size_t* block_bytes);
sinkr_status sinkr_peer_ipc_handle(sinkr_engine* e, void* handle);
sinkr_status sinkr_peer_open(sinkr_engine* e, const void* handles);
sinkr_status sinkr_peer_set_blocks(sinkr_engine* e, void* const* blocks);
void* sinkr_peer_block(sinkr_engine* e);
sinkr_status sinkr_routed_decode_peer_async(sinkr_engine* e, const float* d_queries, size_t layer,
                                            const sinkr_routing_config* config,
                                            const sinkr_engine_options* options,
                                            float* d_outputs);
/* The peer-merged step with host buffers, like sinkr_routed_decode_batch: one
 * graph per call (H2D of the staged input block + the mode-3 step kernel,
 * outputs and routing record zero-copy into pinned host memory), blocking.
 * The outputs are the merge over ALL ranks; the routing record (decisions,
 * scores) is identical on every rank; the load counters and each group's
 * tokens_loaded / kv_floats_loaded cover THIS rank's shard only -- sum them
 * over the ranks for the whole step's traffic (the reference's per-group
 * count, router.cpp:181-182; tests/test_gpu_sharding.py sums them). */
sinkr_status sinkr_routed_decode_peer(sinkr_engine* e, const float* queries, size_t layer,
                                      const sinkr_routing_config* config,
                                      const sinkr_engine_options* options, float* outputs,
                                      sinkr_group_info* groups, double* head_scores,
                                      sinkr_load_counters* counters);

/* ---- instrumentation ------------------------------------------------------- */
/* Launch count of the last step (kernels of this library) and the device
 * time (ms) of its decode kernel, measured with events on the engine stream. */
sinkr_status sinkr_last_step_stats(sinkr_engine* e, uint32_t* kernel_launches,
                                   float* decode_ms, float* step_ms);
/* Bytes one sinkr_routed_decode_step call copies host->device (queries +
 * step parameters) and device->host (outputs + routing record). */
sinkr_status sinkr_step_io_bytes(sinkr_engine* e, size_t* h2d, size_t* d2h);
/* The engine's pinned step buffers: queries [B][H_q][D] f32 (inside the
 * pinned input block the step uploads) and outputs [B][H_q][D] f32 (inside the
 * mapped result block the step kernel writes).  A caller that fills *queries
 * and passes it as sinkr_routed_decode_batch's queries (and *outputs as its
 * outputs) skips both host copies; valid for the engine's lifetime, and only
 * between blocking calls. */
sinkr_status sinkr_step_io_buffers(sinkr_engine* e, float** queries, const float** outputs);
/* Enables per-kernel event timing on the async path (costs two event records). */
sinkr_status sinkr_set_timing(sinkr_engine* e, int enabled);
/* Number of SMs / persistent CTAs used by the decode kernel. */
int sinkr_decode_grid(sinkr_engine* e);

/* ---- calibration (calibration.hpp:14-90, calibration.cpp) --
 * Host control logic of the reference restated in C++ (bit-identical: same
 * expression order, no FMA contraction).  Score populations come from the GPU:
 * sinkr_collect_scores runs the routing phase alone (no KV streaming), so a
 * calibration sample costs one probe launch instead of a decode step. */
#define SINKR_MAX_EXCLUDED_LAYERS 32
#define SINKR_MAX_CALIBRATION_POINTS 64
typedef struct sinkr_calibration_point { /* CalibrationPoint (calibration.hpp:14-18) */
    size_t length;
    double tau;
    double skip;
} sinkr_calibration_point;
typedef struct sinkr_profile { /* ThresholdProfile (calibration.hpp:21-34) */
    sinkr_threshold_profile threshold; /* coeffs, length_normalizer, clamp */
    double target_skip;                /* default 0.60 */
    double gamma;                      /* default 0.65 */
    size_t excluded_layers[SINKR_MAX_EXCLUDED_LAYERS];
    size_t num_excluded_layers;        /* default {0, 1} */
    sinkr_calibration_point points[SINKR_MAX_CALIBRATION_POINTS];
    size_t num_points;
} sinkr_profile;
/* ThresholdProfile{} defaults / ThresholdProfile::constant (calibration.cpp:29-35). */
void sinkr_profile_default(sinkr_profile* out);
void sinkr_profile_constant(double tau, sinkr_profile* out);
/* sweep / skip_ratio_at / solve_threshold (calibration.hpp:52-61). */
sinkr_status sinkr_sweep(const double* scores, size_t n, const double* thresholds, size_t m,
                         double* skip_ratios);
sinkr_status sinkr_skip_ratio_at(const double* scores, size_t n, double threshold, double* out);
sinkr_status sinkr_solve_threshold(const double* scores, size_t n, double target_skip,
                                   double* out);
/* fit_cubic (calibration.hpp:68-70): coeffs a,b,c,d + sum of squared residuals. */
sinkr_status sinkr_fit_cubic(const double* x, const double* y, size_t n, double* coeffs,
                             double* residual);
/* calibrate (calibration.hpp:79-83) over populations the caller collected, one
 * per entry of `lengths`: population i is samples offsets[i] .. offsets[i+1]-1
 * of (scores, sample_layers).  As in the reference, each distinct length is
 * used once (its first population), in ascending order. */
sinkr_status sinkr_calibrate(const size_t* lengths, size_t n_lengths, const double* scores,
                             const size_t* sample_layers, const size_t* offsets,
                             double target_skip, double gamma, const size_t* excluded_layers,
                             size_t num_excluded_layers, sinkr_profile* out);
/* save_profile / load_profile (calibration.hpp:85-86): the reference's JSON
 * schema; files interoperate with the reference's nlohmann-based reader. */
sinkr_status sinkr_save_profile(const char* path, const sinkr_profile* profile);
sinkr_status sinkr_load_profile(const char* path, sinkr_profile* out);
/* Routing-phase-only step (the score-collection mode of SPEC.md:396): proxy
 * scores of every head and group of all B sequences for `layer`, with routing
 * decisions under `config` (NULL: none recorded).  Host buffers; blocking.
 *   head_scores [B][H_q], group_scores [B][H_kv], sink [B][H_kv] (may be NULL). */
sinkr_status sinkr_collect_scores(sinkr_engine* e, const float* queries, size_t layer,
                                  const sinkr_routing_config* config, double* head_scores,
                                  double* group_scores, int32_t* sink);
/* The same for n_samples query sets over the same cache layer in one launch
 * (a calibration length's samples): queries [n][B][H_q][D]; head_scores
 * [n][B][H_q], group_scores [n][B][H_kv], sink [n][B][H_kv] (each may be
 * NULL).  Bit-identical to n sinkr_collect_scores calls. */
sinkr_status sinkr_collect_scores_batch(sinkr_engine* e, const float* queries, size_t n_samples,
                                        size_t layer, const sinkr_routing_config* config,
                                        double* head_scores, double* group_scores, int32_t* sink);

/* ---- snapshots (kv_cache.hpp:72-80, tensor.hpp:86-96) -----
 * SNKT tensor files and the snapshot directory layout of the reference
 * (manifest.json + k_l{layer}_h{head}.snkt / v_...).  K/V are f32 in the
 * files; the engine stores bf16 (RNE) and captures anchors from the stored
 * rows.  A snapshot holds one sequence. */
sinkr_status sinkr_write_tensor(const char* path, const uint64_t* dims, size_t ndim,
                                const float* data);
/* Reads the header (dims, ndim <= 64) and, when data != NULL, the payload
 * (capacity in elements). */
sinkr_status sinkr_read_tensor(const char* path, uint64_t* dims, size_t* ndim, float* data,
                               size_t capacity);
uint64_t sinkr_snkt_file_size(const uint64_t* dims, size_t ndim);
sinkr_status sinkr_save_snapshot(sinkr_engine* e, size_t seq, const char* dir);
/* Creates a single-sequence engine on `device` sized by the manifest. */
sinkr_status sinkr_load_snapshot(const char* dir, int device, sinkr_engine** out);
/* Replays a snapshot into sequence `seq` of an existing (empty) engine. */
sinkr_status sinkr_load_snapshot_into(sinkr_engine* e, size_t seq, const char* dir);
/* Device prefill: f32 rows already on the device, converted to bf16 on the
 * device; anchor capture as in sinkr_kv_append. */
sinkr_status sinkr_kv_append_device_f32(sinkr_engine* e, size_t seq, size_t layer,
                                        size_t kv_head, const float* d_k, const float* d_v,
                                        size_t rows);

/* ---- single-group attention (attention.cpp:185-235, attention.hpp:76-85) ---
 * splitk_attention of the r query heads of ONE cached group (seq, layer,
 * kv_head) over all of its rows, on the GPU: out [r][D] f32, counters with
 * kv_floats_loaded = 2 * len * D (the other fields 0).  num_splits is checked
 * like split_ranges (INVALID_ARGUMENT outside [1, len]); the kernel picks its
 * own split.  Runs as a routed step with the route forced, so it replaces the
 * engine's last routing record (sinkr_fetch_step_info). */
sinkr_status sinkr_group_attention(sinkr_engine* e, const float* group_queries, size_t seq,
                                   size_t layer, size_t kv_head, size_t num_splits, float* out,
                                   sinkr_load_counters* counters);

/* ---- span-level attention operators (attention.hpp:14-85) -------------------
 * The reference's free functions over host spans, on the GPU of the calling
 * thread (current device; a per-device context serialised by a mutex; each
 * call blocks until its results are in host memory).  q is [heads][dim] f32,
 * keys / values [len][dim] f32; the logit scale is QueryGroup::over's
 * 1/sqrt(dim) (attention.cpp:33-40).  Arithmetic is the reference's: logits
 * are fp64 sequential dots of exact f32 products (bit-identical), the softmax
 * state m, l, acc is fp64 (SplitPartial, attention.hpp:26-33).  Errors follow
 * check_shapes (attention.cpp:13-23): INVALID_ARGUMENT for heads/dim 0, len 0,
 * block_size 0, num_splits outside [1, len]; head_dim is limited to 8192.
 * Spans are transfer-bound (uploaded per call); the decode hot path streams
 * the engine's cache instead (sinkr_routed_decode_*). */
/* attend_chunk (attention.hpp:55-60, attention.cpp:101-142): the chunk's
 * SplitPartial: m[heads], l[heads], acc[heads][dim] (fp64, caller-owned),
 * *tokens = len (may be NULL).  block_size is validated (> 0); the GPU tiles
 * the chunk itself (state equal up to fp64 rounding). */
sinkr_status sinkr_attend_chunk(const float* q, size_t heads, size_t dim, const float* keys,
                                const float* values, size_t len, size_t block_size, double* m,
                                double* l, double* acc, uint64_t* tokens);
/* attend_chunk over the cached rows [from, to) of (seq, layer, kv_head) of an
 * engine (KvCache::historical + attend_chunk, router.cpp:149-160) with the
 * group's r query heads: OUT_OF_RANGE past the slot's length
 * (kv_cache.cpp:110-113), INVALID_ARGUMENT for an empty range. */
sinkr_status sinkr_attend_chunk_cached(sinkr_engine* e, const float* group_queries, size_t seq,
                                       size_t layer, size_t kv_head, size_t from, size_t to,
                                       size_t block_size, double* m, double* l, double* acc,
                                       uint64_t* tokens);
/* merge_partials (attention.hpp:62-64, attention.cpp:159-183) of n host
 * SplitPartials packed as m[n][heads], l[n][heads], acc[n][heads][dim],
 * tokens[n]: partials with tokens == 0 are skipped; INVALID_ARGUMENT ("merge
 * needs at least one non-empty partial") when all are empty.  out [heads][dim]. */
sinkr_status sinkr_merge_partials(size_t n, const double* m, const double* l, const double* acc,
                                  const uint64_t* tokens, size_t heads, size_t dim, float* out);
/* The same merge as a device kernel on `stream` (cudaStream_t) over device
 * buffers of that layout (d_tokens may be NULL: all live); does not check for
 * the all-empty case (the host entry does). */
sinkr_status sinkr_merge_partials_async(size_t n, const double* d_m, const double* d_l,
                                        const double* d_acc, const uint64_t* d_tokens, size_t heads,
                                        size_t dim, float* d_out, void* stream);
/* splitk_attention (attention.hpp:76-85, attention.cpp:204-235): split_ranges
 * chunks, one attend_chunk partial each, one merge; counters->kv_floats_loaded
 * = 2 * len * dim (other fields 0; may be NULL). */
sinkr_status sinkr_splitk_attention(const float* q, size_t heads, size_t dim, const float* keys,
                                    const float* values, size_t len, size_t num_splits,
                                    size_t block_size, float* out, sinkr_load_counters* counters);
/* online_attention (attention.hpp:48-53, attention.cpp:144-157): acc / l of
 * one attend_chunk over the whole span. */
sinkr_status sinkr_online_attention(const float* q, size_t heads, size_t dim, const float* keys,
                                    const float* values, size_t len, size_t block_size, float* out);
/* dense_attention (attention.hpp:38-42, attention.cpp:42-73): the reference's
 * two-pass exact softmax; computed here as one fp64 online pass, which equals
 * it up to fp64 rounding (the reference's own online-vs-dense bar is 1e-5,
 * SPEC.md:231). */
sinkr_status sinkr_dense_attention(const float* q, size_t heads, size_t dim, const float* keys,
                                   const float* values, size_t len, float* out);

/* ---- analysis (attention.cpp:75-99, analysis.hpp:12-39) ---
 * Full-attention BOS mass on the GPU for oracle sink labels: for every query
 * head, alpha0 = softmax(scale * q.K^T)[0] over the whole cached context of
 * `layer` (one K-only streaming pass).  alpha0: [B][H_q] f64. */
sinkr_status sinkr_attention_bos_mass(sinkr_engine* e, const float* queries, size_t layer,
                                      double* alpha0);
/* attention_weights (attention.cpp:75-99) for one (seq, kv_head) group on the
 * GPU: weights [r][len] f32 over the slot's cached rows. */
sinkr_status sinkr_attention_weights(sinkr_engine* e, const float* queries, size_t seq,
                                     size_t layer, size_t kv_head, float* weights);
/* Device time of the last sinkr_attention_bos_mass / sinkr_attention_weights
 * call's kernels (stream pass, finish, weights), from CUDA events on the
 * engine stream; host staging and copies excluded.  No reference
 * counterpart (measurement hook, SURVEY.md §8 d). */
sinkr_status sinkr_attention_last_kernel_seconds(sinkr_engine* e, double* seconds);
/* oracle labels (analysis.hpp:12-22) from BOS masses: mode 0 = per head
 * (alpha0 > gamma, strict), mode 1 = group mean over `group` consecutive
 * heads.  n_heads % group == 0.  Outputs have n_heads (mode 0) or
 * n_heads / group (mode 1) entries. */
sinkr_status sinkr_oracle_labels(const double* alpha0, size_t n_heads, size_t group,
                                 double gamma, int mode, double* label_alpha0,
                                 uint8_t* is_sink);
/* pr_curve (analysis.hpp:24-39): operating points at every distinct score
 * (positive iff score >= threshold), descending; AUPRC by average-precision
 * step summation.  points: up to n entries of {threshold, precision, recall, f1}. */
sinkr_status sinkr_pr_curve(const double* scores, const uint8_t* labels, size_t n,
                            double* points, size_t* num_points, double* auprc);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* SINKR_CUDA_H_ */
