/*
 * elis.h -- C ABI of the B200-native ISRTF re-predict + select hot path
 * (ELIS, arXiv 2505.09142).  sm_100a only.  No CUDA or torch types in the
 * signatures: device arrays are plain pointers, streams are `void*`
 * (a cudaStream_t; NULL = the legacy default stream).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section in brackets).
 *
 * What the library computes:
 *   Algorithm 1 (alg:scheduler_flow) lines 10-19: every job in the
 *   Job Pool gets a priority from the predictor -- Predictor.init(job) on the
 *   prompt, Predictor.iter(job) on "the prompt attached with the answer"
 *    -- and the batcher forms "a batched prompt ... starting
 *   with the prompt with the highest priority".  The predictor is a BGE
 *   (BERT) encoder with mean pooling and eight FC layers, ReLU, hidden
 *   1024 (P:359 [Sec. 4.2]); the priority is predicted remaining tokens
 *   (Iterative SRTF, P:22, P:172-174 [Sec. 3.3]).
 *
 * Conventions for every call:
 *   - Host-validated argument errors return immediately; nothing is enqueued.
 *   - ELIS_OK means "enqueued on `stream`"; outputs are valid once the stream
 *     reaches that point.  No call synchronises the host except
 *     elis_sync_status, elis_iteration_host and elis_profile_read.
 *   - Errors detected on the device (a token id >= vocab, a length outside
 *     [1, max_position], sum(lengths) != total_tokens) are STICKY: they set a
 *     device error word that elis_sync_status returns (and clears).
 *   - The caller owns every array it passes; inputs must not alias outputs.
 *     The predictor owns its device weights, workspaces and NCCL communicator.
 *   - One predictor per device; calls on one predictor must be serialised by
 *     the caller.  Several predictors may coexist.
 *   - Determinism: identical inputs give bit-identical out_pred / out_ids.
 */
#ifndef ELIS_H_
#define ELIS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ELIS_ABI_VERSION 5

typedef enum {
  ELIS_OK = 0,
  ELIS_ERR_INVALID_ARG = 1,        /* bad pointer / size / enum value                  */
  ELIS_ERR_CONFIG = 2,             /* elis_config inconsistent or unsupported shape   */
  ELIS_ERR_UNSUPPORTED_DEVICE = 3, /* not compute capability 10.0 (B200, sm_100a)     */
  ELIS_ERR_OOM = 4,                /* device allocation failed                        */
  ELIS_ERR_CUDA = 5,               /* a CUDA runtime/driver call failed               */
  ELIS_ERR_NCCL = 6,               /* an NCCL call failed                             */
  ELIS_ERR_DEVICE_INPUT = 7,       /* sticky device-detected input error (see above)  */
  ELIS_ERR_PEER_TIMEOUT = 8        /* sticky: a peer-memory select waited > 10 s for a rank */
} elis_status;

typedef enum { ELIS_POOL_MEAN = 0, ELIS_POOL_CLS = 1 } elis_pooling;   /* P:359 / P:138 */
typedef enum { ELIS_POLICY_ISRTF = 0, ELIS_POLICY_FCFS = 1 } elis_policy; /* P:22 / P:463 */
/* Operand precision of the encoder GEMMs (the paper never states one, R12).
 * AUTO (0, the zero-initialised default): FP16 for head-dim-64 encoders whose hidden and
 *       intermediate sizes are multiples of 256 (BGE-base / large), BF16 otherwise (the tiny
 *       d = 32 encoder) -- the configuration that meets the north_star parity bars (predictions
 *       1e-2 relative, hidden states 2e-2 absolute) on every tested workload (R21).
 * BF16: bf16 operands, fp32 accumulate.  Measured vs the fp64 oracle: hidden <= 0.019 absolute,
 *       predictions <= 6% relative (5.8% on one request predicted at ~22 tokens, 1.3 tokens
 *       absolute; R21) -- it does NOT meet the 1e-2 prediction bar everywhere.
 * FP8:  E4M3 weights (per-output-channel scale) and E4M3 activations (static power-of-two
 *       scales) on tcgen05 kind::f8f6f4, fp32 accumulate; attention stays bf16, the residual
 *       stream / LayerNorm / head stay fp32 (R20).
 *       Requires head dim 64 and hidden, intermediate multiples of 256 (BGE-base / large).
 * FP16: fp16 weights, GEMM/attention operands (Q, K, V, P) and 16-bit activations, fp32
 *       accumulate; 3 more mantissa bits than bf16, same speed.
 *       Same shape requirements as FP8. */
typedef enum { ELIS_PREC_AUTO = 0, ELIS_PREC_FP8 = 1, ELIS_PREC_FP16 = 2, ELIS_PREC_BF16 = 3 } elis_precision;
/* Residual stream between encoder layers (SURVEY.md Sec. 8b `residual_fp32`, R12, R23).
 * AUTO (0): FP16 when the resolved precision is FP16 and cls_last_layer = 0, else FP32.
 * FP16: the stream is the fp16 copy the GEMMs already read; every LayerNorm is still formed and
 *       normalised in fp32 (LN statistics fp32), only the stored stream is rounded.
 * FP32: an fp32 stream beside the 16-bit GEMM operand copy. */
typedef enum { ELIS_RESID_AUTO = 0, ELIS_RESID_FP16 = 1, ELIS_RESID_FP32 = 2 } elis_residual;

/* Encoder + head shape.  BGE-base = {30522, 512, 2, 12, 768, 12, 3072}
 * (P:121, P:123 [Sec. 3.1]); head = 8 layers, hidden 1024. */
typedef struct {
  int32_t abi_version;        /* must equal ELIS_ABI_VERSION                                  */
  int32_t vocab_size;         /* 30522                                                        */
  int32_t max_position;       /* 512 (max tokens per request)                                 */
  int32_t type_vocab_size;    /* 2 (token type 0 is used everywhere)                          */
  int32_t num_layers;         /* 12 base / 24 large / 2 tiny                                  */
  int32_t hidden;             /* H: 768 / 1024 / 128; multiple of 128                         */
  int32_t num_heads;          /* H / num_heads must be 32 or 64                               */
  int32_t intermediate;       /* F: 4H; multiple of 128                                       */
  float   ln_eps;             /* 1e-12                                                        */
  int32_t pooling;            /* elis_pooling; default MEAN (reading R2)            */
  int32_t head_layers;        /* 8                                              */
  int32_t head_hidden;        /* 1024                                                 */
  int32_t head_predicts_total;/* 0: the head emits remaining tokens (R4); 1: total*/
  int32_t max_tokens;         /* workspace capacity: max sum(lengths) per predict call        */
  int32_t max_requests;       /* workspace capacity: max n per predict / select call          */
  int32_t device;             /* CUDA device ordinal                                          */
  int32_t precision;          /* elis_precision; 0 = AUTO (see above)                         */
  int32_t cls_last_layer;     /* 1 with pooling = CLS: the last layer computes only each      */
                              /* request's CLS row (exact: nothing else reaches the head;     */
                              /* SURVEY.md Sec. 8f row f4(ii)); needs head dim 64             */
  int32_t residual_stream;    /* elis_residual; 0 = AUTO (see above).  FP16 needs precision   */
                              /* FP16 and cls_last_layer = 0                                   */
} elis_config;

typedef struct elis_predictor elis_predictor;

int32_t elis_abi_version(void);

/* Number of fp32 values the weight blob must hold for `cfg` (0 if cfg is invalid).
 * Canonical order: HF BertModel state_dict (no pooler) --
 *   embeddings.{word,position,token_type}_embeddings.weight, embeddings.LayerNorm.{weight,bias},
 *   then per layer l: attention.self.{query,key,value}.{weight,bias},
 *   attention.output.dense.{weight,bias}, attention.output.LayerNorm.{weight,bias},
 *   intermediate.dense.{weight,bias}, output.dense.{weight,bias}, output.LayerNorm.{weight,bias}
 * -- then head fc1..fc{head_layers} (weight [out, in] row-major, bias [out]).
 * Linear weights are [out, in] row-major (nn.Linear).  Encoder matrices are
 * converted to bf16 (round to nearest even) on upload; LN parameters, biases
 * and the whole head stay fp32. */
size_t elis_weight_count(const elis_config* cfg);

/* Validate cfg, check the device is CC 10.0, upload + repack the weights
 * (fused Wqkv [3H, H] bf16; head fp32), allocate workspaces for
 * cfg->max_tokens / cfg->max_requests.  `weights` is a HOST array of
 * `count` floats; it is copied (the caller may free it on return).
 * Errors: INVALID_ARG (NULL / count mismatch), CONFIG, UNSUPPORTED_DEVICE, OOM, CUDA. */
elis_status elis_predictor_create(const elis_config* cfg, const float* weights, size_t count,
                                  elis_predictor** out);
void elis_predictor_destroy(elis_predictor* p);

/* Predictor.init / Predictor.iter for n requests at once (Alg. 1 lines 12/14).
 *   tokens       DEVICE int32 [total_tokens], requests packed back to back; request i
 *                starts at exclusive_scan(lengths)[i]; [CLS] first; token type 0.
 *   lengths      DEVICE int32 [n], each in [1, max_position].
 *   n            0 <= n <= max_requests (n = 0 is a no-op).
 *   total_tokens == sum(lengths) <= max_tokens (checked on device: sticky error).
 *   out_pred     DEVICE fp32: the head output y_i (remaining tokens, NOT clamped).
 *   out_slot     optional DEVICE int32 [n]: if non-NULL, y_i is written to
 *                out_pred[out_slot[i]] (scatter into an in-flight table), else out_pred[i].
 * Per request: embedding + LN, num_layers post-LN BERT blocks over the request's own
 * tokens (bidirectional, no cross-request attention), mean/CLS pooling, 8-FC head. */
elis_status elis_predict_remaining(elis_predictor* p, const int32_t* tokens, const int32_t* lengths,
                                   int32_t n, int64_t total_tokens, float* out_pred,
                                   const int32_t* out_slot, void* stream);

/* Starvation control ("policies that can adjust the frequency of preemption and
 * prevent starvation"; SPEC S:233, S:264 aging; reading R17).  ISRTF keys only, fp32,
 * applied to remaining = max(0, .) inputs before the floor at 0:
 *   remaining -= boost_amount * floor(windows_waited[i] / boost_after)   if windows_waited[i] > 0
 *   remaining -= preempt_margin                                           if running[i]
 * so a job waiting in its buffer gains priority with every batch it is passed over for, and a
 * waiting job displaces a running one only when predicted shorter by more than the margin. */
typedef struct {
  const int32_t* windows_waited; /* DEVICE [n] batches the slot's node formed without it since it  */
                                 /* last ran or arrived; NULL => no aging                          */
  int32_t boost_after;           /* >= 1                                                           */
  float boost_amount;            /* tokens per boost_after windows waited, >= 0                     */
  float preempt_margin;          /* tokens, >= 0                                                    */
} elis_starvation;

/* Preemption controls and tie-break inputs (P:345-348 [Backend Worker]). */
typedef struct {
  int32_t policy;            /* ELIS_POLICY_ISRTF or ELIS_POLICY_FCFS                               */
  int32_t allow_preempt;     /* 1: running jobs may be displaced; 0: running jobs keep their slots   */
  const uint32_t* order;     /* DEVICE [n] unique rank of (arrival, id); NULL => slot index          */
  const uint8_t* running;    /* DEVICE [n] 1 if in the batch that just ran; NULL => none running     */
  uint8_t* out_preempted;    /* DEVICE [n] running && !selected; NULL => not written                 */
  int32_t* out_count;        /* DEVICE [1] number of ids written; NULL => not written                */
  int32_t* out_nan_count;    /* DEVICE [1] NaN predictions seen (keyed as +inf); NULL => not written */
  const elis_starvation* starvation; /* HOST struct; NULL => no aging, no margin                    */
} elis_preempt;

/* Batcher.batch (Alg. 1 line 19): the batch_cap eligible slots with the
 * smallest key (class, remaining, order), ascending.
 *   remaining = pred (or pred - generated if cfg.head_predicts_total), fp32;
 *   key = max(0, remaining), -0 -> +0, NaN -> +inf (lowest priority, counted);
 *   FCFS: remaining ignored (arrival rank alone);
 *   class = 0 for all slots if allow_preempt, else 0 for running slots and 1 for the rest.
 *   pred       DEVICE fp32 [n]; generated DEVICE int32 [n] (< 0 marks an empty slot, never selected).
 *   batch_cap  1 <= batch_cap <= 4096; n <= max(max_requests, 65536).
 *   out_ids    DEVICE int32 [batch_cap], slot indices in priority order, -1 padded. */
elis_status elis_isrtf_select(elis_predictor* p, const float* pred, const int32_t* generated,
                              int32_t n, int32_t batch_cap, const elis_preempt* preempt,
                              int32_t* out_ids, void* stream);

/* ---- per-node Priority Buffers ---------------------------------
 * Load Balancer.get_min_load (Alg. 1 line 3): each of n_new jobs, in arrival order,
 * goes to the node with the fewest assigned jobs (ties -> lowest node id), which then counts it.
 *   node_load  DEVICE int32 [num_nodes], updated in place (the caller decrements a node's count
 *              when one of its jobs finishes); 1 <= num_nodes <= 64.
 *   out_node   DEVICE int32 [n_new]. */
elis_status elis_assign_nodes(elis_predictor* p, int32_t* node_load, int32_t num_nodes, int32_t n_new,
                              int32_t* out_node, void* stream);
/* Batcher.batch per node ("multiple priority queues, where each queue stores jobs
 * assigned to a specific node"; a batch is formed when a node becomes available): for every
 * ready node w, elis_isrtf_select restricted to the slots with node[i] == w, in one launch.
 *   node        DEVICE int32 [n]; slots with a node outside [0, num_nodes) are never selected.
 *   node_ready  DEVICE uint8 [num_nodes] or NULL (all ready); a node that is not ready gets
 *               count 0 and its running slots are not flagged (they are mid-window).
 *   out_ids     DEVICE int32 [num_nodes * batch_cap]: node w's batch at w * batch_cap, -1 padded.
 *   out_counts  DEVICE int32 [num_nodes].
 *   preempt     as for elis_isrtf_select (out_count unused; out_preempted per slot, own node). */
elis_status elis_isrtf_select_nodes(elis_predictor* p, const float* pred, const int32_t* generated,
                                    const int32_t* node, const uint8_t* node_ready, int32_t n,
                                    int32_t num_nodes, int32_t batch_cap, const elis_preempt* preempt,
                                    int32_t* out_ids, int32_t* out_counts, void* stream);

/* ---- multi-GPU (BASELINE.json configs[4]) ------------------------------------------------
 * One process per GPU.  The caller creates a 128-byte ncclUniqueId on rank 0
 * (elis_nccl_unique_id) and broadcasts it (e.g. through torch.distributed). */
elis_status elis_nccl_unique_id(void* out_id128);
elis_status elis_dist_attach(elis_predictor* p, int32_t rank, int32_t world, const void* nccl_unique_id);
/* Global ISRTF select over the union of every rank's slots.  Rank r owns global slots
 * [global_offset, global_offset + n_local).  Each rank keys its slots, takes its local
 * top-cap candidates, all-gathers them over NCCL (NVLink) and merges: the global top-cap
 * is contained in the union of the local top-caps because keys are unique.
 *   preempt->order must hold GLOBAL ranks (NULL => global slot index);
 *   out_ids: DEVICE [batch_cap] GLOBAL slot indices, identical on every rank;
 *   out_preempted (optional): this rank's n_local slots. */
elis_status elis_isrtf_select_dist(elis_predictor* p, const float* pred, const int32_t* generated,
                                   int32_t n_local, int32_t global_offset, int32_t batch_cap,
                                   const elis_preempt* preempt, int32_t* out_ids, void* stream);

/* ---- multi-GPU over peer memory (NVLink 5 / NVSwitch loads and stores, no NCCL) ----------
 * The same global select as elis_isrtf_select_dist (SURVEY.md Sec. 8a row a13, 8e "B200-native
 * stretch"), with the exchange done by ONE kernel: each rank's local top-cap candidates
 * (u64 key + global id) are stored directly into every rank's symmetric receive region through
 * CUDA-IPC-mapped pointers and published by an epoch flag (st.release.sys); each rank then
 * acquires all `world` flags and runs the identical merge.  Results are bit-identical to the
 * NCCL transport.  Setup, once per predictor:
 *   1. elis_peer_export(p, rank, world, handle): allocates (once) and clears this rank's region
 *      (~0.8 MB) and writes its 64-byte cudaIpcMemHandle_t to `handle` (HOST memory);
 *   2. the caller all-gathers the handles in rank order (e.g. torch.distributed);
 *   3. elis_peer_attach(p, handles): maps every other rank's region (HOST array world x 64 B).
 * From then on elis_isrtf_select_dist uses this transport.  Every rank must make the same
 * sequence of elis_isrtf_select_dist calls (like a collective) with the same batch_cap; n_local
 * may differ per rank; world <= 8.  A rank that never
 * arrives makes the waiting ranks give up after 10 s with the sticky ELIS_ERR_PEER_TIMEOUT
 * (outputs: count 0, ids -1).  The call counter lives in device memory (bumped by the kernel), so
 * a sequence of calls may be captured in a CUDA graph and replayed on every rank.
 * elis_peer_attach_local wires predictors that live in ONE process
 * (peers[r] = rank r; devices may repeat -- tests -- or differ, with peer access enabled). */
elis_status elis_peer_export(elis_predictor* p, int32_t rank, int32_t world, void* out_handle64);
elis_status elis_peer_attach(elis_predictor* p, const void* handles);
elis_status elis_peer_attach_local(elis_predictor* const* peers, int32_t world);

/* ---- end-to-end convenience (HOST buffers) ----------------------------------------------
 * One scheduling iteration from host memory: H2D copy of tokens/lengths/generated
 * (+ order/running if given), predict, select, D2H copy of out_ids/out_count (and
 * out_pred if non-NULL).  Synchronises `stream` before returning.  Pinned host memory
 * gives asynchronous copies.  global_offset < 0: single-GPU elis_isrtf_select;
 * global_offset >= 0: elis_isrtf_select_dist over the attached communicator (this
 * rank's slots start at global_offset; out_ids are global). */
elis_status elis_iteration_host(elis_predictor* p, const int32_t* h_tokens, const int32_t* h_lengths,
                                int32_t n, int64_t total_tokens, const int32_t* h_generated,
                                const uint32_t* h_order, const uint8_t* h_running, int32_t policy,
                                int32_t allow_preempt, int32_t batch_cap, int32_t global_offset,
                                int32_t* h_out_ids, int32_t* h_out_count, float* h_out_pred, void* stream);

/* ---- in-flight table (BASELINE.json configs[4]) ------------
 * The Priority Buffer keeps one cached prediction per in-flight slot; each scheduling iteration
 * re-predicts only the due set (jobs returning from a window, Alg. 1 lines 10-18) and
 * the batch is selected over every cached key (line 19).
 *
 * elis_predict_remaining_dist: one rank's share of the due set, with the result visible on EVERY
 * rank ("each rank encodes its slice, an NCCL all-gather over NVLink collects the predictions",
 * BASELINE.json north_star).  A collective: every attached rank calls it once per iteration, in
 * the same order (n may differ, and may be 0).
 *   tokens, lengths, n, total_tokens  as elis_predict_remaining (this rank's requests).
 *   table     DEVICE fp32 [n_table], one replica per rank (identical on every rank afterwards).
 *   out_slot  DEVICE int32 [n]: table slot of each of this rank's requests (required; slots of
 *             different ranks must not collide).
 * After the stream reaches the end of the call: table[out_slot_r[i]] = y_{r,i} on every rank for
 * every rank r's requests; other entries unchanged.  Transport = the last attach call: peer memory
 * (elis_peer_attach*: ONE fused kernel computes the last head layer, stores (slot, y) into every
 * rank's region over NVLink, publishes an epoch flag and scatters the others' pairs; a rank that
 * never arrives -> sticky ELIS_ERR_PEER_TIMEOUT after 10 s, its pairs missing) or NCCL
 * (elis_dist_attach: (slot, y) pairs padded to max_requests -> ncclAllGather -> scatter).  Every
 * rank must use the same cfg.max_requests.  Errors: INVALID_ARG (not attached, NULL arrays, n or
 * total_tokens out of range), CUDA, NCCL. */
elis_status elis_predict_remaining_dist(elis_predictor* p, const int32_t* tokens, const int32_t* lengths,
                                        int32_t n, int64_t total_tokens, float* table, const int32_t* out_slot,
                                        void* stream);

/* Shape-agnostic elis_predict_remaining (SURVEY.md Sec. 3.2 "one CUDA graph for a variable due
 * set"): n and total_tokens are read on the device from dims = {n, total_tokens} (DEVICE int32[2],
 * e.g. written by elis_arena_gather), so the call can be captured into a CUDA graph once and
 * replayed for every iteration whatever the due set's shape.  Every kernel is launched for the
 * predictor's capacity (max_requests, max_tokens) and exits beyond the device values; results are
 * bit-identical to elis_predict_remaining on the same inputs.  n = 0 predicts nothing.  Device-
 * detected: n outside [0, max_requests] or total_tokens > max_tokens (sticky, bit 64), and the
 * usual length / token / sum checks.  Local head output only (no _dist). */
elis_status elis_predict_remaining_dev(elis_predictor* p, const int32_t* tokens, const int32_t* lengths,
                                       const int32_t* dims, float* out_pred, const int32_t* out_slot, void* stream);

/* One scheduling iteration over an in-flight table from HOST buffers (the end-to-end call):
 * H2D copy of this rank's due tokens / lengths / table slots, elis_predict_remaining (or _dist
 * when a transport is attached) into `table` through the slots, elis_isrtf_select over the whole
 * table (n_table slots, DEVICE `table` / `generated`; preempt as for elis_isrtf_select, device
 * arrays, may be NULL = ISRTF with preemption), D2H copy of out_ids [batch_cap] and the count.
 * Synchronises `stream` before returning.  With a transport attached every rank gets the same
 * ids (the table is identical everywhere). */
elis_status elis_iteration_table_host(elis_predictor* p, const int32_t* h_tokens, const int32_t* h_lengths,
                                      int32_t n, int64_t total_tokens, const int32_t* h_slots, float* table,
                                      const int32_t* generated, int32_t n_table, int32_t batch_cap,
                                      const elis_preempt* preempt, int32_t* h_out_ids, int32_t* h_out_count,
                                      void* stream);

/* Cost-balanced split of n requests (in index order) over `world` ranks:
 * contiguous slices whose boundaries sit at the world-quantiles of the prefix sum of
 *   c(L) = num_layers (2 (4 H^2 + 2 H F) L + 4 H L^2)      (the encoder's FLOPs per request;
 *                                                            BGE-base: 169.87e6 L + 36,864 L^2)
 * out_bounds[r] (r = 1..world-1) = the index i >= out_bounds[r-1] whose prefix cost is closest to
 * r/world of the total (ties -> smaller i); out_bounds[0] = 0, out_bounds[world] = n.  Rank r takes
 * [out_bounds[r], out_bounds[r+1]).  HOST arrays (lengths [n], out_bounds [world + 1]); pure host
 * arithmetic in fp64, no device needed. */
elis_status elis_cost_split(const int32_t* lengths, int32_t n, int32_t world, int32_t num_layers, int32_t hidden,
                            int32_t intermediate, int32_t* out_bounds);

/* ---- device-resident token arena of the in-flight table ---------
 * PAPER.md Sec. 3.4 sends each prompt to the scheduler once and then only the fixed-window partial
 * outputs; the predictor re-encodes "the prompt attached with the answer"
 * whenever the job returns to the Job Pool (Alg. 1 lines 10-18).  The arena keeps, in
 * device memory, every slot's prompt ([CLS] ... [SEP], 1..512 tokens) and its 512 most recent
 * response tokens; per iteration the caller uploads only new prompts and the tokens each
 * returning job generated, and gathers the due set's predictor inputs on the device:
 *   prompt ++ response                      if |prompt| + generated <= max_len,
 *   prompt[:max_len - k] ++ last k response otherwise, k = min(generated, 254)   (R7).
 * All arrays are DEVICE pointers, work is enqueued on `stream`.  Device-detected errors (slot
 * outside [0, max_slots), a prompt length outside [1, 512], a negative count, gathering a slot with
 * no prompt) are sticky, reported by elis_arena_sync_status. */
typedef struct elis_arena elis_arena;
elis_status elis_arena_create(int32_t max_slots, int32_t device, elis_arena** out);
void elis_arena_destroy(elis_arena* a);
/* slots [m]: slot k gets prompt tokens[offset_k .. offset_k + lengths[k]) (packed back to back in
 * slot order) and its generated count reset to 0. */
elis_status elis_arena_set_prompts(elis_arena* a, const int32_t* slots, const int32_t* tokens,
                                   const int32_t* lengths, int32_t m, void* stream);
/* slots [m]: slot k appends counts[k] >= 0 generated tokens (packed back to back in slot order). */
elis_status elis_arena_append(elis_arena* a, const int32_t* slots, const int32_t* tokens, const int32_t* counts,
                              int32_t m, void* stream);
/* Predictor inputs of the n due slots: out_lengths [n], out_tokens [sum] (packed, the layout
 * elis_predict_remaining takes), out_dims [2] = {n, sum} (optional; e.g. for the total on the host
 * or a graph).  out_tokens must hold n * max_len tokens.  max_len in [2, 512]. */
elis_status elis_arena_gather(elis_arena* a, const int32_t* slots, int32_t n, int32_t max_len, int32_t* out_tokens,
                              int32_t* out_lengths, int32_t* out_dims, void* stream);
/* Synchronise `stream`, return (and clear) the arena's sticky error: ELIS_ERR_DEVICE_INPUT if set. */
elis_status elis_arena_sync_status(elis_arena* a, void* stream);

/* Synchronise the stream of the last call and return (and clear) the sticky device
 * error word: ELIS_ERR_DEVICE_INPUT if set, else ELIS_OK / ELIS_ERR_CUDA. */
elis_status elis_sync_status(elis_predictor* p);
/* Raw device error bits of the last elis_sync_status (1: token id out of range,
 * 2: length outside [1, max_position], 4: sum(lengths) != total_tokens, 8: peer timeout,
 * 16: a global-memory LayerNorm statistics exchange timed out -- ELIS_GEMM_GX / elis_op_gemm_ln16,
 * 64: a shape-agnostic call's device dims exceed the capacity -- elis_predict_remaining_dev). */
uint32_t elis_last_device_error_bits(elis_predictor* p);
const char* elis_status_string(elis_status s);
const char* elis_last_error(void);                 /* thread-local detail of the last failure */

/* ---- instrumentation (bench / tests) ------------------------------------------------------ */
/* Copy the final-layer hidden states [total_tokens, H] of the last predict call as fp32 (DEVICE
 * dst, `count` floats >= total_tokens * H): the fp32 residual stream, or the fp16 stream widened
 * when residual16 is set -- parity tests compare them with the oracle. */
elis_status elis_get_hidden(elis_predictor* p, float* dst, int64_t count, void* stream);
/* Number of kernels this predictor has launched so far. */
uint64_t elis_launch_count(elis_predictor* p);
/* Per-kernel-class CUDA-event timing on the launching stream.  enable=1 starts recording
 * (resetting the totals); elis_profile_read synchronises, then fills up to `cap` entries:
 * names[i] (static strings), total_ms[i], launches[i]; returns the number of classes. */
elis_status elis_profile_enable(elis_predictor* p, int32_t enable);
int32_t elis_profile_read(elis_predictor* p, const char** names, double* total_ms, int64_t* launches,
                          int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* ELIS_H_ */
