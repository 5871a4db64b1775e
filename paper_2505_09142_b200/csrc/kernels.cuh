// kernels.cuh -- launch interfaces between the libelis host runtime and its kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace elis {

// EPI_BIAS_RESID16_LN: as RESID_LN with the residual stream held in 16 bits (fp16): the residual
// is read from, and the normalised row written to, the same fp16 [M, N] buffer (no fp32 copy)
enum { EPI_BIAS_BF16 = 0, EPI_BIAS_GELU_BF16 = 1, EPI_BIAS_RESID_F32 = 2, EPI_BIAS_RESID_LN = 3,
       EPI_BIAS_RESID16_LN = 4 };

// Device error bits (sticky; see elis.h).
enum : uint32_t { ERR_TOKEN = 1u, ERR_LENGTH = 2u, ERR_TOTAL = 4u, ERR_PEER_TIMEOUT = 8u, ERR_GX_TIMEOUT = 16u,
                  ERR_ARENA = 32u, ERR_DIMS = 64u };
// device-side shape of a shape-agnostic call: dims = {n, total_tokens}, clamped to the capacity
struct DevDims {
  const int32_t* dims;  // nullptr: the host values
};

// ---- GEMM (gemm.cu)
struct GemmArgs {
  const float* bias;
  const float* resid;   // f32 [M, N] (RESID_F32, RESID_LN; may alias out for RESID_LN)
  void* out;            // bf16 or f32 [M, N]
  uint16_t* outb;       // RESID_LN: bf16 copy of the normalised rows
  const float* gamma;   // RESID_LN
  const float* beta;    // RESID_LN
  float eps;
  int M, N, K;
  int out_head_major;   // bf16 output written as [N/64 planes][rows][64] (attention-friendly qkv)
  // FP8 (E4M3) operands (R20): acc * colscale[n] = A W^T in real units (the weight's
  // per-output-channel scale over the A operand's static power-of-two scale); the GELU output
  // and the LN epilogue's normalised copy are written as E4M3(out_scale * value)
  const float* colscale;
  float out_scale;
  // LN row statistics through global memory instead of a cluster (EPI_BIAS_RESID16_LN, long K):
  // the CTA pairs of one row group need not share a cluster, so the grid spans every SM.
  // gstats [ceil(M/256)][N/256][2][128] float2, gflag [ceil(M/256)][2] arrival counters (zeroed
  // before each launch); nullptr: the cluster / DSMEM exchange
  float2* gstats;
  uint32_t* gflag;
  // 1: M tiles in descending order, so a GEMM first reads the A rows its producer wrote last
  // (still in L2) -- the producer / consumer chain alternates direction
  int m_reverse;
  // sticky device error word (GX exchange timeout -> ERR_GX_TIMEOUT); nullptr: not reported
  uint32_t* err;
  // shape-agnostic launches (elis_predict_remaining_dev): the row count is read from this device
  // int (clamped to M, which is then the capacity the grid was sized for); nullptr: M
  const int32_t* M_dev;
};
struct GemmPlan {
  CUtensorMap tmA;   // A operand, bf16 K-major
  CUtensorMap tmB;   // W operand, bf16 K-major
  CUtensorMap tmR;   // residual f32 [rows, N], 32 x 32 boxes (RESID_F32 / RESID_LN)
  CUtensorMap tmO;   // output: f32 32 x 32 boxes (RESID_F32 / RESID_LN) or bf16 32 x 32 boxes
  CUtensorMap tmOb;  // RESID_LN: bf16 copy of the normalised rows, 32 x 32 boxes
  GemmArgs args;
  int epi;
  int f8;            // operands E4M3 (kind::f8f6f4): A [M, K] / W [N, K] bytes, 128-element K blocks
  int f16;           // operands fp16 (kind::f16, A/B format f16); 16-bit outputs written as fp16
  int bn128 = 0;     // fp16 bias / GELU epilogues: 256 x 128 pair tiles (twice the tiles of a small M)
};
// A copy of an fp16 bias / GELU plan for 256 x 128 pair tiles (W boxes of 64 rows).  Each output
// element is the same sum of the same MMAs in the same K order as with 256 x 256 tiles.
bool gemm_plan_bn128(GemmPlan* g, const void* W);
// bf16 output in head-major planes: out[N/64][rows][64] (the QKV projection feeding attention:
// every (head, 128-token) box of Q, K or V is one contiguous 16 KB block)
bool gemm_plan_set_head_major(GemmPlan* g, void* out, uint64_t rows);
// LN epilogue outputs: outb bf16 [rows, N] (E4M3 bytes when g->f8), gamma/beta f32 [N]
bool gemm_plan_set_ln(GemmPlan* g, uint16_t* outb, const float* gamma, const float* beta, float eps, uint64_t rows);
// FP8 variant of make_gemm_plan: A E4M3 [a_rows, K], W E4M3 [N, K], colscale f32 [N]; the
// EPI_BIAS_GELU_BF16 output (and the LN copy) become E4M3 bytes scaled by out_scale
bool make_gemm_plan_f8(GemmPlan* g, const void* A, uint64_t a_rows, const void* W, const float* colscale,
                       const float* bias, const float* resid, void* out, int M, int N, int K, int epi,
                       float out_scale);
int gemm_block_n(int N);
bool make_tmap_bf16_kmajor(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);
// bf16 [rows, cols] row-major, box {box_cols (<= 64 for SWIZZLE_128B), box_rows}, SWIZZLE_128B
bool make_tmap_bf16_box(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_cols,
                        uint32_t box_rows);
// A: [a_rows >= M, K] bf16 (rows M..a_rows-1 are read but their outputs are not stored)
bool make_gemm_plan(GemmPlan* g, const void* A, uint64_t a_rows, const void* W, const float* bias,
                    const float* resid, void* out, int M, int N, int K, int epi);
cudaError_t launch_gemm(const GemmPlan& g, int num_sms, cudaStream_t st);

// ---- varlen metadata / embedding / LayerNorm (norm.cu)
// One attention work item: q rows [q0, q0 + tile_q) of the request at token offset `start`
// with `len` tokens (the request bounds travel with the item: no dependent cu_seqlens load).
struct __align__(16) AttnWork {
  int32_t start, len, q0, req;
};
// Work-list cost classes: keys a tile attends to, in 128-key blocks (1..4 for L <= 512).
constexpr int kAttnCostClasses = 4;
// lengths[n] -> cu_seqlens[n+1], attention work list with q tiles of tile_q rows in
// descending cost class (longest-processing-time-first: the long tiles start in the first
// wave, the short ones fill the tail), and its size; validates lengths and their sum.
// dims (device {n, total}, optional): a shape-agnostic call -- n / total are read there and the host
// values are the capacity (every launcher below that takes `dims` sizes its grid by the capacity and
// exits beyond the device values)
cudaError_t launch_meta(const int32_t* lengths, int n, int64_t total, int max_position, int32_t* cu_seqlens,
                        AttnWork* work, int32_t* num_work, uint32_t* err, int tile_q, cudaStream_t st,
                        const int32_t* dims = nullptr);
cudaError_t launch_embed_ln(const int32_t* tokens, const int32_t* cu_seqlens, int n, int64_t T, int H,
                            int vocab, int max_position, const uint16_t* word, const uint16_t* pos,
                            const uint16_t* type0, const float* gamma, const float* beta, float eps, float* h32,
                            uint16_t* hb, uint32_t* err, float f8_scale, bool f16, cudaStream_t st,
                            const int32_t* dims = nullptr);
// f8_scale > 0: hb receives E4M3(f8_scale * LN(x)) bytes [T, H] instead of bf16; f16: fp16
// FP8 weights: q [rows, cols] = E4M3(W * 448 / amax_row), scale[row] = amax_row / 448 * post
cudaError_t launch_quant_rows_e4m3(const float* W, int rows, int cols, uint8_t* q, float* scale, float post,
                                   cudaStream_t st);
cudaError_t launch_layernorm(const float* u, const float* gamma, const float* beta, float eps, int64_t rows, int H,
                             float* out32, uint16_t* outb, cudaStream_t st);

// ---- attention (attention.cu)
// head dim 64: tcgen05 kernel with 128-row q tiles; head dim 32: mma.sync, 64-row tiles.
inline int attn_tile_q(int head_dim) { return head_dim == 64 ? 128 : 64; }
// upper bound on the number of q-tiles for T tokens in n requests
inline int64_t attn_max_tiles(int64_t T, int n, int tile_q) { return (T + tile_q - 1) / tile_q + n; }
// total work-list entries to allocate for (T, n)
inline int64_t attn_work_capacity(int64_t T, int n, int tile_q) { return attn_max_tiles(T, n, tile_q); }
// head-major qkv planes [3 * H / 64][rows][64] bf16 -> TMA map with 64-column x 128-row boxes, SWIZZLE_128B
bool make_tmap_qkv(CUtensorMap* m, const void* qkv, uint64_t rows, int H);
// the same planes with 64-row boxes (the 64-key-block engine, the default; ELIS_ATTN_ENGINE=128: the
// 128-key-block engine)
bool make_tmap_qkv64(CUtensorMap* m, const void* qkv, uint64_t rows, int H);
// grid: one CTA per (work item, head), head fastest, so the list's cost order is the launch order
// head dim 64: qkv in head-major planes of plane_rows rows (tm_qkv); head dim 32: qkv [T, 3H].
// ctx_f8_scale > 0 (head dim 64 only): ctx is written as E4M3(ctx_f8_scale * ctx) bytes [T, H];
// f16 (head dim 64 only): qkv and ctx are fp16 instead of bf16
cudaError_t launch_attention(const uint16_t* qkv, const CUtensorMap* tm_qkv, const int32_t* cu_seqlens,
                             const AttnWork* work, const int32_t* num_work, int64_t T, int n, int H, int num_heads,
                             int64_t plane_rows, uint16_t* ctx, float ctx_f8_scale, bool f16, cudaStream_t st,
                             const CUtensorMap* tm_qkv64 = nullptr);

// CLS-only last layer: per (request, head) the attention of the CLS
// query row (row cu[i]) over the request's keys, from the head-major qkv planes; writes the
// compact ctx_c [n, H] (out_kind 0 bf16, 1 fp16, 2 E4M3(ctx_scale x)) and gathers the CLS
// residual rows h32[cu[i]] into hres_c [n, H].  Head dim 64.
// err: the sticky device error word; nothing is read or written once it is set (cu_seqlens may
// then point past the token buffers)
cudaError_t launch_attention_cls(const uint16_t* qkv, const int32_t* cu_seqlens, int n, int H, int num_heads,
                                 int64_t plane_rows, const float* h32, uint16_t* ctx_c, float* hres_c, int out_kind,
                                 float ctx_scale, const uint32_t* err, cudaStream_t st, const int32_t* dims = nullptr);

// ---- pooling + regression head (head.cu)
cudaError_t launch_scatter_rows(const float* src, const int32_t* cu_seqlens, int n, int H, const uint32_t* err,
                                float* dst, cudaStream_t st);
// pooled_lo != nullptr: pooled is written as the 3xTF32 pair (pooled = tf32(p), pooled_lo = p - pooled)
cudaError_t launch_pool(const float* h32, const int32_t* cu_seqlens, int n, int H, int pooling, const uint32_t* err,
                        float* pooled, cudaStream_t st, float* pooled_lo = nullptr, const int32_t* dims = nullptr);
// mean / CLS pooling over the fp16 residual stream (elis_config.residual16)
cudaError_t launch_pool16(const uint16_t* h16, const int32_t* cu_seqlens, int n, int H, int pooling,
                          const uint32_t* err, float* pooled, cudaStream_t st, float* pooled_lo = nullptr,
                          const int32_t* dims = nullptr);
cudaError_t launch_f16_to_f32(const uint16_t* src, float* dst, int64_t count, cudaStream_t st);
// split-K workspace of the exact-fp32 head (part == nullptr: no split)
struct FcWork {
  float* part;        // [S][n][N] partial tiles
  size_t part_cap;    // floats
  uint32_t* ctr;      // [tiles] arrival tickets, zero between launches
  int ctr_cap;
  int num_sms;
};
int fc_splits(int n, int N, int K, int num_sms, size_t part_cap, int ctr_cap);
cudaError_t launch_fc_f32(const float* X, const float* W, const float* b, float* Y, int n, int N, int K, int relu,
                          const FcWork& wk, cudaStream_t st, const int32_t* dims = nullptr);
// 3xTF32 tensor-core head layer (kind::tf32): Y = relu?(X W^T + b) with X = Xh + Xl, W = Wh + Wl
// (hi = tf32 rounding, lo = the fp32 remainder) and Y written as the same kind of pair; 128 x 64
// tiles, K in 4 chunks over a cluster of 4 CTAs reduced in chunk order (batch-invariant).
struct FcTcPlan {
  CUtensorMap ah, al, bh, bl;
  const float* bias;
  float *yh, *yl;
  int N, K;
};
bool fc_tc_supported(int N, int K);
bool make_fc_tc_plan(FcTcPlan* f, const float* Xh, const float* Xl, uint64_t x_rows, const float* Wh, const float* Wl,
                     const float* bias, float* Yh, float* Yl, int N, int K);
cudaError_t launch_fc_tf32(const FcTcPlan& f, int n, int relu, cudaStream_t st, const int32_t* dims = nullptr);
// in place: x <- tf32(x), lo <- x - tf32(x)
cudaError_t launch_split_tf32(float* x, float* lo, size_t count, cudaStream_t st);
// y = a + b (the pair recombined, exact)
cudaError_t launch_add_f32(const float* a, const float* b, float* y, size_t count, cudaStream_t st);
// fp32 [rows, cols] row-major, box {box_cols (<= 32 for SWIZZLE_128B), box_rows}, SWIZZLE_128B
bool make_tmap_f32_box(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_cols,
                       uint32_t box_rows);
// out_pairs (optional): (out_slot[i], y_i) also written to out_pairs[i] (the NCCL exchange's send buffer)
// Zl != nullptr: the input row is Z + Zl (the 3xTF32 layers' pair)
cudaError_t launch_head_out(const float* Z, const float* Zl, const float* w, const float* b, int n, int K,
                            float* out_pred, const int32_t* out_slot, int2* out_pairs, cudaStream_t st,
                            const int32_t* dims = nullptr);
// table[pairs[j].x] = pairs[j].y for every pair with x >= 0 (the NCCL exchange's receive side)
cudaError_t launch_scatter_pairs(const int2* pairs, int count, float* table, cudaStream_t st);

// ---- device-resident token arena of the in-flight table (arena.cu)
// per slot: prompt [kArenaLen] int32, ring of the kArenaLen most recent response tokens, prompt length,
// tokens generated so far; the predictor input keeps the prompt head and the kArenaKeepResp most
// recent response tokens when longer than max_len (R7)
constexpr int kArenaLen = 512, kArenaKeepResp = 254;
cudaError_t launch_arena_offsets(const int32_t* counts, int m, int32_t* offsets, cudaStream_t st);
cudaError_t launch_arena_set(const int32_t* slots, const int32_t* tokens, const int32_t* lengths,
                             const int32_t* offsets, int m, int max_slots, int32_t* prompt, int32_t* plen,
                             int32_t* glen, uint32_t* err, cudaStream_t st);
cudaError_t launch_arena_append(const int32_t* slots, const int32_t* tokens, const int32_t* counts,
                                const int32_t* offsets, int m, int max_slots, int32_t* ring, int32_t* glen,
                                uint32_t* err, cudaStream_t st);
// lengths [n], cu [n + 1], dims = {n, total} (optional), out_tokens [total]
cudaError_t launch_arena_gather(const int32_t* slots, int n, int max_slots, int max_len, const int32_t* prompt,
                                const int32_t* ring, const int32_t* plen, const int32_t* glen, int32_t* lengths,
                                int32_t* cu, int32_t* dims, int32_t* out_tokens, uint32_t* err, cudaStream_t st);

// ---- ISRTF select (select.cu)
constexpr int kMaxBatchCap = 4096;
constexpr int kMaxNodes = 64;  // worker nodes of the per-node Priority Buffers
// starvation control inputs of the key pack (R17); waited == nullptr: no aging
struct Starvation {
  const int32_t* waited;
  int boost_after;
  float boost_amount;
  float margin;
};
struct SelectScratch {
  unsigned long long* keys;   // [n]
  uint32_t* info;             // [8 * kMaxNodes]: per node thr lo/hi, -, -, count, n_elig; [6] nan_count
  unsigned long long* sel_keys;  // [cap] selected keys in order (UINT64_MAX padded)
  int32_t* sel_ids;              // [cap]
};
cudaError_t launch_make_keys(const float* pred, const int32_t* generated, const uint32_t* order,
                             const uint8_t* running, int n, int policy, int allow_preempt, int head_predicts_total,
                             uint32_t order_offset, Starvation sv, unsigned long long* keys, uint32_t* info,
                             cudaStream_t st);
// top-cap over keys[n]; ids (optional) map position -> id; writes out_ids / out_count / scratch
cudaError_t launch_select_topk(const unsigned long long* keys, const int32_t* ids, int n, int cap,
                               int32_t* out_ids, int32_t* out_count, int32_t* out_nan, SelectScratch sc,
                               cudaStream_t st);
// single-node top-cap + preemption flags (out_preempted optional) over a cluster of <= 16 CTAs
cudaError_t launch_select_cluster(const unsigned long long* keys, int n, int cap, int32_t* out_ids, int32_t* out_count,
                                  int32_t* out_nan, const uint8_t* running, uint8_t* out_preempted, SelectScratch sc,
                                  cudaStream_t st);
cudaError_t launch_preempt_flags(const unsigned long long* keys, const uint8_t* running, int n, const uint32_t* info,
                                 uint8_t* out_preempted, cudaStream_t st);
// per-node variants (node == nullptr: one node); out_ids [num_nodes * cap], out_count [num_nodes]
cudaError_t launch_select_topk_nodes(const unsigned long long* keys, const int32_t* ids, const int32_t* node,
                                     const uint8_t* node_ready, int num_nodes, int n, int cap, int32_t* out_ids,
                                     int32_t* out_count, int32_t* out_nan, SelectScratch sc, cudaStream_t st);
cudaError_t launch_preempt_flags_nodes(const unsigned long long* keys, const uint8_t* running, const int32_t* node,
                                       const uint8_t* node_ready, int num_nodes, int n, const uint32_t* info,
                                       uint8_t* out_preempted, cudaStream_t st);
// least-loaded assignment of n_new arriving jobs; load [num_nodes] updated in place
cudaError_t launch_assign_nodes(int32_t* load, int num_nodes, int n_new, int32_t* out_node, cudaStream_t st);
cudaError_t launch_pack_candidates(const SelectScratch sc, int cap, int global_offset, void* send, cudaStream_t st);
cudaError_t launch_unpack_candidates(const void* recv, int total, unsigned long long* keys, int32_t* ids,
                                     cudaStream_t st);

// ---- multi-GPU select over peer memory (select.cu).  Every rank owns one
// symmetric region of peer_region_bytes(): candidate keys u64 [2][kMaxPeers * kMaxBatchCap],
// ids i32 [2][kMaxPeers * kMaxBatchCap], epoch flags u32 [2][kMaxPeers] (index = the epoch's
// parity; rank s's candidates at s * cap).  region[r] is rank r's region as mapped here
// (CUDA IPC, or a plain device pointer when the ranks share the process).
constexpr int kMaxPeers = 8;
struct PeerArgs {
  uint8_t* region[kMaxPeers];
  int rank, world;
  uint32_t* epoch;  // this rank's call counter in device memory (the kernel bumps it): identical on
                    // every rank for the same call, and no host state -- the call can be graph-captured
};
// Bytes of one rank's region when it also carries the prediction exchange of
// elis_predict_remaining_dist for up to max_pairs requests per rank (every rank uses the same).
size_t peer_region_bytes(int max_pairs);
// ---- prediction exchange over peer memory (elis_predict_remaining_dist).
// Behind the select area of each region, at peer_pred_offset(): flags u32 [2][kMaxPeers],
// counts u32 [2][kMaxPeers], (slot, pred) pairs [2][kMaxPeers][max_pairs] (8 B each), indexed by
// the epoch's parity and the SOURCE rank.
__host__ __device__ constexpr size_t peer_pred_offset() {
  return (2 * static_cast<size_t>(kMaxPeers) * kMaxBatchCap * 12 + 2 * kMaxPeers * sizeof(uint32_t) + 255) & ~size_t(255);
}
__host__ __device__ inline uint32_t* peer_pred_flags(uint8_t* region, int par) {
  return reinterpret_cast<uint32_t*>(region + peer_pred_offset()) + par * kMaxPeers;
}
__host__ __device__ inline uint32_t* peer_pred_counts(uint8_t* region, int par) {
  return reinterpret_cast<uint32_t*>(region + peer_pred_offset()) + 2 * kMaxPeers + par * kMaxPeers;
}
__host__ __device__ inline int2* peer_pred_pairs(uint8_t* region, int par, int src, int max_pairs) {
  return reinterpret_cast<int2*>(region + peer_pred_offset() + 4 * kMaxPeers * sizeof(uint32_t)) +
         (static_cast<size_t>(par) * kMaxPeers + src) * max_pairs;
}
struct PredPeerArgs {
  uint8_t* region[kMaxPeers];
  int rank, world, max_pairs;
  uint32_t* epoch;   // this rank's call counter of the prediction exchange (device; bumped by the kernel)
  uint32_t* ticket;  // block arrival counter of the fused head-output kernel (zero between calls)
};
// local top-cap -> stores into every rank's region + release flags -> acquire every rank's
// flag of this epoch -> identical merge -> out_ids (global), out_count, merged threshold in
// info[0..1, 4], preempt flags of this rank's n_local slots.  One launch, one CTA.
// Fused last head layer + prediction exchange over peer memory (elis_predict_remaining_dist):
// y_i = Z_i . w + b, table[slot_i] = y_i locally and (slot_i, y_i) stored into every other rank's
// region over NVLink; the last CTA to finish publishes this rank's count + epoch flag to every
// rank (release, system scope), acquires every rank's flag (bounded; ERR_PEER_TIMEOUT) and
// scatters the other ranks' pairs into the local table.  n may be 0 (the rank still exchanges).
cudaError_t launch_head_out_dist(const float* Z, const float* Zl, const float* w, const float* b, int n, int K,
                                 float* table, const int32_t* slot, PredPeerArgs pa, uint32_t* err, cudaStream_t st);
cudaError_t launch_select_dist_peer(const unsigned long long* keys, const uint32_t* local_info, int n_local, int cap,
                                    int global_offset, PeerArgs pa, const uint8_t* running,
                                    unsigned long long* mkeys, int32_t* mids, int32_t* out_ids, int32_t* out_count,
                                    int32_t* out_nan, uint8_t* out_preempted, uint32_t* info, uint32_t* err,
                                    cudaStream_t st);

}  // namespace elis
