// attention.cu -- fused varlen bidirectional multi-head attention.
//
// For every request i and head h (BERT self-attention,
// P:42 "process tokens in parallel"):
//     ctx_h = softmax(Q_h K_h^T / sqrt(d)) V_h   over the request's own L_i tokens,
// no causal mask, no cross-request attention, no padding: the work list holds one
// 64-row query tile per (request, q0) so ragged lengths cost at most one partial tile.
//
// v1 engine: flash-style online softmax (fp32 statistics, exp2 with the log2(e)/sqrt(d)
// scale folded in), Q/K/V staged in shared memory with cp.async double buffering,
// products on mma.sync m16n8k16 bf16 -> fp32 (P rounded to bf16 for the PV product).
// The whole K/V of one (request, head) is <= 512 x 64 x 2 x 2 B = 128 KB.

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace elis {

#ifdef ELIS_ATTN_TRACE
// Diagnostic build only (python -m paper_2505_09142_b200.build --variant=trace -DELIS_ATTN_TRACE):
// thread 0 of every tcgen05 attention CTA stamps %globaltimer at its phase boundaries.
constexpr size_t kTraceCap = 1 << 16;
__device__ unsigned long long g_attn_trace[kTraceCap * 8];
static void* g_attn_trace_ptr() {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_attn_trace);
  return p;
}
#define ATTN_TRACE(slot, val)                                                          \
  do {                                                                                 \
    if (threadIdx.x == 0) {                                                            \
      const size_t id_ = blockIdx.x;      \
      if (id_ < kTraceCap) g_attn_trace[id_ * 8 + (slot)] = (val);                     \
    }                                                                                  \
  } while (0)
__device__ __forceinline__ unsigned long long attn_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned attn_smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#else
#define ATTN_TRACE(slot, val) \
  do {                        \
  } while (0)
#endif

#ifdef ELIS_ATTN_TRACE
// Diagnostic build only (python -m paper_2505_09142_b200.build --variant=atrace -DELIS_ATTN_TRACE):
// thread 0 of every 64-key-engine CTA stamps %globaltimer (event code in the low 8 bits) at its
// phase boundaries; scripts/attn_trace.py decodes them.
constexpr int kTrCtas = 1 << 16, kTrEv = 48;
__device__ unsigned long long g_attn64_trace[static_cast<size_t>(kTrCtas) * kTrEv];
__device__ unsigned g_attn64_trace_n[kTrCtas];
extern "C" int elis_debug_attn64_trace(unsigned long long* host, unsigned* counts) {
  cudaError_t e = cudaMemcpyFromSymbol(host, g_attn64_trace, sizeof(g_attn64_trace));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(counts, g_attn64_trace_n, sizeof(g_attn64_trace_n));
  return static_cast<int>(e);
}
#define ATR(code)                                                                                  \
  do {                                                                                             \
    if (threadIdx.x == 0 && blockIdx.x < kTrCtas) {                                                \
      unsigned long long t_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
      if (tr_k < kTrEv) g_attn64_trace[static_cast<size_t>(blockIdx.x) * kTrEv + tr_k] = (t_ << 8) | (code); \
      ++tr_k;                                                                                      \
    }                                                                                              \
  } while (0)
#define ATR_DONE() do { if (threadIdx.x == 0 && blockIdx.x < kTrCtas) g_attn64_trace_n[blockIdx.x] = tr_k; } while (0)
#else
#define ATR(code) do { } while (0)
#define ATR_DONE() do { } while (0)
#endif

namespace {

constexpr int BQ = 64;          // 64 query rows per CTA (4 warps x 16)
constexpr int BKV = 64;         // keys per block

ELIS_DEV void ldmatrix_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
ELIS_DEV void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
ELIS_DEV void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Load `rows` x D bf16 rows (global row stride `ld` elements) into padded smem rows of LDS.
template <int D, int LDS>
ELIS_DEV void load_tile(uint16_t* s, const uint16_t* g, int ld, int row0, int L) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
  for (int c = threadIdx.x; c < 64 * CH; c += blockDim.x) {
    const int r = c / CH, k = c % CH;
    const bool valid = (row0 + r) < L;
    const uint16_t* src = valid ? g + static_cast<size_t>(row0 + r) * ld + k * 8 : g;
    cp_async16(s + r * LDS + k * 8, src, valid);
  }
}

template <int D>
__global__ void __launch_bounds__(128) k_attention(const uint16_t* __restrict__ qkv, const int32_t* __restrict__ cu,
                                                   const AttnWork* __restrict__ work,
                                                   const int32_t* __restrict__ num_work, int H, int nh,
                                                   uint16_t* __restrict__ ctx, float scale_log2) {
  constexpr int LDS = D + 8;  // padded row: conflict-free ldmatrix
  __shared__ __align__(16) uint16_t sQ[BQ * LDS];
  __shared__ __align__(16) uint16_t sK[2][BKV * LDS];
  __shared__ __align__(16) uint16_t sV[2][BKV * LDS];

  const int item = static_cast<int>(blockIdx.x) / nh, h = static_cast<int>(blockIdx.x) % nh;
  if (item >= __ldg(num_work)) return;
  const AttnWork w = work[item];
  const int start = w.start, L = w.len, q0 = w.q0;
  const int ld = 3 * H;
  const uint16_t* gQ = qkv + static_cast<size_t>(start) * ld + h * D;
  const uint16_t* gK = gQ + H;
  const uint16_t* gV = gQ + 2 * H;

  const int warp = warp_id(), lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int nkv = (L + BKV - 1) / BKV;

  // Q tile rows [q0, q0 + 64) (relative to the request), then K/V block 0
  load_tile<D, LDS>(sQ, gQ, ld, q0, L);
  load_tile<D, LDS>(sK[0], gK, ld, 0, L);
  load_tile<D, LDS>(sV[0], gV, ld, 0, L);
  cp_async_commit();

  uint32_t qf[D / 16][4];
  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int j = 0; j < nkv; ++j) {
    const int buf = j & 1;
    if (j + 1 < nkv) {
      load_tile<D, LDS>(sK[buf ^ 1], gK, ld, (j + 1) * BKV, L);
      load_tile<D, LDS>(sV[buf ^ 1], gV, ld, (j + 1) * BKV, L);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (j == 0) {
#pragma unroll
      for (int kc = 0; kc < D / 16; ++kc) {
        const uint16_t* p = sQ + (warp * 16 + (lane & 15)) * LDS + kc * 16 + (lane >> 4) * 8;
        ldmatrix_x4(qf[kc], p);
      }
    }
    // S = Q K^T  (16 rows x 64 keys per warp)
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
    const uint16_t* K = sK[buf];
#pragma unroll
    for (int np = 0; np < 4; ++np) {
#pragma unroll
      for (int kc = 0; kc < D / 16; ++kc) {
        uint32_t b[4];
        const uint16_t* p = K + (np * 16 + (lane & 7) + ((lane >> 4) << 3)) * LDS + kc * 16 + ((lane >> 3) & 1) * 8;
        ldmatrix_x4(b, p);
        mma_bf16_16816(s[2 * np], qf[kc], b[0], b[1]);
        mma_bf16_16816(s[2 * np + 1], qf[kc], b[2], b[3]);
      }
    }
    // scale, mask keys beyond L, online softmax
    const int kbase = j * BKV;
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int k0 = kbase + nt * 8 + 2 * t;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool valid = (k0 + e) < L;
        s[nt][e] = valid ? s[nt][e] * scale_log2 : -INFINITY;
        s[nt][2 + e] = valid ? s[nt][2 + e] * scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[nt][e]);
        mx1 = fmaxf(mx1, s[nt][2 + e]);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);  // finite: block j has >= 1 valid key
    const float c0 = exp2f(m0 - mn0), c1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    l0 *= c0;
    l1 *= c1;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= c0; o[i][1] *= c0;
      o[i][2] *= c1; o[i][3] *= c1;
    }
    uint32_t pf[4][4];  // P as A fragments, 4 key chunks of 16
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = exp2f(s[nt][0] - mn0), p1 = exp2f(s[nt][1] - mn0);
      const float p2 = exp2f(s[nt][2] - mn1), p3 = exp2f(s[nt][3] - mn1);
      l0 += p0 + p1;
      l1 += p2 + p3;
      const int kc = nt >> 1, hi = nt & 1;
      pf[kc][hi * 2 + 0] = pack_bf16x2(p0, p1);
      pf[kc][hi * 2 + 1] = pack_bf16x2(p2, p3);
    }
    // O += P V
    const uint16_t* V = sV[buf];
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
#pragma unroll
      for (int dp = 0; dp < D / 16; ++dp) {
        uint32_t b[4];
        const uint16_t* p = V + (kc * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * LDS + dp * 16 + (lane >> 4) * 8;
        ldmatrix_x4_trans(b, p);
        mma_bf16_16816(o[2 * dp], pf[kc], b[0], b[1]);
        mma_bf16_16816(o[2 * dp + 1], pf[kc], b[2], b[3]);
      }
    }
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float inv0 = 1.0f / l0, inv1 = 1.0f / l1;
  const int r0 = q0 + warp * 16 + g, r1 = r0 + 8;
  uint16_t* out = ctx + static_cast<size_t>(start) * H + h * D;
#pragma unroll
  for (int dt = 0; dt < D / 8; ++dt) {
    const int col = dt * 8 + 2 * t;
    if (r0 < L)
      *reinterpret_cast<uint32_t*>(out + static_cast<size_t>(r0) * H + col) = pack_bf16x2(o[dt][0] * inv0, o[dt][1] * inv0);
    if (r1 < L)
      *reinterpret_cast<uint32_t*>(out + static_cast<size_t>(r1) * H + col) = pack_bf16x2(o[dt][2] * inv1, o[dt][3] * inv1);
  }
}
// ============================================================================ tcgen05 engine
// One CTA (4 warps) = (request, head, 128-row q tile), head dim 64; thread = query row = TMEM
// lane.  Q, K, V come from the head-major qkv planes the QKV GEMM writes ([3 nh][T][64]), so
// every TMA box is one contiguous 16 KB block.  Keys are processed in blocks of 128 (<= 4 per
// request, BERT max 512 tokens):
//   S_j = Q K_j^T        tcgen05 M 128 x N 128 x K 64, into TMEM columns [0, 128)
//   softmax block j      2 passes over the TMEM row (block max, then exp2 / sum), online
//                        rescaling of (m, l, O) with fp32 statistics; P_j packed to bf16
//                        pairs into TMEM columns [0, 64) over consumed scores
//   O_j = P_j V_j        tcgen05 with A = P_j from TMEM, B = V_j (MN-major) from shared memory,
//                        into TMEM columns [64, 128); accumulated in registers as O = a O + O_j
//   ctx = O / l          bf16
// Thread 0 issues the TMA loads (K_{j+1} overlaps softmax j, V_{j+1} overlaps S_{j+1}) and
// the MMAs in program order.  128 TMEM columns, 48 KB of shared memory and <= 128 registers
// per thread let 4 CTAs share an SM, so one CTA's loads and MMAs overlap another's softmax.
// (A persistent warp-specialised variant -- producer / MMA / softmax warps, 2 CTAs per SM --
// measured slower: 2.17 vs 1.75 ms per BGE-base step; see git history.)
// Keys >= L (the next request's) are masked; 32-key chunks / 16-key MMA steps with no valid
// key and query warps whose rows all lie beyond L are skipped.
constexpr int TQ = 128;        // q rows per CTA (= TMEM lanes)
constexpr int TKB = 128;       // keys per K/V block
constexpr int TD = 64;         // head dim
constexpr int kBlkBytes = TKB * TD * 2;  // 16 KB
constexpr int kAttnTcSmem = 3 * kBlkBytes + 1024 + 256;
constexpr uint32_t kOCol = 64;
// packed fp32 pairs (Blackwell FFMA2 / FADD2: two lanes of fp32 math per instruction)
ELIS_DEV unsigned long long f2_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
ELIS_DEV void f2_unpack(unsigned long long v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
ELIS_DEV unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
ELIS_DEV unsigned long long f2_add(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
ELIS_DEV unsigned long long f2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
constexpr float kLazyRescale = 8.f;  // log2 units: P <= 2^8 before O is rescaled
ELIS_DEV float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
ELIS_DEV float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// exp2 of a pair on the FMA pipe, to take part of the softmax exponentials off the MUFU
// (16 ex2 / clk / SM, the softmax bound when 4 CTAs share an SM):
//   j = rint(x) (x + 1.5 * 2^23 leaves j in the low mantissa bits), f = x - j in [-1/2, 1/2],
//   2^f = degree-3 minimax polynomial (max relative error 7.5e-5, scripts/fit_exp2.py; P is then
//   rounded to bf16, relative step 3.9e-3), 2^x = bits(2^f) + (j << 23).
// x is clamped at -125 so the exponent stays normal (the true value is then < 2^-125 next to the
// row maximum's 1).
#ifndef ELIS_EXP2_POLY
#define ELIS_EXP2_POLY 6  // pairs of every 16 in a 32-key chunk evaluated by exp2_poly2
#endif
ELIS_DEV unsigned long long exp2_poly2(float x0, float x1) {
  const unsigned long long xx = f2_pack(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
  const unsigned long long t = f2_add(xx, f2_pack(12582912.f, 12582912.f));
  const unsigned long long j = f2_add(t, f2_pack(-12582912.f, -12582912.f));
  const unsigned long long f = f2_fma(j, f2_pack(-1.f, -1.f), xx);
  unsigned long long p = f2_fma(f2_pack(0.0551716685f, 0.0551716685f), f, f2_pack(0.2426111251f, 0.2426111251f));
  p = f2_fma(p, f, f2_pack(0.6932609677f, 0.6932609677f));
  p = f2_fma(p, f, f2_pack(0.9999280572f, 0.9999280572f));
  float p0, p1, t0, t1;
  f2_unpack(p, p0, p1);
  f2_unpack(t, t0, t1);
  return f2_pack(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(t0) << 23)),
                 __uint_as_float(__float_as_uint(p1) + (__float_as_uint(t1) << 23)));
}
ELIS_DEV constexpr bool exp2_on_fma(int pair) {
  return ((pair + 1) * ELIS_EXP2_POLY) / 16 != (pair * ELIS_EXP2_POLY) / 16;  // spread over the chunk
}

// F8OUT: ctx written as E4M3(ctx_scale * ctx) bytes [T, H] (the FP8 out-projection's A operand)
// F16: Q, K, V, P and ctx in fp16 instead of bf16 (fp16 operand precision)
template <bool F8OUT, bool F16>
__global__ void __launch_bounds__(128, 4)
    k_attention_tc(const __grid_constant__ CUtensorMap tm,
                   const AttnWork* __restrict__ work, const int32_t* __restrict__ num_work, int H, int nh,
                   uint16_t* __restrict__ ctx, float scale_log2, int Tp, float ctx_scale) {
#ifdef ELIS_ATTN_TRACE
  const unsigned long long t_start = attn_gtime();
#endif
  // the work entry is read together with num_work (the list has capacity for every CTA; entries
  // past num_work are never used) and carries the request bounds: no dependent loads
  pdl_wait();  // the work list and the qkv planes come from earlier kernels (common.cuh)
  pdl_trigger();
  const int item = static_cast<int>(blockIdx.x) / nh, h = static_cast<int>(blockIdx.x) % nh;
  const AttnWork w = work[item];
  if (item >= __ldg(num_work)) return;
  ATTN_TRACE(0, t_start);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kBlkBytes;
  uint8_t* sV = sK + kBlkBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kBlkBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = bars + 2;
  uint64_t* s_full = bars + 3;
  uint64_t* o_full = bars + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);

  const int start = w.start, L = w.len, q0 = w.q0;
  const int nkb = (L + TKB - 1) / TKB;  // 1..4
  const int warp = warp_id(), lane = lane_id();
  const bool issuer = threadIdx.x == 0;

  if (issuer) {  // barriers + the first loads go out before the TMEM allocation / CTA barrier
    tma_prefetch_desc(&tm);
    mbar_init(q_full, 1);
    mbar_init(k_full, 1);
    mbar_init(v_full, 1);
    mbar_init(s_full, 1);
    mbar_init(o_full, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(q_full, kBlkBytes);
    tma_load_2d(sQ, &tm, q_full, 0, h * Tp + start + q0);
    mbar_arrive_expect_tx(k_full, kBlkBytes);
    tma_load_2d(sK, &tm, k_full, 0, (nh + h) * Tp + start);
    mbar_arrive_expect_tx(v_full, kBlkBytes);
    tma_load_2d(sV, &tm, v_full, 0, (2 * nh + h) * Tp + start);
  }
  if (warp == 1) tmem_alloc<128>(tmem_slot);  // warp 0's thread 0 is issuing the loads
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ATTN_TRACE(1, attn_gtime());
  const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int row = warp * 32 + lane;
  // warps whose 32 query rows all lie beyond L skip the softmax (their rows are never stored;
  // MMA rows are independent)
  const bool warp_active = q0 + warp * 32 < L;

  constexpr uint32_t idesc_s = F16 ? make_idesc_f16_f32(TQ, TKB) : make_idesc_bf16_f32(TQ, TKB);
  constexpr uint32_t idesc_o = (F16 ? make_idesc_f16_f32(TQ, TD) : make_idesc_bf16_f32(TQ, TD)) | (1u << 16);  // V MN-major
  if (issuer) mbar_wait(q_full, 0);
  float m = -INFINITY, l = 0.f;   // running row max (scaled, log2 domain) and row sum
  unsigned long long o2[TD / 2];  // O as fp32 pairs
  const unsigned long long zero2 = f2_pack(0.f, 0.f);

  for (int j = 0; j < nkb; ++j) {
    const uint32_t ph = j & 1;
    if (issuer) {
      // S_j = Q K_j^T (4 x K16 steps, +32 B inside the 128 B swizzle row)
      mbar_wait(k_full, ph);
      tc_fence_after();
      const uint64_t dq = make_sw128_desc(smem_u32(sQ));
      const uint64_t dk = make_sw128_desc(smem_u32(sK));
#pragma unroll
      for (int k = 0; k < TD / 16; ++k) tc_mma_f16(tmem, dq + 2 * k, dk + 2 * k, idesc_s, k > 0);
      tc_commit(s_full);
    }
    mbar_wait(s_full, ph);
    tc_fence_after();
    if (j == 0) ATTN_TRACE(2, attn_gtime());
    if (issuer && j + 1 < nkb) {  // the S MMA has consumed K_j: prefetch K_{j+1}
      mbar_arrive_expect_tx(k_full, kBlkBytes);
      tma_load_2d(sK, &tm, k_full, 0, (nh + h) * Tp + start + (j + 1) * TKB);
    }
    const int nvalid_blk = L - j * TKB;  // keys >= L belong to other requests: masked
    // 32-key chunks holding valid keys
    const int nch = warp_active ? min(TKB / 32, (nvalid_blk + 31) / 32) : 0;
    // pass A: block max (single-buffered TMEM loads: registers are budgeted for 4 CTAs / SM).
    // Only the chunk holding the last valid key is masked.
    uint32_t r[32];
    float bm = -INFINITY;
#pragma unroll
    for (int c = 0; c < TKB / 32; ++c) {
      if (c < nch) {
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tc_wait_ld();
        const int nv = nvalid_blk - c * 32;
        if (nv < 32) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e >= nv) r[e] = __float_as_uint(-INFINITY);
        }
        float t[11];
#pragma unroll
        for (int e = 0; e < 10; ++e)
          t[e] = fmax3(__uint_as_float(r[3 * e]), __uint_as_float(r[3 * e + 1]), __uint_as_float(r[3 * e + 2]));
        t[10] = fmax3(__uint_as_float(r[30]), __uint_as_float(r[31]), bm);
        bm = fmax3(fmax3(t[0], t[1], t[2]), fmax3(t[3], t[4], t[5]), fmax3(t[6], t[7], fmax3(t[8], t[9], t[10])));
      }
    }
    const float m_new = fmaxf(m, bm * scale_log2);  // finite: every block has >= 1 valid key
    const float alpha = ex2_approx(m - m_new);      // 0 on the first block
    m = m_new;
    // pass B: p = exp2(s*scale - m), block sum, P (bf16 pairs) over consumed score columns
    const unsigned long long sc2 = f2_pack(scale_log2, scale_log2);
    const unsigned long long nm2 = f2_pack(-m, -m);
    unsigned long long acc0 = zero2, acc1 = zero2;  // 2 x 2 independent partial sums, fixed order
#pragma unroll
    for (int c = 0; c < TKB / 32; ++c) {
      if (c < nch) {
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tc_wait_ld();
        const int nv = nvalid_blk - c * 32;
        float p[32];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          float x0, x1;
          f2_unpack(f2_fma(f2_pack(__uint_as_float(r[2 * e]), __uint_as_float(r[2 * e + 1])), sc2, nm2), x0, x1);
          if (exp2_on_fma(e)) {
            f2_unpack(exp2_poly2(x0, x1), p[2 * e], p[2 * e + 1]);
          } else {
            p[2 * e] = ex2_approx(x0);
            p[2 * e + 1] = ex2_approx(x1);
          }
        }
        if (nv < 32) {
#pragma unroll
          for (int e = 0; e < 32; ++e) p[e] = (e < nv) ? p[e] : 0.f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          acc0 = f2_add(acc0, f2_pack(p[4 * e], p[4 * e + 1]));
          acc1 = f2_add(acc1, f2_pack(p[4 * e + 2], p[4 * e + 3]));
        }
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) pk[e] = pack16x2<F16>(p[2 * e], p[2 * e + 1]);
        tmem_st_32x32b_x16(taddr + c * 16, pk);
      }
    }
    float a0, a1, a2, a3;
    f2_unpack(acc0, a0, a1);
    f2_unpack(acc1, a2, a3);
    l = l * alpha + ((a0 + a1) + (a2 + a3));
    tc_wait_st();
    tc_fence_before();
    __syncthreads();  // P_j complete in TMEM (all 128 rows)
    if (j == 0) ATTN_TRACE(3, attn_gtime());
    if (issuer) {
      tc_fence_after();
      mbar_wait(v_full, ph);
      const int nks = min(TKB / 16, (nvalid_blk + 15) / 16);  // 16-key steps holding valid keys
      for (int ks = 0; ks < nks; ++ks) {
        const uint64_t dv = make_sw128_desc(smem_u32(sV + ks * (16 * TD * 2)));
        tc_mma_f16_tmem_a(tmem + kOCol, tmem + ks * 8, dv, idesc_o, ks > 0);
      }
      tc_commit(o_full);
    }
    mbar_wait(o_full, ph);
    tc_fence_after();
    if (j == 0) ATTN_TRACE(4, attn_gtime());
    if (issuer && j + 1 < nkb) {  // the PV MMA has consumed V_j: prefetch V_{j+1}
      mbar_arrive_expect_tx(v_full, kBlkBytes);
      tma_load_2d(sV, &tm, v_full, 0, (2 * nh + h) * Tp + start + (j + 1) * TKB);
    }
    // O = alpha O + O_j  (the first block just takes O_0)
    if (warp_active) {
      const unsigned long long al2 = f2_pack(alpha, alpha);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        tmem_ld_32x32b_x32(taddr + kOCol + hf * 32, r);
        tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const unsigned long long oj = f2_pack(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
          o2[hf * 16 + i] = (j == 0) ? oj : f2_fma(o2[hf * 16 + i], al2, oj);
        }
      }
    }
    tc_fence_before();
    __syncthreads();  // every row has read O_j before the next S MMA overwrites columns [0, 128)
    if (j == 0) ATTN_TRACE(5, attn_gtime());
  }
  // epilogue: ctx = O / l (bf16).  Rows are staged in shared memory (sQ: the last S MMA has
  // completed) with 16-byte chunks XOR-swizzled by row, then written back 4 rows per warp
  // instruction, each row one contiguous 128-byte line (thread-per-row stores would touch 32
  // lines per instruction).
  {
    float o[TD];
#pragma unroll
    for (int i = 0; i < TD / 2; ++i) f2_unpack(o2[i], o[2 * i], o[2 * i + 1]);
    if constexpr (F8OUT) {  // 64-byte rows: 4 pieces, XOR-swizzled by row & 3
      const float inv = ctx_scale / l;
      uint4* srow = reinterpret_cast<uint4*>(sQ + row * TD);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        srow[k ^ (row & 3)] =
            make_uint4(pack_e4m3x4(o[16 * k + 0] * inv, o[16 * k + 1] * inv, o[16 * k + 2] * inv, o[16 * k + 3] * inv),
                       pack_e4m3x4(o[16 * k + 4] * inv, o[16 * k + 5] * inv, o[16 * k + 6] * inv, o[16 * k + 7] * inv),
                       pack_e4m3x4(o[16 * k + 8] * inv, o[16 * k + 9] * inv, o[16 * k + 10] * inv, o[16 * k + 11] * inv),
                       pack_e4m3x4(o[16 * k + 12] * inv, o[16 * k + 13] * inv, o[16 * k + 14] * inv,
                                   o[16 * k + 15] * inv));
    } else {
      const float inv = 1.0f / l;
      uint4* srow = reinterpret_cast<uint4*>(sQ + row * (TD * 2));
#pragma unroll
      for (int k = 0; k < 8; ++k)
        srow[k ^ (row & 7)] = make_uint4(pack16x2<F16>(o[8 * k + 0] * inv, o[8 * k + 1] * inv),
                                         pack16x2<F16>(o[8 * k + 2] * inv, o[8 * k + 3] * inv),
                                         pack16x2<F16>(o[8 * k + 4] * inv, o[8 * k + 5] * inv),
                                         pack16x2<F16>(o[8 * k + 6] * inv, o[8 * k + 7] * inv));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
  {
    const int nrows = min(TQ, L - q0);
    if constexpr (F8OUT) {
      uint8_t* c8 = reinterpret_cast<uint8_t*>(ctx);
      const int c = lane & 3;
      for (int rr = warp * 8 + (lane >> 2); rr < nrows; rr += 32) {
        const uint4 v = reinterpret_cast<const uint4*>(sQ + rr * TD)[c ^ (rr & 3)];
        *reinterpret_cast<uint4*>(c8 + static_cast<size_t>(start + q0 + rr) * H + h * TD + c * 16) = v;
      }
    } else {
      const int c = lane & 7;
      for (int rr = warp * 4 + (lane >> 3); rr < nrows; rr += 16) {
        const uint4 v = reinterpret_cast<const uint4*>(sQ + rr * (TD * 2))[c ^ (rr & 7)];
        *reinterpret_cast<uint4*>(ctx + static_cast<size_t>(start + q0 + rr) * H + h * TD + c * 8) = v;
      }
    }
  }
#ifdef ELIS_ATTN_TRACE
  ATTN_TRACE(6, attn_gtime());
  ATTN_TRACE(7, (static_cast<unsigned long long>(attn_smid()) << 32) | (static_cast<unsigned>(L) << 8) | nkb);
#endif
}

// ---------------------------------------------------------------------- 64-key-block engine (default)
// Same CTA shape (128 q rows x one head, 4 warps, 4 CTAs per SM, 128 TMEM columns), keys in
// blocks of 64 so that O can stay in TMEM:
//   S_j = Q K_j^T        M 128 x N 64 x K 64 into TMEM columns [0, 64)
//   softmax block j      one pass: the row's 64 scores read into registers (2 loads, one wait),
//                        block max, lazy running max (it moves only when the block's exceeds it
//                        by more than 2^8; then O is rescaled in TMEM), exp2, row sum, P packed
//                        to 16 bits into columns [0, 32) over the consumed scores
//   O += P_j V_j         A = P_j from TMEM, B = V_j (MN-major) from shared memory, accumulated in
//                        TMEM columns [64, 128) across blocks; S_{j+1} is issued right behind it
//                        (MMAs execute in issue order), so the next softmax waits for S only
//   ctx = O / l          after the last block
// No O in registers (the round-1 block of 128 keys folded O_j into 64 registers per thread, with
// two serial TMEM passes per block).  Once S_j has completed, K_{j+2} is loaded into K_j's buffer
// and V_{j+1} into V_{j-1}'s (S_j's completion implies PV_{j-1}'s).  Measured (A/B, one session,
// profiles/r02_ab_attention_64key.txt): cfg2 attention 1.58 / 1.53 vs 1.60 / 1.54 ms per step,
// cfg5 8.42 vs 8.58 ms; ELIS_ATTN_ENGINE=128 selects the 128-key engine above.
// MMA issue in the 64-key engine: 1 (default) = warp 0 converged with one lane elected in the asm,
// 0 = thread 0 alone (per-operand uniform-register broadcasts around every MMA)
#ifndef ELIS_ATTN_WARP_ISSUE
#define ELIS_ATTN_WARP_ISSUE 1
#endif
#if ELIS_ATTN_WARP_ISSUE
#define ATTN_MMA_SS tc_mma_f16_w
#define ATTN_MMA_TS tc_mma_f16_tmem_a_w
#define ATTN_COMMIT tc_commit_w
#else
#define ATTN_MMA_SS tc_mma_f16
#define ATTN_MMA_TS tc_mma_f16_tmem_a
#define ATTN_COMMIT tc_commit
#endif
constexpr int TKB64 = 64;
constexpr int kBlk64 = TKB64 * TD * 2;                        // 8 KB
constexpr int kAttn64Smem = kBlkBytes + 4 * kBlk64 + 1024 + 256;  // Q, K[2], V[2]
template <bool F8OUT, bool F16>
__global__ void __launch_bounds__(128, 4)
    k_attention_tc64(const __grid_constant__ CUtensorMap tm, const AttnWork* __restrict__ work,
                     const int32_t* __restrict__ num_work, int H, int nh, uint16_t* __restrict__ ctx,
                     float scale_log2, int Tp, float ctx_scale) {
  pdl_wait();  // the work list and the qkv planes come from earlier kernels (common.cuh)
  pdl_trigger();
  const int item = static_cast<int>(blockIdx.x) / nh, h = static_cast<int>(blockIdx.x) % nh;
  const AttnWork w = work[item];
  if (item >= __ldg(num_work)) return;
  unsigned tr_k = 0;
  (void)tr_k;
  ATR(1);  // start
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* sQ = smem;                      // 128 rows
  uint8_t* sK = sQ + kBlkBytes;            // [2][64 rows]
  uint8_t* sV = sK + 2 * kBlk64;           // [2][64 rows]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * kBlk64);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;             // [2]
  uint64_t* v_full = bars + 3;             // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* o_full = bars + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7);

  const int start = w.start, L = w.len, q0 = w.q0;
  const int nkb = (L + TKB64 - 1) / TKB64;  // 1..8
  const int warp = warp_id(), lane = lane_id();
  const bool issuer = threadIdx.x == 0;
  const int rq = h * Tp + start, rk = (nh + h) * Tp + start, rv = (2 * nh + h) * Tp + start;
  // K_j / V_j into buffer j & 1 (64-row boxes).  K_j is consumed by S_j, V_j only by PV_j one
  // step later, so K is loaded two blocks ahead and V one.
  auto load_k = [&](int j) {
    mbar_arrive_expect_tx(&k_full[j & 1], kBlk64);
    tma_load_2d(sK + (j & 1) * kBlk64, &tm, &k_full[j & 1], 0, rk + j * TKB64);
  };
  auto load_v = [&](int j) {
    mbar_arrive_expect_tx(&v_full[j & 1], kBlk64);
    tma_load_2d(sV + (j & 1) * kBlk64, &tm, &v_full[j & 1], 0, rv + j * TKB64);
  };
  if (issuer) {
    tma_prefetch_desc(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(o_full, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(q_full, kBlkBytes);
    tma_load_2d(sQ, &tm, q_full, 0, rq + q0);
    tma_load_2d(sQ + kBlk64, &tm, q_full, 0, rq + q0 + 64);
    load_k(0);
    load_v(0);
    if (nkb > 1) load_k(1);
  }
  if (warp == 1) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int row = warp * 32 + lane;
  const bool warp_active = q0 + warp * 32 < L;
  constexpr uint32_t idesc_s = F16 ? make_idesc_f16_f32(TQ, TKB64) : make_idesc_bf16_f32(TQ, TKB64);
  constexpr uint32_t idesc_o = (F16 ? make_idesc_f16_f32(TQ, TD) : make_idesc_bf16_f32(TQ, TD)) | (1u << 16);
  const uint64_t dq = make_sw128_desc(smem_u32(sQ));
  ATR(2);  // setup done (barriers, TMEM)
  if (ELIS_ATTN_WARP_ISSUE ? warp == 0 : issuer) {  // S_0 (MMAs: warp 0 converged, one lane elected)
    mbar_wait(q_full, 0);
    mbar_wait(&k_full[0], 0);
    ATR(3);  // Q, K_0, V_0 loaded
    if (ELIS_ATTN_WARP_ISSUE) __syncwarp();  // the elect.sync in the MMA issue needs the whole warp converged
    tc_fence_after();
    const uint64_t dk = make_sw128_desc(smem_u32(sK));
#pragma unroll
    for (int k = 0; k < TD / 16; ++k) ATTN_MMA_SS(tmem, dq + 2 * k, dk + 2 * k, idesc_s, k > 0);
    ATTN_COMMIT(s_full);
  }
  float m = 0.f, l = 0.f;
  const unsigned long long sc2 = f2_pack(scale_log2, scale_log2);
  for (int j = 0; j < nkb; ++j) {
    ATR(4);  // wait S_j
    mbar_wait(s_full, j & 1);
    ATR(5);  // S_j ready
    tc_fence_after();
    // S_j complete (so K_j consumed, and PV_{j-1} complete): K_{j+2} into K_j's buffer, V_{j+1}
    // into V_{j-1}'s
    if (issuer) {
      if (j + 2 < nkb) load_k(j + 2);
      if (j + 1 < nkb) load_v(j + 1);
    }
    const int nk = min(TKB64, L - j * TKB64);   // valid keys of this block (keys >= L: other requests)
    const int nch = (nk + 31) >> 5;             // 1..2
    if (warp_active) {
      uint32_t r[2][32];
      tmem_ld_32x32b_x32(taddr, r[0]);
      if (nch > 1) tmem_ld_32x32b_x32(taddr + 32, r[1]);
      tc_wait_ld();
      // the chunk holding the last valid key (if partial) is masked; each test names its chunk at
      // compile time (no dynamic indexing of the score registers)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c < nch && nk < 32 * (c + 1)) {
          const int tail = nk - 32 * c;
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e >= tail) r[c][e] = __float_as_uint(-INFINITY);
        }
      }
      float mx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = __uint_as_float(r[0][i]);
#pragma unroll
      for (int e = 8; e < 32; e += 2) mx[(e >> 1) & 7] = fmax3(mx[(e >> 1) & 7], __uint_as_float(r[0][e]), __uint_as_float(r[0][e + 1]));
      if (nch > 1) {
#pragma unroll
        for (int e = 0; e < 32; e += 2) mx[(e >> 1) & 7] = fmax3(mx[(e >> 1) & 7], __uint_as_float(r[1][e]), __uint_as_float(r[1][e + 1]));
      }
      const float bm = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
      const float ms = bm * scale_log2;  // finite: the block holds >= 1 valid key
      float alpha = 1.f;
      bool resc = false;
      if (j == 0) {
        m = ms;
      } else if (ms > m + kLazyRescale) {  // rare: O rescaled below, once the scores are consumed
        alpha = ex2_approx(m - ms);
        m = ms;
        l *= alpha;
        resc = true;
      }
      const unsigned long long nm2 = f2_pack(-m, -m);
      unsigned long long acc0 = f2_pack(0.f, 0.f), acc1 = acc0;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c < nch) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float x0, x1, p0, p1;
            f2_unpack(f2_fma(f2_pack(__uint_as_float(r[c][2 * e]), __uint_as_float(r[c][2 * e + 1])), sc2, nm2), x0, x1);
            if (exp2_on_fma(e)) {
              f2_unpack(exp2_poly2(x0, x1), p0, p1);
            } else {
              p0 = ex2_approx(x0);
              p1 = ex2_approx(x1);
            }
            r[c][2 * e] = __float_as_uint(p0);
            r[c][2 * e + 1] = __float_as_uint(p1);
          }
          if (nk < 32 * (c + 1)) {  // masked keys contribute exactly 0
            const int tail = nk - 32 * c;
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e >= tail) r[c][e] = 0u;
          }
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            acc0 = f2_add(acc0, f2_pack(__uint_as_float(r[c][4 * e]), __uint_as_float(r[c][4 * e + 1])));
            acc1 = f2_add(acc1, f2_pack(__uint_as_float(r[c][4 * e + 2]), __uint_as_float(r[c][4 * e + 3])));
          }
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) pk[e] = pack16x2<F16>(__uint_as_float(r[c][2 * e]), __uint_as_float(r[c][2 * e + 1]));
          tmem_st_32x32b_x16(taddr + c * 16, pk);
        }
      }
      float a0, a1, a2, a3;
      f2_unpack(acc0, a0, a1);
      f2_unpack(acc1, a2, a3);
      l += (a0 + a1) + (a2 + a3);
      // O (complete: PV_{j-1} preceded S_j) *= alpha, before PV_j is issued; warp-uniform because
      // tcgen05.ld / st are warp-collective (alpha = 1 exactly in the rows that did not rescale)
      if (__any_sync(0xffffffffu, resc)) {
        const unsigned long long al2 = f2_pack(alpha, alpha);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(taddr + kOCol + x * 32, o);
          tc_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float o0, o1;
            f2_unpack(f2_mul(f2_pack(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1])), al2), o0, o1);
            o[2 * i] = __float_as_uint(o0);
            o[2 * i + 1] = __float_as_uint(o1);
          }
          tmem_st_32x32b_x32(taddr + kOCol + x * 32, o);
        }
      }
      tc_wait_st();
    }
    ATR(6);  // thread 0's softmax done
    tc_fence_before();
    __syncthreads();  // P_j complete in TMEM (all 128 rows)
    ATR(7);  // all warps' P_j in TMEM
    if (ELIS_ATTN_WARP_ISSUE ? warp == 0 : issuer) {
      tc_fence_after();
      const int b = j & 1;
      mbar_wait(&v_full[b], (j >> 1) & 1);
      ATR(8);  // V_j (and K_j) loaded
      if (ELIS_ATTN_WARP_ISSUE) __syncwarp();  // the elect.sync in the MMA issue needs the whole warp converged
      const int nks = (nk + 15) / 16;  // 16-key steps holding valid keys
      for (int ks = 0; ks < nks; ++ks) {
        const uint64_t dv = make_sw128_desc(smem_u32(sV + b * kBlk64 + ks * (16 * TD * 2)));
        ATTN_MMA_TS(tmem + kOCol, tmem + ks * 8, dv, idesc_o, (j | ks) != 0 ? 1u : 0u);
      }
      if (j + 1 < nkb) {  // S_{j+1} right behind PV_j (in issue order: P_j is read before S overwrites it)
        const int b1 = (j + 1) & 1;
        mbar_wait(&k_full[b1], ((j + 1) >> 1) & 1);
        if (ELIS_ATTN_WARP_ISSUE) __syncwarp();  // the elect.sync in the MMA issue needs the whole warp converged
        tc_fence_after();
        const uint64_t dk = make_sw128_desc(smem_u32(sK + b1 * kBlk64));
#pragma unroll
        for (int k = 0; k < TD / 16; ++k) ATTN_MMA_SS(tmem, dq + 2 * k, dk + 2 * k, idesc_s, k > 0);
        ATTN_COMMIT(s_full);
      } else {
        ATTN_COMMIT(o_full);
      }
    }
  }
  ATR(9);  // wait last PV
  mbar_wait(o_full, 0);
  ATR(10);  // O complete
  tc_fence_after();
  // epilogue: ctx = O / l, staged in sQ (every MMA has completed), 4 rows per warp instruction
  if (warp_active) {
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(taddr + kOCol + x * 32, v);
      tc_wait_ld();
      if constexpr (F8OUT) {  // 64-byte rows: 4 pieces, XOR-swizzled by row & 3
        const float inv = ctx_scale / l;
        uint4* srow = reinterpret_cast<uint4*>(sQ + row * TD);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const uint32_t* u = v + 16 * k;
          srow[(2 * x + k) ^ (row & 3)] = make_uint4(
              pack_e4m3x4(__uint_as_float(u[0]) * inv, __uint_as_float(u[1]) * inv, __uint_as_float(u[2]) * inv,
                          __uint_as_float(u[3]) * inv),
              pack_e4m3x4(__uint_as_float(u[4]) * inv, __uint_as_float(u[5]) * inv, __uint_as_float(u[6]) * inv,
                          __uint_as_float(u[7]) * inv),
              pack_e4m3x4(__uint_as_float(u[8]) * inv, __uint_as_float(u[9]) * inv, __uint_as_float(u[10]) * inv,
                          __uint_as_float(u[11]) * inv),
              pack_e4m3x4(__uint_as_float(u[12]) * inv, __uint_as_float(u[13]) * inv, __uint_as_float(u[14]) * inv,
                          __uint_as_float(u[15]) * inv));
        }
      } else {
        const float inv = 1.0f / l;
        uint4* srow = reinterpret_cast<uint4*>(sQ + row * (TD * 2));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t* u = v + 8 * k;
          srow[(4 * x + k) ^ (row & 7)] =
              make_uint4(pack16x2<F16>(__uint_as_float(u[0]) * inv, __uint_as_float(u[1]) * inv),
                         pack16x2<F16>(__uint_as_float(u[2]) * inv, __uint_as_float(u[3]) * inv),
                         pack16x2<F16>(__uint_as_float(u[4]) * inv, __uint_as_float(u[5]) * inv),
                         pack16x2<F16>(__uint_as_float(u[6]) * inv, __uint_as_float(u[7]) * inv));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
  {
    const int nrows = min(TQ, L - q0);
    if constexpr (F8OUT) {
      uint8_t* c8 = reinterpret_cast<uint8_t*>(ctx);
      const int c = lane & 3;
      for (int rr = warp * 8 + (lane >> 2); rr < nrows; rr += 32) {
        const uint4 v = reinterpret_cast<const uint4*>(sQ + rr * TD)[c ^ (rr & 3)];
        *reinterpret_cast<uint4*>(c8 + static_cast<size_t>(start + q0 + rr) * H + h * TD + c * 16) = v;
      }
    } else {
      const int c = lane & 7;
      for (int rr = warp * 4 + (lane >> 3); rr < nrows; rr += 16) {
        const uint4 v = reinterpret_cast<const uint4*>(sQ + rr * (TD * 2))[c ^ (rr & 7)];
        *reinterpret_cast<uint4*>(ctx + static_cast<size_t>(start + q0 + rr) * H + h * TD + c * 8) = v;
      }
    }
  }
  ATR(11);  // end
  ATR_DONE();
}

// ---------------------------------------------------------------------- persistent 64-key engine
// The 64-key engine above as a persistent kernel: 4 CTAs per SM (same 128 TMEM columns, 48 KB of
// shared memory, thread = query row), each looping over work items c, c + G, c + 2G, ... (G = grid
// size; the list is in descending cost order, so the stride schedule balances).  Per CTA the barrier
// init, TMEM allocation and tensor-map prefetch happen once, and the K / V stream runs across item
// boundaries: blocks are numbered g = 0, 1, ... over the CTA's whole sequence, K_g and V_g live in
// buffer g & 1, and "S_g complete" (which implies PV_{g-1} complete: MMAs finish in issue order)
// releases the loads of K_{g+2} and V_{g+1} even when those belong to the next item (only the
// current and the next item are looked ahead; a block two items ahead waits for the next event).
// The next item's Q is loaded once the current item's last S has completed, and its first S is
// issued right behind the last PV, so it runs under the epilogue (O read from TMEM, ctx = O / l
// stored straight from registers, one 128-byte row per thread).  The per-item arithmetic -- every
// MMA, the softmax and the epilogue rounding -- is the 64-key engine's, in the same order, so
// results are bitwise those of k_attention_tc64.
#ifdef ELIS_ATTN_DBG
// diagnostic build: bounded waits that report which barrier / block a persistent CTA is stuck on
__device__ void mbar_wait_dbg(uint64_t* bar, uint32_t parity, int id, int g, int it) {  // g: block, it: item
  for (long long i = 0; i < (1ll << 22); ++i) {
    uint32_t ok;
    asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (ok) return;
  }
  if ((threadIdx.x & 31) == 0)
    printf("stuck: cta %d thread %d barrier %d parity %u g %d it %d\n", blockIdx.x, threadIdx.x, id, parity, g, it);
}
#define PWAIT(bar, par, id) mbar_wait_dbg(bar, par, id, g, it)
#define EWAIT(bar, par, id, j) mbar_wait_dbg(bar, par, id, j, -1)
#else
#define EWAIT(bar, par, id, j) mbar_wait(bar, par)
#define PWAIT(bar, par, id) mbar_wait(bar, par)
#endif
// ---------------------------------------------------------------------- early-S 64-key engine
// The 64-key engine with S_{j+1} issued while softmax j runs.  In the engines above P_j overwrites
// S_j in TMEM, so S_{j+1} can only be issued after PV_j, and every block pays PV issue + S issue +
// S latency (~650 cycles) with its softmax warps idle -- and the 4 CTAs of an SM fall into step
// (all in softmax, then all waiting on the shared tensor pipe).  Here P_j goes to shared memory
// (128 rows x 64 keys, the SWIZZLE_128B K-major layout TMA gives Q, so PV_j is an SS MMA), and
// TMEM holds only S (64 columns) and O (64 columns).  A fifth warp issues TMA and MMAs:
//   S_{j+1}   as soon as the 4 softmax warps have read S_j into registers (s_free) and K_{j+1} landed
//   PV_j      once P_j is in shared memory (p_full); committed to pv_done
//   K_{j+2}   into K_j's buffer once S_{j+1} is issued (S_j completed before s_free)
//   V_{j+1}   into V_{j-1}'s buffer once PV_{j-1} completed
// The softmax warps wait for PV_{j-1} (pv_done) before writing P_j over P_{j-1} and before a lazy
// O rescale.  64 KB of shared memory and 160 threads: 3 CTAs per SM.  Per-block arithmetic (MMA
// shapes and order, softmax, P rounding, epilogue) is the 64-key engine's, so results are bitwise
// those of k_attention_tc64.
constexpr int kAttnESmem = kBlkBytes + 4 * kBlk64 + kBlkBytes + 1024 + 256;  // Q, K[2], V[2], P
template <bool F8OUT, bool F16>
__global__ void __launch_bounds__(160, 3)
    k_attention_tc64e(const __grid_constant__ CUtensorMap tm, const AttnWork* __restrict__ work,
                      const int32_t* __restrict__ num_work, int H, int nh, uint16_t* __restrict__ ctx,
                      float scale_log2, int Tp, float ctx_scale) {
  pdl_wait();  // the work list and the qkv planes come from earlier kernels (common.cuh)
  pdl_trigger();
  const int item = static_cast<int>(blockIdx.x) / nh, h = static_cast<int>(blockIdx.x) % nh;
  const AttnWork w = work[item];
  if (item >= __ldg(num_work)) return;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* sQ = smem;                      // 128 rows
  uint8_t* sK = sQ + kBlkBytes;            // [2][64 rows]
  uint8_t* sV = sK + 2 * kBlk64;           // [2][64 rows]
  uint8_t* sP = sV + 2 * kBlk64;           // 128 rows x 64 keys, SWIZZLE_128B K-major
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kBlkBytes);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;             // [2]
  uint64_t* v_full = bars + 3;             // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* s_free = bars + 6;             // 4 arrivals: S_j read by every softmax warp
  uint64_t* p_full = bars + 7;             // 4 arrivals: P_j written by every softmax warp
  uint64_t* pv_done = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);

  const int start = w.start, L = w.len, q0 = w.q0;
  const int nkb = (L + TKB64 - 1) / TKB64;  // 1..8
  const int warp = warp_id(), lane = lane_id();
  const bool issuer = threadIdx.x == 128;   // warp 4, lane 0
  const int rq = h * Tp + start, rk = (nh + h) * Tp + start, rv = (2 * nh + h) * Tp + start;
  auto load_k = [&](int j) {
    mbar_arrive_expect_tx(&k_full[j & 1], kBlk64);
    tma_load_2d(sK + (j & 1) * kBlk64, &tm, &k_full[j & 1], 0, rk + j * TKB64);
  };
  auto load_v = [&](int j) {
    mbar_arrive_expect_tx(&v_full[j & 1], kBlk64);
    tma_load_2d(sV + (j & 1) * kBlk64, &tm, &v_full[j & 1], 0, rv + j * TKB64);
  };
  if (issuer) {
    tma_prefetch_desc(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(q_full, kBlkBytes);
    tma_load_2d(sQ, &tm, q_full, 0, rq + q0);
    tma_load_2d(sQ + kBlk64, &tm, q_full, 0, rq + q0 + 64);
    load_k(0);
    load_v(0);
    if (nkb > 1) {
      load_k(1);
      load_v(1);
    }
  }
  if (warp == 1) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc_s = F16 ? make_idesc_f16_f32(TQ, TKB64) : make_idesc_bf16_f32(TQ, TKB64);
  constexpr uint32_t idesc_o = (F16 ? make_idesc_f16_f32(TQ, TD) : make_idesc_bf16_f32(TQ, TD)) | (1u << 16);

  float m = 0.f, l = 0.f;  // softmax warps: running row max (log2 units) and row sum
  if (warp == 4) {
    // ------------------------------------------------ TMA + MMA issuer
    if (issuer) {
      const uint64_t dq = make_sw128_desc(smem_u32(sQ));
      const uint64_t dp = make_sw128_desc(smem_u32(sP));
      auto issue_s = [&](int j) {
        const int b = j & 1;
        EWAIT(&k_full[b], (j >> 1) & 1, 1, j);
        tc_fence_after();
        const uint64_t dk = make_sw128_desc(smem_u32(sK + b * kBlk64));
#pragma unroll
        for (int k = 0; k < TD / 16; ++k) tc_mma_f16(tmem, dq + 2 * k, dk + 2 * k, idesc_s, k > 0);
        tc_commit(s_full);
      };
      EWAIT(q_full, 0, 0, 0);
      issue_s(0);
      for (int j = 0; j < nkb; ++j) {
        if (j + 1 < nkb) {
          EWAIT(s_free, j & 1, 7, j);  // S_j is in the softmax warps' registers (and S_j completed)
          tc_fence_after();
          issue_s(j + 1);
          if (j + 2 < nkb) load_k(j + 2);  // K_j consumed by S_j
          if (j >= 1) {                    // V_{j+1} over V_{j-1}: PV_{j-1} must have completed
            EWAIT(pv_done, (j - 1) & 1, 9, j);
            load_v(j + 1);
          }
        }
        const int nk = min(TKB64, L - j * TKB64);
        const int b = j & 1;
        EWAIT(p_full, j & 1, 8, j);
        EWAIT(&v_full[b], (j >> 1) & 1, 3, j);
        tc_fence_after();
        const int nks = (nk + 15) / 16;
        for (int ks = 0; ks < nks; ++ks) {
          const uint64_t dv = make_sw128_desc(smem_u32(sV + b * kBlk64 + ks * (16 * TD * 2)));
          tc_mma_f16(tmem + kOCol, dp + 2 * ks, dv, idesc_o, (j | ks) != 0 ? 1u : 0u);
        }
        tc_commit(pv_done);
      }
    }
  } else {
    // ------------------------------------------------ softmax warps (thread = query row)
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const int row = warp * 32 + lane;
    const bool warp_active = q0 + warp * 32 < L;
    uint8_t* prow = sP + row * 128;
    const unsigned long long sc2 = f2_pack(scale_log2, scale_log2);
    for (int j = 0; j < nkb; ++j) {
      const int nk = min(TKB64, L - j * TKB64);
      const int nch = (nk + 31) >> 5;
      if (!warp_active) {
        // rows all beyond L: nothing to compute, but s_free / p_full count 4 warps, and an arrival
        // lands in the barrier's current phase -- so arrive only once that phase is the block's own
        // (S_j issued implies s_free phase j-1 complete; PV_{j-1} complete implies p_full phase j-1)
        EWAIT(s_full, j & 1, 15, j);
        if (lane == 0) mbar_arrive(s_free);
        __syncwarp();  // reconverge before the next spin loop (the arriving lane must not be starved)
        if (j > 0) EWAIT(pv_done, (j - 1) & 1, 19, j);
        if (lane == 0) mbar_arrive(p_full);
        __syncwarp();
        continue;
      }
      {
        uint32_t r[2][32];
        EWAIT(s_full, j & 1, 5, j);
        tc_fence_after();
        tmem_ld_32x32b_x32(taddr, r[0]);
        if (nch > 1) tmem_ld_32x32b_x32(taddr + 32, r[1]);
        tc_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(s_free);  // S_j may now be overwritten by S_{j+1}
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c < nch && nk < 32 * (c + 1)) {
            const int tail = nk - 32 * c;
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e >= tail) r[c][e] = __float_as_uint(-INFINITY);
          }
        }
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = __uint_as_float(r[0][i]);
#pragma unroll
        for (int e = 8; e < 32; e += 2) mx[(e >> 1) & 7] = fmax3(mx[(e >> 1) & 7], __uint_as_float(r[0][e]), __uint_as_float(r[0][e + 1]));
        if (nch > 1) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) mx[(e >> 1) & 7] = fmax3(mx[(e >> 1) & 7], __uint_as_float(r[1][e]), __uint_as_float(r[1][e + 1]));
        }
        const float bm = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
        const float ms = bm * scale_log2;
        float alpha = 1.f;
        bool resc = false;
        if (j == 0) {
          m = ms;
        } else if (ms > m + kLazyRescale) {
          alpha = ex2_approx(m - ms);
          m = ms;
          l *= alpha;
          resc = true;
        }
        const unsigned long long nm2 = f2_pack(-m, -m);
        unsigned long long acc0 = f2_pack(0.f, 0.f), acc1 = acc0;
        uint32_t pk[2][16];  // P_j as 16-bit pairs
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c < nch) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float x0, x1, p0, p1;
              f2_unpack(f2_fma(f2_pack(__uint_as_float(r[c][2 * e]), __uint_as_float(r[c][2 * e + 1])), sc2, nm2), x0, x1);
              if (exp2_on_fma(e)) {
                f2_unpack(exp2_poly2(x0, x1), p0, p1);
              } else {
                p0 = ex2_approx(x0);
                p1 = ex2_approx(x1);
              }
              r[c][2 * e] = __float_as_uint(p0);
              r[c][2 * e + 1] = __float_as_uint(p1);
            }
            if (nk < 32 * (c + 1)) {
              const int tail = nk - 32 * c;
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (e >= tail) r[c][e] = 0u;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              acc0 = f2_add(acc0, f2_pack(__uint_as_float(r[c][4 * e]), __uint_as_float(r[c][4 * e + 1])));
              acc1 = f2_add(acc1, f2_pack(__uint_as_float(r[c][4 * e + 2]), __uint_as_float(r[c][4 * e + 3])));
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[c][e] = pack16x2<F16>(__uint_as_float(r[c][2 * e]), __uint_as_float(r[c][2 * e + 1]));
          }
        }
        float a0, a1, a2, a3;
        f2_unpack(acc0, a0, a1);
        f2_unpack(acc1, a2, a3);
        l += (a0 + a1) + (a2 + a3);
        // PV_{j-1} must have completed: it reads P_{j-1} (overwritten below) and accumulates into O
        if (j > 0) {
          EWAIT(pv_done, (j - 1) & 1, 29, j);
          tc_fence_after();
        }
        if (__any_sync(0xffffffffu, resc)) {  // warp-uniform (tcgen05.ld / st); alpha = 1 where !resc
          const unsigned long long al2 = f2_pack(alpha, alpha);
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(taddr + kOCol + x * 32, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float o0, o1;
              f2_unpack(f2_mul(f2_pack(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1])), al2), o0, o1);
              o[2 * i] = __float_as_uint(o0);
              o[2 * i + 1] = __float_as_uint(o1);
            }
            tmem_st_32x32b_x32(taddr + kOCol + x * 32, o);
          }
          tc_wait_st();
        }
        // P_j row -> shared memory: 16-byte chunk c of the 128-byte row at chunk c ^ (row & 7)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c < nch) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int chunk = 4 * c + q;
              *reinterpret_cast<uint4*>(prow + 16 * (chunk ^ (row & 7))) =
                  make_uint4(pk[c][4 * q], pk[c][4 * q + 1], pk[c][4 * q + 2], pk[c][4 * q + 3]);
            }
          }
        }
        fence_proxy_async_smem();  // generic-proxy P stores -> the MMA's async-proxy reads
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        __syncwarp();
      }
    }
  }
  // epilogue: ctx = O / l once the last PV has completed (every MMA has: sQ is free), rows staged in
  // sQ with 16-byte chunks XOR-swizzled by row, then written back 4 rows per warp instruction
  const int row = warp * 32 + lane;
  if (warp < 4 && q0 + warp * 32 < L) {
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    EWAIT(pv_done, (nkb - 1) & 1, 39, nkb);
    tc_fence_after();
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(taddr + kOCol + x * 32, v);
      tc_wait_ld();
      if constexpr (F8OUT) {
        const float inv = ctx_scale / l;
        uint4* srow = reinterpret_cast<uint4*>(sQ + row * TD);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const uint32_t* u = v + 16 * k;
          srow[(2 * x + k) ^ (row & 3)] = make_uint4(
              pack_e4m3x4(__uint_as_float(u[0]) * inv, __uint_as_float(u[1]) * inv, __uint_as_float(u[2]) * inv,
                          __uint_as_float(u[3]) * inv),
              pack_e4m3x4(__uint_as_float(u[4]) * inv, __uint_as_float(u[5]) * inv, __uint_as_float(u[6]) * inv,
                          __uint_as_float(u[7]) * inv),
              pack_e4m3x4(__uint_as_float(u[8]) * inv, __uint_as_float(u[9]) * inv, __uint_as_float(u[10]) * inv,
                          __uint_as_float(u[11]) * inv),
              pack_e4m3x4(__uint_as_float(u[12]) * inv, __uint_as_float(u[13]) * inv, __uint_as_float(u[14]) * inv,
                          __uint_as_float(u[15]) * inv));
        }
      } else {
        const float inv = 1.0f / l;
        uint4* srow = reinterpret_cast<uint4*>(sQ + row * (TD * 2));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t* u = v + 8 * k;
          srow[(4 * x + k) ^ (row & 7)] =
              make_uint4(pack16x2<F16>(__uint_as_float(u[0]) * inv, __uint_as_float(u[1]) * inv),
                         pack16x2<F16>(__uint_as_float(u[2]) * inv, __uint_as_float(u[3]) * inv),
                         pack16x2<F16>(__uint_as_float(u[4]) * inv, __uint_as_float(u[5]) * inv),
                         pack16x2<F16>(__uint_as_float(u[6]) * inv, __uint_as_float(u[7]) * inv));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
  if (warp < 4) {
    const int nrows = min(TQ, L - q0);
    if constexpr (F8OUT) {
      uint8_t* c8 = reinterpret_cast<uint8_t*>(ctx);
      const int c = lane & 3;
      for (int rr = warp * 8 + (lane >> 2); rr < nrows; rr += 32) {
        const uint4 v = reinterpret_cast<const uint4*>(sQ + rr * TD)[c ^ (rr & 3)];
        *reinterpret_cast<uint4*>(c8 + static_cast<size_t>(start + q0 + rr) * H + h * TD + c * 16) = v;
      }
    } else {
      const int c = lane & 7;
      for (int rr = warp * 4 + (lane >> 3); rr < nrows; rr += 16) {
        const uint4 v = reinterpret_cast<const uint4*>(sQ + rr * (TD * 2))[c ^ (rr & 7)];
        *reinterpret_cast<uint4*>(ctx + static_cast<size_t>(start + q0 + rr) * H + h * TD + c * 8) = v;
      }
    }
  }
}

struct AttnItem {
  int start, L, q0, h, nkb;
};
struct IssuerState {
  AttnItem cur, nxt;  // the items K / V loads may target
  AttnWork nn;        // the item after nxt, fetched one item early
  int gbase, nk, nv;  // global index of cur's block 0; K / V blocks issued so far
};
static_assert(8 * 8 + sizeof(IssuerState) + 2 * sizeof(AttnItem) <= 256, "persistent engine smem tail");
template <bool F8OUT, bool F16>
__global__ void __launch_bounds__(128, 4)
    k_attention_tc64p(const __grid_constant__ CUtensorMap tm, const AttnWork* __restrict__ work,
                      const int32_t* __restrict__ num_work, int H, int nh, uint16_t* __restrict__ ctx,
                      float scale_log2, int Tp, float ctx_scale) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* sQ = smem;                      // 128 rows
  uint8_t* sK = sQ + kBlkBytes;            // [2][64 rows]
  uint8_t* sV = sK + 2 * kBlk64;           // [2][64 rows]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * kBlk64);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;             // [2]
  uint64_t* v_full = bars + 3;             // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* o_full = bars + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 7);
  const int warp = warp_id(), lane = lane_id();
  const bool issuer = threadIdx.x == 0;
  if (issuer) {
    tma_prefetch_desc(&tm);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&v_full[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<128>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  const int row = warp * 32 + lane;
  constexpr uint32_t idesc_s = F16 ? make_idesc_f16_f32(TQ, TKB64) : make_idesc_bf16_f32(TQ, TKB64);
  constexpr uint32_t idesc_o = (F16 ? make_idesc_f16_f32(TQ, TD) : make_idesc_bf16_f32(TQ, TD)) | (1u << 16);
  const uint64_t dq = make_sw128_desc(smem_u32(sQ));

  pdl_wait();  // the work list and the qkv planes come from earlier kernels (common.cuh)
  pdl_trigger();
  const int total = __ldg(num_work) * nh;  // (work item, head) pairs
  const int G = static_cast<int>(gridDim.x);
  // The issuer's look-ahead state lives in shared memory (thread 0 only), so that it is not live
  // in registers across the softmax; every thread reads the next item from islot[] at the item
  // boundary (written by thread 0 before the item's first block barrier).
  IssuerState* ist = reinterpret_cast<IssuerState*>(bars + 8);
  AttnItem* islot = reinterpret_cast<AttnItem*>(ist + 1);  // [2]: item k in slot k & 1
  auto decode = [&](int i, const AttnWork& w) -> AttnItem {
    if (i >= total) return AttnItem{0, 0, 0, 0, 0};
    return AttnItem{w.start, w.len, w.q0, i % nh, (w.len + TKB64 - 1) / TKB64};
  };
  auto fetch = [&](int i) -> AttnWork { return i < total ? work[i / nh] : AttnWork{0, 0, 0, 0}; };
  int it = static_cast<int>(blockIdx.x);
  AttnItem cur = decode(it, fetch(it));
  uint32_t items_done = 0;
  int g = 0;  // global block index over the CTA's sequence
  // at "S_g complete" (g = -1 before the first S): K up to g + 2, V up to g + 1, over cur and nxt
  auto issue_loads = [&](int g) {
    const AttnItem c = ist->cur, n = ist->nxt;
    const int gb = ist->gbase;
    auto blk_row = [&](int mb, int plane, int& r) -> bool {
      int rel = mb - gb;
      if (rel < c.nkb) {
        r = (plane * nh + c.h) * Tp + c.start + rel * TKB64;
        return true;
      }
      rel -= c.nkb;
      if (rel < n.nkb) {
        r = (plane * nh + n.h) * Tp + n.start + rel * TKB64;
        return true;
      }
      return false;
    };
    int r, nk = ist->nk, nv = ist->nv;
    while (nk <= g + 2 && blk_row(nk, 1, r)) {
      mbar_arrive_expect_tx(&k_full[nk & 1], kBlk64);
      tma_load_2d(sK + (nk & 1) * kBlk64, &tm, &k_full[nk & 1], 0, r);
      ++nk;
    }
    while (nv <= g + 1 && blk_row(nv, 2, r)) {
      mbar_arrive_expect_tx(&v_full[nv & 1], kBlk64);
      tma_load_2d(sV + (nv & 1) * kBlk64, &tm, &v_full[nv & 1], 0, r);
      ++nv;
    }
    ist->nk = nk;
    ist->nv = nv;
  };
  auto load_q = [&](const AttnItem& x) {
    const int r = x.h * Tp + x.start + x.q0;
    mbar_arrive_expect_tx(q_full, kBlkBytes);
    tma_load_2d(sQ, &tm, q_full, 0, r);
    tma_load_2d(sQ + kBlk64, &tm, q_full, 0, r + 64);
  };
  auto issue_s = [&](int gnext) {  // S_gnext = Q K_gnext^T into columns [0, 64)
    const int b = gnext & 1;
    PWAIT(&k_full[b], (gnext >> 1) & 1, 1);
    tc_fence_after();
    const uint64_t dk = make_sw128_desc(smem_u32(sK + b * kBlk64));
#pragma unroll
    for (int k = 0; k < TD / 16; ++k) tc_mma_f16(tmem, dq + 2 * k, dk + 2 * k, idesc_s, k > 0);
    tc_commit(s_full);
  };
  if (issuer) {
    ist->cur = cur;
    ist->nxt = decode(it + G, fetch(it + G));
    ist->nn = fetch(it + 2 * G);
    ist->gbase = 0;
    ist->nk = 0;
    ist->nv = 0;
    if (cur.nkb > 0) {
      load_q(cur);
      issue_loads(-1);
      PWAIT(q_full, 0, 0);
      issue_s(0);
    }
  }

  const unsigned long long sc2 = f2_pack(scale_log2, scale_log2);
  while (it < total) {
    const int L = cur.L, q0 = cur.q0, nkb = cur.nkb;
    const bool warp_active = q0 + warp * 32 < L;
    float m = 0.f, l = 0.f;
    for (int j = 0; j < nkb; ++j, ++g) {
      PWAIT(s_full, g & 1, 5);
      tc_fence_after();
      if (issuer) {
        if (j == 0) islot[(items_done + 1) & 1] = ist->nxt;  // read by every thread at the item boundary
        if (j == nkb - 1 && ist->nxt.nkb > 0) load_q(ist->nxt);  // the last S of this item has read Q
        issue_loads(g);
      }
      const int nk = min(TKB64, L - j * TKB64);
      const int nch = (nk + 31) >> 5;
      if (warp_active) {
        uint32_t r[2][32];
        tmem_ld_32x32b_x32(taddr, r[0]);
        if (nch > 1) tmem_ld_32x32b_x32(taddr + 32, r[1]);
        tc_wait_ld();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c < nch && nk < 32 * (c + 1)) {
            const int tail = nk - 32 * c;
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (e >= tail) r[c][e] = __float_as_uint(-INFINITY);
          }
        }
        float mx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = __uint_as_float(r[0][i]);
#pragma unroll
        for (int e = 8; e < 32; e += 2) mx[(e >> 1) & 7] = fmax3(mx[(e >> 1) & 7], __uint_as_float(r[0][e]), __uint_as_float(r[0][e + 1]));
        if (nch > 1) {
#pragma unroll
          for (int e = 0; e < 32; e += 2) mx[(e >> 1) & 7] = fmax3(mx[(e >> 1) & 7], __uint_as_float(r[1][e]), __uint_as_float(r[1][e + 1]));
        }
        const float bm = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
        const float ms = bm * scale_log2;
        float alpha = 1.f;
        bool resc = false;
        if (j == 0) {
          m = ms;
        } else if (ms > m + kLazyRescale) {
          alpha = ex2_approx(m - ms);
          m = ms;
          l *= alpha;
          resc = true;
        }
        const unsigned long long nm2 = f2_pack(-m, -m);
        unsigned long long acc0 = f2_pack(0.f, 0.f), acc1 = acc0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          if (c < nch) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              float x0, x1, p0, p1;
              f2_unpack(f2_fma(f2_pack(__uint_as_float(r[c][2 * e]), __uint_as_float(r[c][2 * e + 1])), sc2, nm2), x0, x1);
              if (exp2_on_fma(e)) {
                f2_unpack(exp2_poly2(x0, x1), p0, p1);
              } else {
                p0 = ex2_approx(x0);
                p1 = ex2_approx(x1);
              }
              r[c][2 * e] = __float_as_uint(p0);
              r[c][2 * e + 1] = __float_as_uint(p1);
            }
            if (nk < 32 * (c + 1)) {
              const int tail = nk - 32 * c;
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if (e >= tail) r[c][e] = 0u;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              acc0 = f2_add(acc0, f2_pack(__uint_as_float(r[c][4 * e]), __uint_as_float(r[c][4 * e + 1])));
              acc1 = f2_add(acc1, f2_pack(__uint_as_float(r[c][4 * e + 2]), __uint_as_float(r[c][4 * e + 3])));
            }
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[e] = pack16x2<F16>(__uint_as_float(r[c][2 * e]), __uint_as_float(r[c][2 * e + 1]));
            tmem_st_32x32b_x16(taddr + c * 16, pk);
          }
        }
        float a0, a1, a2, a3;
        f2_unpack(acc0, a0, a1);
        f2_unpack(acc1, a2, a3);
        l += (a0 + a1) + (a2 + a3);
        if (__any_sync(0xffffffffu, resc)) {  // warp-uniform (tcgen05.ld / st); alpha = 1 where !resc
          const unsigned long long al2 = f2_pack(alpha, alpha);
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(taddr + kOCol + x * 32, o);
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float o0, o1;
              f2_unpack(f2_mul(f2_pack(__uint_as_float(o[2 * i]), __uint_as_float(o[2 * i + 1])), al2), o0, o1);
              o[2 * i] = __float_as_uint(o0);
              o[2 * i + 1] = __float_as_uint(o1);
            }
            tmem_st_32x32b_x32(taddr + kOCol + x * 32, o);
          }
        }
        tc_wait_st();
      }
      tc_fence_before();
      __syncthreads();  // P_g complete in TMEM (all 128 rows); the previous item's O has been read
      if (issuer) {
        tc_fence_after();
        const int b = g & 1;
        PWAIT(&v_full[b], (g >> 1) & 1, 3);
        const int nks = (nk + 15) / 16;
        for (int ks = 0; ks < nks; ++ks) {
          const uint64_t dv = make_sw128_desc(smem_u32(sV + b * kBlk64 + ks * (16 * TD * 2)));
          tc_mma_f16_tmem_a(tmem + kOCol, tmem + ks * 8, dv, idesc_o, (j | ks) != 0 ? 1u : 0u);
        }
        if (j + 1 < nkb) {
          issue_s(g + 1);
        } else {
          tc_commit(o_full);
          if (ist->nxt.nkb > 0) {  // the next item's first S runs under this item's epilogue
            PWAIT(q_full, (items_done + 1) & 1, 10);
            issue_s(g + 1);
          }
        }
      }
    }
    PWAIT(o_full, items_done & 1, 6);
    tc_fence_after();
    // epilogue: ctx = O / l, one row per thread straight from registers
    if (warp_active) {  // tcgen05.ld is warp-collective: whole warps load, rows < L store
      const bool store = q0 + row < L;
      const int h = cur.h;
      const size_t grow = static_cast<size_t>(cur.start + q0 + row);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(taddr + kOCol + x * 32, v);
        tc_wait_ld();
        if constexpr (F8OUT) {
          const float inv = ctx_scale / l;
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(ctx) + grow * H + h * TD + x * 32);
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const uint32_t* u = v + 16 * k;
            if (store) dst[k] = make_uint4(
                pack_e4m3x4(__uint_as_float(u[0]) * inv, __uint_as_float(u[1]) * inv, __uint_as_float(u[2]) * inv,
                            __uint_as_float(u[3]) * inv),
                pack_e4m3x4(__uint_as_float(u[4]) * inv, __uint_as_float(u[5]) * inv, __uint_as_float(u[6]) * inv,
                            __uint_as_float(u[7]) * inv),
                pack_e4m3x4(__uint_as_float(u[8]) * inv, __uint_as_float(u[9]) * inv, __uint_as_float(u[10]) * inv,
                            __uint_as_float(u[11]) * inv),
                pack_e4m3x4(__uint_as_float(u[12]) * inv, __uint_as_float(u[13]) * inv, __uint_as_float(u[14]) * inv,
                            __uint_as_float(u[15]) * inv));
          }
        } else {
          const float inv = 1.0f / l;
          uint4* dst = reinterpret_cast<uint4*>(ctx + grow * H + h * TD + x * 32);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t* u = v + 8 * k;
            if (store) dst[k] = make_uint4(pack16x2<F16>(__uint_as_float(u[0]) * inv, __uint_as_float(u[1]) * inv),
                                pack16x2<F16>(__uint_as_float(u[2]) * inv, __uint_as_float(u[3]) * inv),
                                pack16x2<F16>(__uint_as_float(u[4]) * inv, __uint_as_float(u[5]) * inv),
                                pack16x2<F16>(__uint_as_float(u[6]) * inv, __uint_as_float(u[7]) * inv));
          }
        }
      }
    }
    it += G;
    if (issuer) {  // advance the look-ahead: cur <- nxt <- nn
      ist->gbase += nkb;
      ist->cur = ist->nxt;
      ist->nxt = decode(it + G, ist->nn);
      ist->nn = fetch(it + 2 * G);
    }
    cur = islot[(items_done + 1) & 1];
    ++items_done;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

// ============================================================================ CLS-only last layer
// with CLS pooling only row 0 of each request leaves the
// last encoder layer, so its attention needs one query row per (request, head) against the
// request's L keys.  One 128-thread CTA per (head, request), fp32 throughout:
//   s_j = q . k_j * log2(e) / sqrt(d)   (thread j mod 128 takes keys j, j + 128, ...)
//   p_j = exp2(s_j - max s),  l = sum p_j
//   ctx = sum_j p_j v_j / l            (thread t: column t mod 64, keys of parity t / 64)
// Head 0's CTA also gathers the request's CLS residual row h32[cu_i] into the compact hres.
// OUT: 0 bf16, 1 fp16, 2 E4M3(ctx_scale * ctx).
template <int OUT>
__global__ void __launch_bounds__(128) k_attention_cls(const uint16_t* __restrict__ qkv, const int32_t* __restrict__ cu,
                                                       int nh, int Tp, int H, float scale_log2,
                                                       const float* __restrict__ h32, uint16_t* __restrict__ ctx_c,
                                                       float* __restrict__ hres_c, float ctx_scale,
                                                       const uint32_t* __restrict__ err,
                                                       const int32_t* __restrict__ dims) {
  if (err && *err) return;  // invalid lengths (sticky error): cu may point past the planes
  const int h = blockIdx.x, i = blockIdx.y;
  if (i >= dev_n(dims, static_cast<int>(gridDim.y))) return;
  const int start = __ldg(cu + i), L = __ldg(cu + i + 1) - start;
  __shared__ float q[TD];
  __shared__ float p[512];
  __shared__ float red[8];
  __shared__ float part[2][TD];
  auto to_f = [](uint16_t b) {
    if constexpr (OUT == 1) return __half2float(__ushort_as_half(b));
    else return bf16_bits_to_f32(b);
  };
  const uint16_t* Q = qkv + (static_cast<size_t>(h) * Tp + start) * TD;
  const uint16_t* K = qkv + (static_cast<size_t>(nh + h) * Tp + start) * TD;
  const uint16_t* V = qkv + (static_cast<size_t>(2 * nh + h) * Tp + start) * TD;
  const int t = threadIdx.x;
  if (t < TD) q[t] = to_f(Q[t]);
  if (h == 0)
    for (int c = t; c < H; c += blockDim.x) hres_c[static_cast<size_t>(i) * H + c] = h32[static_cast<size_t>(start) * H + c];
  __syncthreads();
  float mx = -INFINITY;
  for (int j = t; j < L; j += blockDim.x) {
    const uint4* kr = reinterpret_cast<const uint4*>(K + static_cast<size_t>(j) * TD);
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < TD / 8; ++c) {
      const uint4 v = __ldg(kr + c);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc = fmaf(q[8 * c + 2 * e], to_f(static_cast<uint16_t>(w[e] & 0xFFFFu)), acc);
        acc = fmaf(q[8 * c + 2 * e + 1], to_f(static_cast<uint16_t>(w[e] >> 16)), acc);
      }
    }
    p[j] = acc * scale_log2;
    mx = fmaxf(mx, p[j]);
  }
  mx = warp_max(mx);
  if (lane_id() == 0) red[warp_id()] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  float sum = 0.f;
  for (int j = t; j < L; j += blockDim.x) {
    const float e = exp2f(p[j] - mx);
    p[j] = e;
    sum += e;
  }
  sum = warp_sum(sum);
  if (lane_id() == 0) red[4 + warp_id()] = sum;
  __syncthreads();
  const float l = (red[4] + red[5]) + (red[6] + red[7]);
  const int col = t & (TD - 1), par = t >> 6;
  float acc = 0.f;
  for (int j = par; j < L; j += 2) acc = fmaf(p[j], to_f(V[static_cast<size_t>(j) * TD + col]), acc);
  part[par][col] = acc;
  __syncthreads();
  if (t < TD) {
    const float o = (part[0][t] + part[1][t]) / l;
    const size_t dst = static_cast<size_t>(i) * H + h * TD + t;
    if constexpr (OUT == 2) {
      __shared__ float ob[TD];
      ob[t] = o * ctx_scale;
      __syncwarp();
      if ((t & 3) == 0) {
        // 4 E4M3 bytes per thread (t, t+1, t+2, t+3 of this warp)
        reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(ctx_c) + static_cast<size_t>(i) * H + h * TD)[t >> 2] =
            pack_e4m3x4(ob[t], ob[t + 1], ob[t + 2], ob[t + 3]);
      }
    } else if constexpr (OUT == 1) {
      ctx_c[dst] = __half_as_ushort(__float2half_rn(o));
    } else {
      ctx_c[dst] = static_cast<uint16_t>(pack_bf16x2(o, 0.f) & 0xFFFFu);
    }
  }
}

}  // namespace

bool make_tmap_qkv64(CUtensorMap* m, const void* qkv, uint64_t rows, int H) {
  return make_tmap_bf16_box(m, qkv, rows * static_cast<uint64_t>(3 * (H / 64)), 64, 64, 64);
}

bool make_tmap_qkv(CUtensorMap* m, const void* qkv, uint64_t rows, int H) {
  // 64 bf16 = 128 B inner box (one SWIZZLE_128B row), 128 rows
  // head-major planes [3 * nh][rows][64] viewed as one [3 * nh * rows, 64] matrix: 128-token boxes of one
  // head's Q, K or V are contiguous 16 KB blocks (64 bf16 = one SWIZZLE_128B row)
  return make_tmap_bf16_box(m, qkv, rows * static_cast<uint64_t>(3 * (H / 64)), 64, 64, 128);
}

cudaError_t launch_attention(const uint16_t* qkv, const CUtensorMap* tm_qkv, const int32_t* cu_seqlens,
                             const AttnWork* work, const int32_t* num_work, int64_t T, int n, int H, int num_heads,
                             int64_t plane_rows, uint16_t* ctx, float ctx_f8_scale, bool f16, cudaStream_t st,
                             const CUtensorMap* tm_qkv64) {
  if (T <= 0 || n <= 0) return cudaSuccess;
  const int d = H / num_heads;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(d));
  const int64_t max_tiles = attn_max_tiles(T, n, attn_tile_q(d));
  const unsigned grid = static_cast<unsigned>(max_tiles * num_heads);
  if (d == 64) {
    if (!tm_qkv) return cudaErrorInvalidValue;
    if (f16 && ctx_f8_scale > 0.f) return cudaErrorInvalidValue;
    static const int engine = getenv("ELIS_ATTN_ENGINE") ? atoi(getenv("ELIS_ATTN_ENGINE")) : 64;
    if (engine == 65 && tm_qkv64) {  // persistent 64-key engine: 4 CTAs per SM loop over the items
      auto kern = f16 ? k_attention_tc64p<false, true> : ctx_f8_scale > 0.f ? k_attention_tc64p<true, false>
                                                                            : k_attention_tc64p<false, false>;
      if (!attr_once(reinterpret_cast<const void*>(kern))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttn64Smem);
        if (e != cudaSuccess) return e;
      }
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const unsigned pgrid = std::min<unsigned>(grid, 4u * static_cast<unsigned>(sms));
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(pgrid);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = kAttn64Smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      pdl_attr(attr[0]);
      cfg.attrs = attr;
      cfg.numAttrs = pdl_enabled() ? 1 : 0;
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, *tm_qkv64, work, num_work, H, num_heads, ctx, scale_log2,
                                         static_cast<int>(plane_rows), ctx_f8_scale);
      if (e != cudaSuccess) return e;
      return cudaGetLastError();
    }
    if (engine == 66 && tm_qkv64) {  // early-S 64-key engine: P in shared memory, issuer warp
      auto kern = f16 ? k_attention_tc64e<false, true> : ctx_f8_scale > 0.f ? k_attention_tc64e<true, false>
                                                                            : k_attention_tc64e<false, false>;
      if (!attr_once(reinterpret_cast<const void*>(kern))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnESmem);
        if (e != cudaSuccess) return e;
      }
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(160);
      cfg.dynamicSmemBytes = kAttnESmem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      pdl_attr(attr[0]);
      cfg.attrs = attr;
      cfg.numAttrs = pdl_enabled() ? 1 : 0;
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, *tm_qkv64, work, num_work, H, num_heads, ctx, scale_log2,
                                         static_cast<int>(plane_rows), ctx_f8_scale);
      if (e != cudaSuccess) return e;
      return cudaGetLastError();
    }
    if (engine == 64 && tm_qkv64) {  // 64-key blocks, O in TMEM
      auto kern = f16 ? k_attention_tc64<false, true> : ctx_f8_scale > 0.f ? k_attention_tc64<true, false>
                                                                           : k_attention_tc64<false, false>;
      if (!attr_once(reinterpret_cast<const void*>(kern))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttn64Smem);
        if (e != cudaSuccess) return e;
      }
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = kAttn64Smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      pdl_attr(attr[0]);
      cfg.attrs = attr;
      cfg.numAttrs = pdl_enabled() ? 1 : 0;
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, *tm_qkv64, work, num_work, H, num_heads, ctx, scale_log2,
                                         static_cast<int>(plane_rows), ctx_f8_scale);
      if (e != cudaSuccess) return e;
      return cudaGetLastError();
    }
    auto kern = f16 ? k_attention_tc<false, true> : ctx_f8_scale > 0.f ? k_attention_tc<true, false>
                                                                       : k_attention_tc<false, false>;
    if (!attr_once(reinterpret_cast<const void*>(kern))) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnTcSmem);
      if (e != cudaSuccess) return e;
    }
    kern<<<grid, 128, kAttnTcSmem, st>>>(*tm_qkv, work, num_work, H, num_heads, ctx, scale_log2,
                                         static_cast<int>(plane_rows), ctx_f8_scale);
  } else if (d == 32) {
    if (ctx_f8_scale > 0.f || f16) return cudaErrorInvalidValue;
    k_attention<32><<<grid, 128, 0, st>>>(qkv, cu_seqlens, work, num_work, H, num_heads, ctx, scale_log2);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_attention_cls(const uint16_t* qkv, const int32_t* cu_seqlens, int n, int H, int num_heads,
                                 int64_t plane_rows, const float* h32, uint16_t* ctx_c, float* hres_c, int out_kind,
                                 float ctx_scale, const uint32_t* err, cudaStream_t st, const int32_t* dims) {
  if (n <= 0) return cudaSuccess;
  if (H / num_heads != TD) return cudaErrorInvalidValue;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(TD));
  const dim3 grid(num_heads, n);
  const int Tp = static_cast<int>(plane_rows);
  switch (out_kind) {
    case 0: k_attention_cls<0><<<grid, 128, 0, st>>>(qkv, cu_seqlens, num_heads, Tp, H, scale_log2, h32, ctx_c, hres_c, ctx_scale, err, dims); break;
    case 1: k_attention_cls<1><<<grid, 128, 0, st>>>(qkv, cu_seqlens, num_heads, Tp, H, scale_log2, h32, ctx_c, hres_c, ctx_scale, err, dims); break;
    case 2: k_attention_cls<2><<<grid, 128, 0, st>>>(qkv, cu_seqlens, num_heads, Tp, H, scale_log2, h32, ctx_c, hres_c, ctx_scale, err, dims); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

#ifdef ELIS_ATTN_TRACE
extern "C" int elis_debug_attn_trace(unsigned long long* host, size_t n, int reset) {
  if (reset) return static_cast<int>(cudaMemset(g_attn_trace_ptr(), 0, sizeof(g_attn_trace)));
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_attn_trace, std::min(n, kTraceCap * 8) * 8));
}
#endif

}  // namespace elis
