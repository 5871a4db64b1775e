// attention.cu -- fused varlen bidirectional multi-head attention.
//
// For every request i and head h (BERT self-attention,
// P:42 "process tokens in parallel"):
//     ctx_h = softmax(Q_h K_h^T / sqrt(d)) V_h   over the request's own L_i tokens,
// no causal mask, no cross-request attention, no padding: the work list (k_meta) holds the
// q tiles of the long requests and packs of short ones, so ragged lengths cost at most one
// partial 32-row segment per request.
//
// Head dim 64 (BGE-base / large): the persistent tcgen05 engine below.  Head dim 32 (the tiny
// test encoder): flash-style online softmax on mma.sync m16n8k16 (fp32 statistics, exp2 with
// the log2(e)/sqrt(d) scale folded in, P rounded to bf16 for the PV product), 64-row tiles.

#include <algorithm>

#include "common.cuh"
#include "kernels.cuh"

namespace elis {

#ifdef ELIS_ATTN_TRACE
// Diagnostic build only (python -m paper_2505_09142_b200.build --variant=atrace -DELIS_ATTN_TRACE):
// %globaltimer stamps of the persistent engine's phases, per pipeline (CTA, pp): event code in the
// low 8 bits (scripts/attn_trace.py decodes them).
constexpr int kTrPipes = 512, kTrEvents = 2048;
__device__ unsigned long long g_attn_trace[kTrPipes * kTrEvents];
__device__ unsigned g_attn_trace_n[kTrPipes * 4];
// the stamping thread keeps its event count in a register (a global counter's load would add an
// L2 round trip to every stamp); the counts are stored once at the end
ELIS_DEV void attn_tr(int pipe, int role, unsigned code, unsigned& k) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (pipe < kTrPipes && k < kTrEvents / 4) g_attn_trace[pipe * kTrEvents + role * (kTrEvents / 4) + k] = (t << 8) | code;
  ++k;
}
#define ATR(role, code) attn_tr(2 * static_cast<int>(blockIdx.x) + pp, role, code, tr_k)
#define ATR_DONE(role) \
  do { if (2 * static_cast<int>(blockIdx.x) + pp < kTrPipes) g_attn_trace_n[(2 * blockIdx.x + pp) * 4 + (role)] = tr_k; } while (0)
extern "C" int elis_debug_attn_trace(unsigned long long* host, unsigned* counts, int reset) {
  if (reset) {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, g_attn_trace_n);
    return static_cast<int>(cudaMemset(p, 0, sizeof(g_attn_trace_n)));
  }
  cudaError_t e = cudaMemcpyFromSymbol(host, g_attn_trace, sizeof(g_attn_trace));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(counts, g_attn_trace_n, sizeof(g_attn_trace_n));
  return static_cast<int>(e);
}
#else
#define ATR(role, code) do { } while (0)
#define ATR_DONE(role) do { } while (0)
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
  const int start = w.start[0], L = w.len[0], q0 = w.q0;
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
// Persistent, warp-specialised; one CTA per SM running two independent pipelines, each:
//   TMA warp   producer: a work item's Q rows (double-buffered slot) and its K and V key blocks
//              (2-stage rings each) as 32-row boxes from the head-major qkv planes the QKV GEMM
//              writes ([3 nh][T][64]: plane h = Q of head h, nh + h = K, 2 nh + h = V);
//   MMA warp   issuer (one thread), in the order S_0, S_1, PV_0, S_2, PV_1, ... over the
//              pipeline's blocks (across items):  S_g = Q K_g^T (tcgen05 M 128 x N 128 x K 64,
//              TMEM columns [0, 128)) as soon as the softmax has read S_{g-1} into registers;
//              O += P_g V_g (A = P_g from TMEM columns [128, 192), B = V_g MN-major from shared
//              memory, accumulator in columns [192, 256)) once the softmax has written P_g;
//   4 warps    softmax + epilogue, thread = query row = TMEM lane: a block's scores are read once
//              into registers (then S is released to the next block's MMA), block max, exp2 (part
//              on the FMA pipe), row sum, P packed to 16 bits into the P columns once the previous
//              PV has read them; O stays in TMEM across key blocks and is rescaled only when the
//              running max grows by more than 2^8 (lazy rescale: P <= 256); after the last block
//              ctx = O / l is staged in the item's Q slot and written back 4 rows per instruction.
// So the next block's S (and the next item's first S) is computed while the softmax of the
// current one runs, and the loads run up to two blocks ahead; the other pipeline overlaps its own
// chain with this one (TMEM 2 x 256 columns, shared memory 2 x 96 KB).  Registers: the launch
// gives 168 per thread; setmaxnreg moves them from the control warpgroup (40) to the two softmax
// warpgroups (232 each: a block's 128 scores per row held in registers).
// Short requests (<= 128 tokens) arrive packed (AttnWork): request k owns 32-row segments
// [f_k, f_k + ceil(L_k / 32)) of the tile -- one softmax warp per segment -- and attends only to
// its own key segments (block-diagonal mask; P is zero elsewhere), so a request costs
// ceil(L / 32) x 32 rows instead of a 128-row tile.  Its arithmetic is independent of f_k: the
// same 32-key chunks in the same order, the PV MMA's 16-key steps hold keys of one request only
// and the other steps add exact zeros (batch invariance).
constexpr int TQ = 128;        // q rows per tile (= TMEM lanes)
constexpr int TKB = 128;       // keys per block
constexpr int TD = 64;         // head dim
constexpr int kBoxRows = 32;   // TMA box: 32 rows x 64 columns (one 128-byte SWIZZLE_128B row each)
constexpr int kBoxBytes = kBoxRows * TD * 2;  // 4 KB
constexpr int kBlkBytes = TKB * TD * 2;       // 16 KB
constexpr int kAwsKV = 2;                     // K/V ring stages (K + V per stage)
// warps 0-3: TMA producer / MMA issuer of pipelines 0 and 1; warps 4-7 / 8-11: softmax of pipeline 0 / 1
constexpr int kAwsThreads = 384;
constexpr uint32_t kAwsRegsCtl = 40, kAwsRegsSoftmax = 232;  // 128 x 40 + 256 x 232 = 384 x 168 registers
constexpr int kPipeSmem = 2 * kBlkBytes + kAwsKV * 2 * kBlkBytes;  // Q slots + K and V rings: 96 KB
constexpr int kAttnTcSmem = 2 * kPipeSmem + 1024 + 512;
constexpr uint32_t kPCol = 128;               // P (16-bit pairs): TMEM columns [128, 192)
constexpr uint32_t kOCol = 192;               // O accumulator: TMEM columns [192, 256)
constexpr float kLazyRescale = 8.f;           // log2 units
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
// (16 ex2 / clk / SM, measured: scripts/tmem_bw.cu):
//   j = rint(x) (x + 1.5 * 2^23 leaves j in the low mantissa bits), f = x - j in [-1/2, 1/2],
//   2^f = degree-3 minimax polynomial (max relative error 7.5e-5, scripts/fit_exp2.py; P is then
//   rounded to 16 bits), 2^x = bits(2^f) + (j << 23).
// x is clamped at -125 so the exponent stays normal (the true value is then < 2^-125 next to the
// row maximum's >= 1).
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

ELIS_DEV AttnWork load_work(const AttnWork* w) {
  const int4 a = __ldg(reinterpret_cast<const int4*>(w));
  const int4 b = __ldg(reinterpret_cast<const int4*>(w) + 1);
  AttnWork r;
  *reinterpret_cast<int4*>(&r) = a;
  *(reinterpret_cast<int4*>(&r) + 1) = b;
  return r;
}
ELIS_DEV bool tile_packed(const AttnWork& w) { return w.len[0] <= TKB; }
ELIS_DEV int tile_nkb(const AttnWork& w) { return tile_packed(w) ? 1 : (w.len[0] + TKB - 1) / TKB; }
ELIS_DEV int ceil32(int x) { return (x + 31) >> 5; }
// keys of block j the PV product runs over (the last request's end, for a packed tile)
ELIS_DEV int tile_key_hi(const AttnWork& w, int j) {
  if (!tile_packed(w)) return min(TKB, w.len[0] - TKB * j);
  int f = 0, hi = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < w.nreq) { hi = 32 * f + w.len[k]; f += ceil32(w.len[k]); }
  return hi;
}
// one softmax warp's share of a tile: query rows 32 q .. 32 q + 31 of the tile
struct WarpRows {
  bool active;
  int tok;    // token of row 32 q
  int rows;   // valid rows (1..32)
  int ch0;    // first key chunk (32 keys) of the warp's keys within a block
  int klen;   // packed: the request's length (its keys); long: the request length L
};
ELIS_DEV WarpRows warp_rows(const AttnWork& w, int q) {
  WarpRows r{false, 0, 0, 0, 0};
  if (tile_packed(w)) {
    int f = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < w.nreq) {
        const int sg = ceil32(w.len[k]);
        if (q >= f && q < f + sg) {
          r.active = true;
          r.tok = w.start[k] + 32 * (q - f);
          r.rows = min(32, w.len[k] - 32 * (q - f));
          r.ch0 = f;
          r.klen = w.len[k];
        }
        f += sg;
      }
    }
  } else {
    const int L = w.len[0], q0 = w.q0 + 32 * q;
    r.active = q0 < L;
    r.tok = w.start[0] + q0;
    r.rows = min(32, L - q0);
    r.ch0 = 0;
    r.klen = L;
  }
  return r;
}

// One key block's softmax for one warp's 32 rows (thread = row), NCH = 32-key chunks holding the
// row's nk valid keys from chunk ch0 of the block; straight-line code per NCH.  S is read once into
// registers, then `release` (the S columns may be overwritten by the next S MMA) runs; block max;
// lazy running max (j > 0: it moves only when the block's exceeds it by more than 2^8);
// p = exp2(s scale - m) (part on the FMA pipe); row sum in a fixed order; then `before_p` (the
// previous PV has read the P columns; O rescaled if needed) runs and P is packed to 16 bits into
// the P columns (chunk c at 16 (ch0 + c)).  Returns the block's row sum.
template <int NCH, bool F16, class Release, class BeforeP>
ELIS_DEV float softmax_block(uint32_t taddr, int ch0, int nk, int j, float scale_log2, float& m, bool& resc,
                             float& alpha, Release&& release, BeforeP&& before_p) {
  uint32_t r[NCH][32];
#pragma unroll
  for (int c = 0; c < NCH; ++c) tmem_ld_32x32b_x32(taddr + (ch0 + c) * 32, r[c]);
  tc_wait_ld();
  release();
  const int tail = nk - 32 * (NCH - 1);  // valid keys of the last chunk (1..32)
  if (tail < 32) {
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (e >= tail) r[NCH - 1][e] = __float_as_uint(-INFINITY);
  }
  float mx[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) mx[i] = __uint_as_float(r[0][i]);
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int e = (c == 0 ? 8 : 0); e < 32; e += 2) {
      const int i = (e >> 1) & 7;
      mx[i] = fmax3(mx[i], __uint_as_float(r[c][e]), __uint_as_float(r[c][e + 1]));
    }
  const float bm = fmaxf(fmax3(mx[0], mx[1], mx[2]), fmax3(fmax3(mx[3], mx[4], mx[5]), mx[6], mx[7]));
  const float ms = bm * scale_log2;  // finite: every block has >= 1 valid key
  alpha = 1.f;
  resc = false;
  if (j == 0) {
    m = ms;
  } else if (ms > m + kLazyRescale) {
    alpha = ex2_approx(m - ms);
    m = ms;
    resc = true;
  }
  const unsigned long long sc2 = f2_pack(scale_log2, scale_log2);
  const unsigned long long nm2 = f2_pack(-m, -m);
#pragma unroll
  for (int e = 0; e < 16; ++e) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
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
  }
  float bsum = 0.f;
  uint32_t pk[NCH][16];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    unsigned long long a0 = f2_pack(__uint_as_float(r[c][0]), __uint_as_float(r[c][1]));
    unsigned long long a1 = f2_pack(__uint_as_float(r[c][2]), __uint_as_float(r[c][3]));
    unsigned long long a2 = f2_pack(__uint_as_float(r[c][4]), __uint_as_float(r[c][5]));
    unsigned long long a3 = f2_pack(__uint_as_float(r[c][6]), __uint_as_float(r[c][7]));
#pragma unroll
    for (int e = 8; e < 32; e += 8) {
      a0 = f2_add(a0, f2_pack(__uint_as_float(r[c][e]), __uint_as_float(r[c][e + 1])));
      a1 = f2_add(a1, f2_pack(__uint_as_float(r[c][e + 2]), __uint_as_float(r[c][e + 3])));
      a2 = f2_add(a2, f2_pack(__uint_as_float(r[c][e + 4]), __uint_as_float(r[c][e + 5])));
      a3 = f2_add(a3, f2_pack(__uint_as_float(r[c][e + 6]), __uint_as_float(r[c][e + 7])));
    }
    float s0, s1, s2, s3;
    f2_unpack(f2_add(a0, a1), s0, s1);
    f2_unpack(f2_add(a2, a3), s2, s3);
    bsum += (s0 + s1) + (s2 + s3);
#pragma unroll
    for (int e = 0; e < 16; ++e) pk[c][e] = pack16x2<F16>(__uint_as_float(r[c][2 * e]), __uint_as_float(r[c][2 * e + 1]));
  }
  before_p();
#pragma unroll
  for (int c = 0; c < NCH; ++c) tmem_st_32x32b_x16(taddr + kPCol + (ch0 + c) * 16, pk[c]);
  return bsum;
}

// F8OUT: ctx written as E4M3(ctx_scale * ctx) bytes [T, H] (the FP8 out-projection's A operand)
// F16: Q, K, V, P and ctx in fp16 instead of bf16 (fp16 operand precision)
template <bool F8OUT, bool F16>
__global__ void __launch_bounds__(kAwsThreads, 1)
    k_attention_tc(const __grid_constant__ CUtensorMap tm, const AttnWork* __restrict__ work,
                   const int32_t* __restrict__ num_work, int H, int nh, uint16_t* __restrict__ ctx,
                   float scale_log2, int Tp, float ctx_scale) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  const int warp = warp_id(), lane = lane_id();
  // pipeline of this warp: control warps 2 pp (TMA) / 2 pp + 1 (MMA), softmax warps 4 + 4 pp .. 7 + 4 pp
  const int pp = warp < 4 ? warp >> 1 : (warp - 4) >> 2;
  uint8_t* sQ = smem + pp * kPipeSmem;                 // [2][16 KB]
  uint8_t* sK = sQ + 2 * kBlkBytes;                    // [kAwsKV][16 KB]
  uint8_t* sV = sK + kAwsKV * kBlkBytes;               // [kAwsKV][16 KB]
  uint64_t* bars_all = reinterpret_cast<uint64_t*>(smem + 2 * kPipeSmem);
  constexpr int kBarsPerPipe = 24;
  uint64_t* bars = bars_all + pp * kBarsPerPipe;
  uint64_t* q_full = bars;                  // [2]  Q slot loaded (TMA bytes)
  uint64_t* q_empty = bars + 2;             // [2]  Q slot free (4 softmax warps, after the epilogue)
  uint64_t* k_full = bars + 4;              // [kAwsKV]
  uint64_t* k_empty = bars + 6;             // [kAwsKV]  (commit: S_g done)
  uint64_t* v_full = bars + 8;              // [kAwsKV]
  uint64_t* v_empty = bars + 10;            // [kAwsKV]  (commit: PV_g done)
  uint64_t* s_full = bars + 12;             // S_g in TMEM (commit)
  uint64_t* s_free = bars + 13;             // S_g read into registers (4 softmax warps)
  uint64_t* p_full = bars + 14;             // P_g in TMEM (4 softmax warps)
  uint64_t* p_free = bars + 15;             // PV_g done: P columns free, O stable (commit)
  uint64_t* o_full = bars + 16;             // the item's last PV done (commit)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars_all + 2 * kBarsPerPipe);

  const int nitems = __ldg(num_work) * nh;
  const int G = 2 * static_cast<int>(gridDim.x);       // pipelines in the grid
  const int first = 2 * static_cast<int>(blockIdx.x) + pp;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    for (int x = 0; x < 2; ++x) {
      uint64_t* b = bars_all + x * kBarsPerPipe;
      for (int i = 0; i < 2; ++i) {
        mbar_init(&b[i], 1);
        mbar_init(&b[2 + i], 4);
        mbar_init(&b[4 + i], 1);
        mbar_init(&b[6 + i], 1);
        mbar_init(&b[8 + i], 1);
        mbar_init(&b[10 + i], 1);
      }
      mbar_init(&b[12], 1);
      mbar_init(&b[13], 4);
      mbar_init(&b[14], 4);
      mbar_init(&b[15], 1);
      mbar_init(&b[16], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot + pp * 256;   // this pipeline's S [0,128), P [128,192), O [192,256)

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kAwsRegsCtl));
    if ((warp & 1) == 0 && lane == 0) {
      // ---------------- TMA producer: the 32-row boxes of the tile's Q and of each key block; box s
      // of the tile's request k (packed) lands in slot f_k + s, a long request's rows in slots 0..
      uint32_t kvn = 0, itn = 0;
      unsigned tr_k = 0;
      (void)tr_k;
      for (int item = first; item < nitems; item += G, ++itn) {
        const AttnWork w = load_work(work + item / nh);
        const int h = item % nh;
        const int qs = itn & 1;
        const bool packed = tile_packed(w);
        ATR(0, 1);
        mbar_wait(&q_empty[qs], ((itn >> 1) & 1) ^ 1u);
        ATR(0, 2);
        uint8_t* dq = sQ + qs * kBlkBytes;
        int nbq = 0;
        if (packed) {
#pragma unroll
          for (int k = 0; k < 4; ++k) nbq += k < w.nreq ? ceil32(w.len[k]) : 0;
        } else {
          nbq = ceil32(min(TKB, w.len[0] - w.q0));
        }
        mbar_arrive_expect_tx(&q_full[qs], nbq * kBoxBytes);
        if (packed) {
          int f = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (k < w.nreq) {
              const int sg = ceil32(w.len[k]);
              for (int x = 0; x < sg; ++x)
                tma_load_2d(dq + (f + x) * kBoxBytes, &tm, &q_full[qs], 0, h * Tp + w.start[k] + 32 * x);
              f += sg;
            }
          }
        } else {
          for (int x = 0; x < nbq; ++x)
            tma_load_2d(dq + x * kBoxBytes, &tm, &q_full[qs], 0, h * Tp + w.start[0] + w.q0 + 32 * x);
        }
        const int nkb = tile_nkb(w);
        for (int j = 0; j < nkb; ++j, ++kvn) {
          const int s = kvn % kAwsKV;
          const uint32_t par = ((kvn / kAwsKV) & 1) ^ 1u;
          const int nb = packed ? nbq : ceil32(min(TKB, w.len[0] - TKB * j));  // packed: Q's boxes
          for (int kv = 0; kv < 2; ++kv) {  // K_j, then V_j (each ring frees at its own MMA)
            uint64_t* fullb = kv ? &v_full[s] : &k_full[s];
            ATR(0, 3);
            mbar_wait(kv ? &v_empty[s] : &k_empty[s], par);
            ATR(0, 4);
            mbar_arrive_expect_tx(fullb, nb * kBoxBytes);
            uint8_t* dst = (kv ? sV : sK) + s * kBlkBytes;
            const int rowp = (kv ? 2 * nh + h : nh + h) * Tp;
            if (packed) {
              int f = 0;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if (k < w.nreq) {
                  const int sg = ceil32(w.len[k]);
                  for (int x = 0; x < sg; ++x)
                    tma_load_2d(dst + (f + x) * kBoxBytes, &tm, fullb, 0, rowp + w.start[k] + 32 * x);
                  f += sg;
                }
              }
            } else {
              const int t0 = w.start[0] + TKB * j;
              for (int x = 0; x < nb; ++x) tma_load_2d(dst + x * kBoxBytes, &tm, fullb, 0, rowp + t0 + 32 * x);
            }
          }
        }
      }
      ATR_DONE(0);
    } else if ((warp & 1) == 1 && lane == 0) {
      // ---------------- MMA issuer: S_0, S_1, PV_0, S_2, PV_1, ... over the pipeline's blocks
      constexpr uint32_t idesc_s = F16 ? make_idesc_f16_f32(TQ, TKB) : make_idesc_bf16_f32(TQ, TKB);
      constexpr uint32_t idesc_o =
          (F16 ? make_idesc_f16_f32(TQ, TD) : make_idesc_bf16_f32(TQ, TD)) | (1u << 16);  // V MN-major
      unsigned tr_k = 0;
      (void)tr_k;
      // S cursor (ahead) and PV cursor (one block behind), each (item, block, global block, item count)
      int s_item = first, s_j = 0, p_item = first, p_j = 0;
      uint32_t s_g = 0, s_itn = 0, p_g = 0;
      AttnWork s_w{}, p_w{};
      if (s_item < nitems) s_w = load_work(work + s_item / nh);
      p_w = s_w;
      auto issue_s = [&]() {  // S of the S cursor's block; advances the cursor
        const int qs = s_itn & 1;
        if (s_j == 0) {
          ATR(1, 10);
          mbar_wait(&q_full[qs], (s_itn >> 1) & 1);
          ATR(1, 11);
        }
        const int s = s_g % kAwsKV;
        ATR(1, 12);
        mbar_wait(&k_full[s], (s_g / kAwsKV) & 1);
        if (s_g > 0) mbar_wait(s_free, (s_g - 1) & 1);  // the softmax has read S_{g-1}
        ATR(1, 13);
        tc_fence_after();
        const uint64_t dq = make_sw128_desc(smem_u32(sQ + qs * kBlkBytes));
        const uint64_t dk = make_sw128_desc(smem_u32(sK + s * kBlkBytes));
#pragma unroll
        for (int k = 0; k < TD / 16; ++k) tc_mma_f16(tmem, dq + 2 * k, dk + 2 * k, idesc_s, k > 0);
        tc_commit(s_full);
        tc_commit(&k_empty[s]);
        ++s_g;
        if (++s_j == tile_nkb(s_w)) {
          s_j = 0;
          ++s_itn;
          s_item += G;
          if (s_item < nitems) s_w = load_work(work + s_item / nh);
        }
      };
      if (s_item < nitems) issue_s();
      while (p_item < nitems) {
        // within an item S_{g+1} goes before PV_g (the softmax of block g + 1 overlaps PV_g); the
        // next item's first S after the item's last PV (its Q / K may still be loading)
        if (s_item == p_item) issue_s();
        const int s = p_g % kAwsKV;
        ATR(1, 14);
        mbar_wait(p_full, p_g & 1);
        mbar_wait(&v_full[s], (p_g / kAwsKV) & 1);
        ATR(1, 15);
        tc_fence_after();
        const int nks = (tile_key_hi(p_w, p_j) + 15) / 16;  // 16-key steps holding keys of the tile
        const uint8_t* sv = sV + s * kBlkBytes;
        for (int ks = 0; ks < nks; ++ks) {
          const uint64_t dv = make_sw128_desc(smem_u32(sv + ks * (16 * TD * 2)));
          tc_mma_f16_tmem_a(tmem + kOCol, tmem + kPCol + ks * 8, dv, idesc_o, (p_j | ks) != 0 ? 1u : 0u);
        }
        tc_commit(&v_empty[s]);
        tc_commit(p_free);
        ++p_g;
        if (++p_j == tile_nkb(p_w)) {
          tc_commit(o_full);
          p_j = 0;
          p_item += G;
          if (p_item < nitems) p_w = load_work(work + p_item / nh);
          if (s_item < nitems && s_item == p_item) issue_s();  // the next item's first S
        }
      }
      ATR_DONE(1);
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kAwsRegsSoftmax));
    // ---------------- softmax + epilogue (TMEM lane quarter q = warp & 3)
    const int q = warp & 3;
    const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const int row = q * 32 + lane;
    uint32_t g = 0, itn = 0;
    unsigned tr_k = 0;
    (void)tr_k;
    AttnWork wn = load_work(work + min(first, max(nitems - 1, 0)) / nh);  // prefetched work entry
    for (int item = first; item < nitems; item += G, ++itn) {
      const AttnWork w = wn;
      if (item + G < nitems) wn = load_work(work + (item + G) / nh);
      const int h = item % nh;
      const int nkb = tile_nkb(w);
      const WarpRows wr = warp_rows(w, q);
      const bool packed = tile_packed(w);
      // packed tiles: P is zero outside the warp's own key chunks within [0, tile_nch)
      const int tile_nch = packed ? ceil32(tile_key_hi(w, 0)) : 0;
      float m = 0.f, l = 0.f;  // running row max (scaled, log2 domain) and row sum
      for (int j = 0; j < nkb; ++j, ++g) {
        if (q == 0 && lane == 0) ATR(2, 20);
        mbar_wait(s_full, g & 1);
        if (q == 0 && lane == 0) ATR(2, 21);
        tc_fence_after();
        auto release = [&]() {  // S_g is in registers: the next S may overwrite the columns
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_free);
        };
        if (wr.active) {
          const int nk = packed ? wr.klen : min(TKB, wr.klen - TKB * j);  // valid keys of this block
          const int nch = ceil32(nk);
          float alpha = 1.f;
          bool resc = false;
          auto before_p = [&]() {  // PV_{g-1} has read the P columns and O is complete
            if (g > 0) mbar_wait(p_free, (g - 1) & 1);
            tc_fence_after();
            if (resc) {  // O *= alpha
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
            if (packed) {  // other requests' key chunks of the tile: P = 0
              uint32_t z[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) z[e] = 0u;
              for (int c = 0; c < tile_nch; ++c)
                if (c < wr.ch0 || c >= wr.ch0 + nch) tmem_st_32x32b_x16(taddr + kPCol + c * 16, z);
            }
          };
          float bsum;
          switch (nch) {
            case 1: bsum = softmax_block<1, F16>(taddr, wr.ch0, nk, j, scale_log2, m, resc, alpha, release, before_p); break;
            case 2: bsum = softmax_block<2, F16>(taddr, wr.ch0, nk, j, scale_log2, m, resc, alpha, release, before_p); break;
            case 3: bsum = softmax_block<3, F16>(taddr, wr.ch0, nk, j, scale_log2, m, resc, alpha, release, before_p); break;
            default: bsum = softmax_block<4, F16>(taddr, wr.ch0, nk, j, scale_log2, m, resc, alpha, release, before_p); break;
          }
          l = (j == 0) ? bsum : (resc ? l * alpha : l) + bsum;
          tc_wait_st();
        } else {
          release();
          // no P to write, but p_full(g) must not be arrived before phase g - 1 completed: an early
          // second arrival would count toward the wrong phase
          if (g > 0) mbar_wait(p_free, (g - 1) & 1);
        }
        if (q == 0 && lane == 0) ATR(2, 28);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        if (q == 0 && lane == 0) ATR(2, 22);
      }
      // ---- epilogue: ctx = O / l, staged in this item's Q slot (every S MMA of the item is complete
      // once o_full fires), rows XOR-swizzled in 16-byte pieces, then 4 rows per warp instruction
      if (q == 0 && lane == 0) ATR(2, 23);
      mbar_wait(o_full, itn & 1);
      if (q == 0 && lane == 0) ATR(2, 24);
      tc_fence_after();
      const int qs = itn & 1;
      uint8_t* stg = sQ + qs * kBlkBytes;
      if (wr.active) {
#pragma unroll
        for (int x = 0; x < 2; ++x) {  // one 32-column half of O at a time
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + kOCol + x * 32, v);
          tc_wait_ld();
          if constexpr (F8OUT) {  // 64-byte rows: 4 pieces, XOR-swizzled by row & 3
            const float inv = ctx_scale / l;
            uint4* srow = reinterpret_cast<uint4*>(stg + row * TD);
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
            uint4* srow = reinterpret_cast<uint4*>(stg + row * (TD * 2));
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
        __syncwarp();
        if constexpr (F8OUT) {
          uint8_t* c8 = reinterpret_cast<uint8_t*>(ctx);
          const int c = lane & 3;
          for (int rr = lane >> 2; rr < wr.rows; rr += 8) {
            const int sr = q * 32 + rr;
            const uint4 val = reinterpret_cast<const uint4*>(stg + sr * TD)[c ^ (sr & 3)];
            *reinterpret_cast<uint4*>(c8 + static_cast<size_t>(wr.tok + rr) * H + h * TD + c * 16) = val;
          }
        } else {
          const int c = lane & 7;
          for (int rr = lane >> 3; rr < wr.rows; rr += 4) {
            const int sr = q * 32 + rr;
            const uint4 val = reinterpret_cast<const uint4*>(stg + sr * (TD * 2))[c ^ (sr & 7)];
            *reinterpret_cast<uint4*>(ctx + static_cast<size_t>(wr.tok + rr) * H + h * TD + c * 8) = val;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&q_empty[qs]);  // the slot's staging has been read
      if (q == 0 && lane == 0) ATR(2, 25);
    }
    if (q == 0 && lane == 0) ATR_DONE(2);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(*tmem_slot);
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
                                                       const uint32_t* __restrict__ err) {
  if (err && *err) return;  // invalid lengths (sticky error): cu may point past the planes
  const int h = blockIdx.x, i = blockIdx.y;
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

bool make_tmap_qkv(CUtensorMap* m, const void* qkv, uint64_t rows, int H) {
  // head-major planes [3 * nh][rows][64] viewed as one [3 * nh * rows, 64] matrix; 32-row boxes of
  // 64 16-bit values (one SWIZZLE_128B row each): a request segment's rows of one head's Q, K or V
  return make_tmap_bf16_box(m, qkv, rows * static_cast<uint64_t>(3 * (H / 64)), 64, 64, kBoxRows);
}

cudaError_t launch_attention(const uint16_t* qkv, const CUtensorMap* tm_qkv, const int32_t* cu_seqlens,
                             const AttnWork* work, const int32_t* num_work, int64_t T, int n, int H, int num_heads,
                             int64_t plane_rows, uint16_t* ctx, float ctx_f8_scale, bool f16, int num_sms,
                             cudaStream_t st) {
  if (T <= 0 || n <= 0) return cudaSuccess;
  const int d = H / num_heads;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(d));
  const int64_t max_tiles = attn_max_tiles(T, n, attn_tile_q(d));
  if (d == 64) {
    if (!tm_qkv) return cudaErrorInvalidValue;
    if (f16 && ctx_f8_scale > 0.f) return cudaErrorInvalidValue;
    auto kern = f16 ? k_attention_tc<false, true> : ctx_f8_scale > 0.f ? k_attention_tc<true, false>
                                                                       : k_attention_tc<false, false>;
    if (!attr_once(reinterpret_cast<const void*>(kern))) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnTcSmem);
      if (e != cudaSuccess) return e;
    }
    // persistent: one CTA per SM (TMEM 512 columns, shared memory ~194 KB), two pipelines each
    const int64_t items = max_tiles * num_heads;
    const unsigned grid = static_cast<unsigned>((items + 1) / 2 < num_sms ? (items + 1) / 2 : num_sms);
    kern<<<grid, kAwsThreads, kAttnTcSmem, st>>>(*tm_qkv, work, num_work, H, num_heads, ctx, scale_log2,
                                                 static_cast<int>(plane_rows), ctx_f8_scale);
  } else if (d == 32) {
    if (ctx_f8_scale > 0.f || f16) return cudaErrorInvalidValue;
    const unsigned grid = static_cast<unsigned>(max_tiles * num_heads);
    k_attention<32><<<grid, 128, 0, st>>>(qkv, cu_seqlens, work, num_work, H, num_heads, ctx, scale_log2);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_attention_cls(const uint16_t* qkv, const int32_t* cu_seqlens, int n, int H, int num_heads,
                                 int64_t plane_rows, const float* h32, uint16_t* ctx_c, float* hres_c, int out_kind,
                                 float ctx_scale, const uint32_t* err, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (H / num_heads != TD) return cudaErrorInvalidValue;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(TD));
  const dim3 grid(num_heads, n);
  const int Tp = static_cast<int>(plane_rows);
  switch (out_kind) {
    case 0: k_attention_cls<0><<<grid, 128, 0, st>>>(qkv, cu_seqlens, num_heads, Tp, H, scale_log2, h32, ctx_c, hres_c, ctx_scale, err); break;
    case 1: k_attention_cls<1><<<grid, 128, 0, st>>>(qkv, cu_seqlens, num_heads, Tp, H, scale_log2, h32, ctx_c, hres_c, ctx_scale, err); break;
    case 2: k_attention_cls<2><<<grid, 128, 0, st>>>(qkv, cu_seqlens, num_heads, Tp, H, scale_log2, h32, ctx_c, hres_c, ctx_scale, err); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}


}  // namespace elis
