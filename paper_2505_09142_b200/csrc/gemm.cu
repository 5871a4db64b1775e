// gemm.cu -- dense encoder GEMMs on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
//   C[M, N] = A[M, K] * W[N, K]^T + bias  (+ GELU | + fp32 residual | + residual -> LayerNorm)
//
// The QKV, attention-output and FFN contractions of every BERT block (SURVEY.md Sec. 8a
// rows a3/a5/a7/a8; BGE = BERT-base).  Both operands are K-major (activations
// row-major, nn.Linear weights [out, in]), the natural tcgen05 layout.
//
// Design (sm_100a):
//   * CTA pairs (tcgen05 cta_group::2): a 256 x BN output tile per pair; each CTA stages
//     its 128 rows of A and half (BN/2 rows) of the B slab, the leader CTA issues
//     tcgen05.mma M=256 for both, each CTA's TMEM holds its 128 accumulator rows (per CTA
//     this halves the B bytes fetched from L2 per FLOP);
//   * persistent grid, static tile schedule; warp 0 = TMA producer (SWIZZLE_128B slabs,
//     mbarrier ring, completion counted on the leader's barrier), warp 1 (leader) = the
//     single-thread MMA issuer, warp 2 = TMEM allocator, warps 4..11 = epilogue (two warps
//     per TMEM lane quarter, each owning half of the tile's columns);
//   * two TMEM accumulators (2 x BN columns): the epilogue of tile i overlaps the mainloop
//     of tile i+1;
//   * epilogue global I/O goes through TMA in 32-row x 32-column boxes: the fp32 residual is
//     TMA-loaded into per-warp swizzled slots (2-deep ring, issued before the accumulator is
//     ready), results are staged in shared memory and written by TMA bulk stores.  (Thread =
//     row stores would hit 32 cache lines per warp instruction.)  TMA also clips the ragged
//     M tail, so T is never padded;
//   * no split-K: every output row depends on its own A row only (batch invariance).
//
// EPI_BIAS_RESID_LN (attention-output and FFN2 + LayerNorm, rows a5+a6 / a8): a row of
// H = 768 / 1024 columns spans CS = H / BN pairs, launched as one cluster of 2 x CS CTAs.
// Each CTA adds bias + residual, keeps v in TMEM (tcgen05.st), computes per-row (mean, M2)
// over its columns and pushes them into every peer's shared memory over DSMEM
// (st.shared::cluster + remote mbarrier arrive); every CTA then merges the CS partials in
// rank order (Chan) and normalises its columns.  The fp32 residual stream is updated in
// place and the bf16 copy for the next GEMM is written in the same pass: 10 B/element of
// epilogue traffic instead of 18 B with a separate LayerNorm kernel.
#include "common.cuh"
#include "kernels.cuh"

namespace elis {

#ifdef ELIS_GEMM_TRACE
// Diagnostic build only (--variant=gtrace -DELIS_GEMM_TRACE): per-CTA clock64 totals of the
// GEMM roles' waits, overwritten by every launch.  Slots: 0 producer wait(empty), 1 MMA
// wait(tempty), 2 MMA wait(full), 3 MMA busy span, 4 epi wait(tfull), 5 epi pass 1,
// 6 epi wait(stats), 7 epi pass 2, 8 epi total span, 9 tiles, 10 smid.
constexpr int kGemmTraceCtas = 1024;
__device__ long long g_gemm_trace[kGemmTraceCtas * 16];
#define GT_ADD(slot, v) \
  do { if (blockIdx.x < kGemmTraceCtas) g_gemm_trace[blockIdx.x * 16 + (slot)] += (v); } while (0)
#define GT_CLK() clock64()
#else
#define GT_ADD(slot, v) do { } while (0)
#define GT_CLK() 0ll
#endif

namespace {

constexpr int BM = 128;  // rows per CTA (256 per pair)
constexpr int BK = 64;
// Epilogue warps: 8, except the FP8 GELU epilogue: with the E4M3 mainloop twice as fast it is the
// bound of FFN1 and runs 16 warps (<= 96 registers each; measured FFN1 1.84 -> 1.65 ms per cfg2
// step, while 16 warps made the bf16 / fp16 QKV and FFN1 3-5% slower).
template <int EPI, int PREC>
constexpr int epi_warps() { return (PREC == 1 && EPI == EPI_BIAS_GELU_BF16) ? 16 : 8; }
template <int EPI, int PREC>
constexpr int gemm_threads() { return 128 + epi_warps<EPI, PREC>() * 32; }  // 4 control warps + epilogue warps
constexpr int kMaxEpiWarps = 16;
constexpr int kMaxCluster = 4;                       // max N-tiles (pairs) per LN row
constexpr int kBox = 32;                             // epilogue TMA boxes: 32 rows x 32 columns

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_ROWS = BN / 2;              // this CTA's half of the B slab
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
};
// Shared-memory plan per epilogue kind.  DEEP (long-K residual GEMMs, e.g. FFN2: the mainloop
// dominates and the epilogue has slack) keeps one residual slot per warp and, for LN, stages the
// fp32 output in that slot too (the next tile's residual is fetched once the slot's store has
// been read): the freed 64 KB buy a fourth and a fifth operand stage.
template <int BN, int EPI, bool DEEP, int PREC>
struct SmemPlan {
  static constexpr bool LN16 = EPI == EPI_BIAS_RESID16_LN;  // 16-bit residual stream, no fp32 output
  static constexpr bool LN = EPI == EPI_BIAS_RESID_LN || LN16;
  static constexpr bool RES = LN || EPI == EPI_BIAS_RESID_F32;
  static constexpr bool OUT_F32 = RES && !LN16;        // f32 staging (4 KB per warp)
  static constexpr bool OUT_BF16 = LN || !RES;         // bf16 staging (2 KB per warp)
  static constexpr int EW = epi_warps<EPI, PREC>();
  static constexpr int NSTG = (RES || EW == 16) ? 1 : 2;  // staging buffers per warp
  static constexpr int NRES = (RES && DEEP) ? 1 : 2;   // residual slots per warp
  static constexpr bool F32_IN_RES = LN && DEEP && !LN16;  // fp32 output staged in the residual slot
  // LN16 halves the residual slots and drops the fp32 staging: 5 operand stages either way
  static constexpr int STAGES = RES ? ((DEEP || LN16) ? (F32_IN_RES || LN16 ? 5 : 4) : 3) : 5;
  static constexpr int RES_SLOT = kBox * kBox * (LN16 ? 2 : 4);  // 4 KB fp32 / 2 KB fp16 residual box
  static constexpr int RES_BYTES = RES ? EW * NRES * RES_SLOT : 0;
  static constexpr int STG_F32 = kBox * kBox * 4;      // 4 KB
  static constexpr int STG_BF16 = kBox * kBox * 2;     // 2 KB
  static constexpr int STG_WARP = NSTG * (((OUT_F32 && !F32_IN_RES) ? STG_F32 : 0) + (OUT_BF16 ? STG_BF16 : 0));
  static constexpr int STG_BYTES = EW * STG_WARP;
  // barriers (512) + LN stats[2][kMaxCluster][128] f2 + part[2][128] f2 + bias/gamma/beta/colscale[256] f32
  static constexpr int AUX_BYTES = 512 + 2 * kMaxCluster * 128 * 8 + 2 * 128 * 8 + 4 * 256 * 4;
  static constexpr int SMEM_BYTES = STAGES * GemmCfg<BN>::STAGE_BYTES + RES_BYTES + STG_BYTES + AUX_BYTES + 1024;
  static_assert(SMEM_BYTES <= 232448, "shared memory");
};

// GELU(x) = x * Phi(x) (erf form).  Phi is evaluated as sigmoid(x * (c0 + c1 x^2 + c2 x^4))
// with minimax coefficients fitted to the exact erf form: max |error| of GELU over all x is
// 2.6e-5 (scripts/fit_gelu.py), < 1/75 of the bf16 rounding of the output this epilogue
// writes.  10 instructions incl. 2 MUFU instead of ~28 for erff (the FFN1 epilogue is
// instruction-issue bound).
// Same minimax sigmoid form evaluated as x sigmoid(y) = 0.5 x (1 + tanh(y / 2)): one MUFU
// (tanh.approx) instead of two, max |error| 3.0e-5 (scripts/gelu_acc.cu).  Used by the FP8 FFN1
// epilogue (MUFU-heavy once the E4M3 mainloop halves: 1.65 -> 1.53 ms per cfg2 step); the 16-bit
// paths keep the two-MUFU form, which measured faster there.
ELIS_DEV float gelu_tanh_form(float x) {
  constexpr float a0 = 0.5f * 1.5950205882421884f, a1 = 0.5f * 0.07400664121448398f,
                  a2 = -0.5f * 0.0007022165804436097f;
  const float xc = fminf(fmaxf(x, -9.0f), 9.0f);
  const float x2 = xc * xc;
  const float q = fmaf(fmaf(a2, x2, a1), x2, a0);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(xc * q));
  const float h = 0.5f * x;
  return fmaf(h, t, h);
}

// Two GELUs of the sigmoid form with the polynomial / products on packed fp32x2 (FFMA2 / FMUL2 /
// FADD2): per element x * 1 / (1 + 2^(x (c0 + c1 x^2 + c2 x^4) log2 e)), the clamp at |x| <= 9,
// two MUFU ops (ex2, rcp) -- the same operations per lane as scalar code, half the FMA-pipe issues.
ELIS_DEV unsigned long long gf2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
ELIS_DEV void gf2_unpack(unsigned long long v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
ELIS_DEV unsigned long long gf2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
ELIS_DEV unsigned long long gf2_mul(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
ELIS_DEV unsigned long long gf2_add(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
ELIS_DEV void gelu_fast2(float& x0, float& x1) {
  constexpr float kL2E = 1.4426950408889634f;
  constexpr float c0 = -1.5950205882421884f * kL2E, c1 = -0.07400664121448398f * kL2E,
                  c2 = 0.0007022165804436097f * kL2E;
  const unsigned long long xc = gf2(fminf(fmaxf(x0, -9.0f), 9.0f), fminf(fmaxf(x1, -9.0f), 9.0f));
  const unsigned long long x2 = gf2_mul(xc, xc);
  const unsigned long long p = gf2_fma(gf2_fma(gf2(c2, c2), x2, gf2(c1, c1)), x2, gf2(c0, c0));
  float a0, a1, e0, e1, r0, r1;
  gf2_unpack(gf2_mul(xc, p), a0, a1);
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(a0));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(a1));
  gf2_unpack(gf2_add(gf2(e0, e1), gf2(1.0f, 1.0f)), a0, a1);
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(a0));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(a1));
  gf2_unpack(gf2_mul(gf2(x0, x1), gf2(r0, r1)), x0, x1);
}

ELIS_DEV unsigned long long gx_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
ELIS_DEV uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Chan et al. merge of (count, mean, M2) partial statistics.
ELIS_DEV void chan_merge(float& n_a, float& mean_a, float& m2_a, float n_b, float mean_b, float m2_b) {
  const float n = n_a + n_b;
  const float d = mean_b - mean_a;
  mean_a = mean_a + d * (n_b / n);
  m2_a = m2_a + m2_b + d * d * (n_a * n_b / n);
  n_a = n;
}

// Byte offset of 16-byte piece k of row r in a 32-row box with 128-byte rows, SWIZZLE_128B.
ELIS_DEV uint32_t sw128_off(int r, int k) { return static_cast<uint32_t>(r * 128 + ((k ^ (r & 7)) << 4)); }
// Same for 64-byte rows, SWIZZLE_64B (16-byte pieces XOR bits [7,9) of the offset).
ELIS_DEV uint32_t sw64_off(int r, int k) { return static_cast<uint32_t>(r * 64 + ((k ^ ((r >> 1) & 3)) << 4)); }
// Same for 32-byte rows, SWIZZLE_32B (16-byte pieces XOR bit 7 of the offset): the E4M3 boxes.
ELIS_DEV uint32_t sw32_off(int r, int k) { return static_cast<uint32_t>(r * 32 + ((k ^ ((r >> 2) & 1)) << 4)); }

// 32 values of one row -> E4M3(scale * v) into a 32-byte row of a SWIZZLE_32B staging box.
ELIS_DEV void stage_e4m3_row(uint8_t* b, int lane, const float (&v)[32], float scale) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      w[j] = pack_e4m3x4(v[16 * k + 4 * j] * scale, v[16 * k + 4 * j + 1] * scale, v[16 * k + 4 * j + 2] * scale,
                         v[16 * k + 4 * j + 3] * scale);
    *reinterpret_cast<uint4*>(b + sw32_off(lane, k)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// PREC: 0 bf16 operands, 1 E4M3 operands (kind::f8f6f4), 2 fp16 operands (16-bit outputs in fp16)
// GX (LN epilogues): row statistics exchanged through global memory (args.gstats / gflag) by CTA
// pairs that need not share a cluster -- the grid spans every SM instead of the 132 that clusters
// of 6 fill; the pairs of a row group work on the same m tile at the same step of the schedule.
template <int BN, int EPI, bool DEEP, int PREC, bool GX = false>
__global__ void __launch_bounds__(gemm_threads<EPI, PREC>(), 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmO,
              const __grid_constant__ CUtensorMap tmOb, const GemmArgs args) {
  using C = GemmCfg<BN>;
  using SP = SmemPlan<BN, EPI, DEEP, PREC>;
  constexpr int NRES = SP::NRES;
  constexpr bool LN = SP::LN;
  constexpr bool RES = SP::RES;
  constexpr int STAGES = SP::STAGES;
  constexpr bool F8 = PREC == 1;
  constexpr int EW = SP::EW;                 // epilogue warps
  static_assert(!LN || EW == 8, "the LN statistics exchange assumes two column halves per CTA");
  constexpr bool F16 = PREC == 2;
  // K elements per 128-byte operand row: 64 bf16 or 128 E4M3 (4 MMAs of K 16 / K 32 either way)
  constexpr int BKE = F8 ? 2 * BK : BK;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  uint8_t* sRes = sB + STAGES * C::B_BYTES;   // [warp][2 slots][4 KB]
  uint8_t* sStg = sRes + SP::RES_BYTES;       // [warp][NSTG][f32 4 KB | bf16 2 KB]
  uint8_t* aux = sStg + SP::STG_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(aux);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;    // LN: stats slots filled by every CTA of the row group
  uint64_t* rfull = sfull + 2;     // [warp][2]: residual slot landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + 2 * EW);
  float2* stats = reinterpret_cast<float2*>(aux + 512);    // [2][kMaxCluster][128]
  float2* part = stats + 2 * kMaxCluster * 128;             // [2 halves][128]
  float* sbias = reinterpret_cast<float*>(part + 2 * 128);   // [256]
  float* sgam = sbias + 256;                                 // [256]
  float* sbet = sgam + 256;                                  // [256]
  float* sscale = sbet + 256;                                // [256] F8: per-column dequant scale

  const int warp = warp_id();
  const int lane = lane_id();
  const int N = args.N, K = args.K;
  const int num_n = N / BN;
  const int num_k = K / BKE;
  // Cluster = (LN ? num_n : 1) pairs.  CTA rank r: pair r >> 1, half (row half / B half) r & 1.
  const int crank = static_cast<int>(cluster_ctarank());
  constexpr bool LNC = LN && !GX;          // LN statistics over the cluster (DSMEM)
  const int cpairs = LNC ? num_n : 1;
  const int pair_in_cluster = crank >> 1;
  const int hrow = crank & 1;              // which 128-row half of the pair tile
  const bool leader = hrow == 0;
  const int leader_rank = crank & ~1;
  const int cid = static_cast<int>(blockIdx.x) / (2 * cpairs);
  const int ncl = static_cast<int>(gridDim.x) / (2 * cpairs);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EW);  // one arrive per epilogue warp of both CTAs (leader's copy used)
#ifdef ELIS_LN_RELEASE_ARRIVES
      mbar_init(&sfull[a], 4 * cpairs);      // one arrive per half-0 epilogue warp of every row peer
#else
      mbar_init(&sfull[a], 1);               // the local expect_tx; the peers' st.async complete the bytes
#endif
    }
    for (int i = 0; i < 2 * EW; ++i) mbar_init(&rfull[i], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // everything above touches only this kernel's parameters; the row count and every operand below
  // may come from the preceding kernel (programmatic dependent launch, common.cuh)
  pdl_wait();
  pdl_trigger();
  const int M = args.M_dev ? min(max(__ldg(args.M_dev), 0), args.M) : args.M;
  const int num_m = (M + 2 * BM - 1) / (2 * BM);  // 256-row pair tiles
  const int num_iter_tiles = LNC ? num_m : num_m * num_n;
  auto tile_mn = [&](int t, int& m, int& n) {
    if (LNC) { m = t; n = pair_in_cluster; } else { m = t / num_n; n = t % num_n; }
    if (args.m_reverse) m = num_m - 1 - m;
  };

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs); bytes counted on the leader's full barrier
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = cid; t < num_iter_tiles; t += ncl) {
        int m, n;
        tile_mn(t, m, n);
        for (int kb = 0; kb < num_k; ++kb) {
          const long long g0 = GT_CLK();
          mbar_wait(&empty[s], ph ^ 1u);
          GT_ADD(0, GT_CLK() - g0);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * C::STAGE_BYTES);
          const uint32_t bar = mapa_shared(smem_u32(&full[s]), leader_rank);
          tma_load_2d_pair(sA + s * C::A_BYTES, &tmA, bar, kb * BKE, m * 2 * BM + hrow * BM);
          tma_load_2d_pair(sB + s * C::B_BYTES, &tmB, bar, kb * BKE, n * BN + hrow * C::B_ROWS);
          if (++s == STAGES) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA, one thread) for the pair
    if (leader && lane == 0) {
      constexpr uint32_t idesc = F8    ? make_idesc_e4m3_f32(2 * BM, BN)
                                 : F16 ? make_idesc_f16_f32(2 * BM, BN)
                                       : make_idesc_bf16_f32(2 * BM, BN);
      const uint16_t mask = static_cast<uint16_t>(3u << leader_rank);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      const long long gstart = GT_CLK();
      for (int t = cid; t < num_iter_tiles; t += ncl, ++it) {
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        long long g0 = GT_CLK();
        mbar_wait_acquire_cluster(&tempty[acc], aph ^ 1u);
        GT_ADD(1, GT_CLK() - g0);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          g0 = GT_CLK();
          mbar_wait(&full[s], ph);
          GT_ADD(2, GT_CLK() - g0);
          tc_fence_after();
          const uint64_t da = make_sw128_desc(smem_u32(sA + s * C::A_BYTES));
          const uint64_t db = make_sw128_desc(smem_u32(sB + s * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            // advance 32 bytes (16 bf16 / 32 E4M3) along K inside the 128-byte swizzle row
            if constexpr (F8) tc_mma_f8_pair(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
            else tc_mma_f16_pair(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          tc_commit_pair_mc(&empty[s], mask);
          if (++s == STAGES) { s = 0; ph ^= 1u; }
        }
        tc_commit_pair_mc(&tfull[acc], mask);
      }
      GT_ADD(3, GT_CLK() - gstart);
      GT_ADD(9, it);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (each CTA: its 128 rows; warp: 32 rows x BN/2 columns)
    constexpr int CPW = BN / (EW / 4);   // tile columns per epilogue warp
    constexpr int CH = CPW / 32;         // 32-column chunks per epilogue warp
    const int ew = warp - 4;             // 0..7
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int half = ew >> 2;            // which column part of the tile (a half when EW = 8)
    const int row_in_tile = q * 32 + lane;
    const int etid = ew * 32 + lane;     // 0..255
    uint8_t* rslot = sRes + ew * NRES * SP::RES_SLOT;
    uint64_t* rbar = rfull + 2 * ew;
    uint8_t* stg = sStg + ew * SP::STG_WARP;
    uint32_t rpar = 0;                   // parity bits of the two residual slots
    int nstore = 0;                      // store groups issued by this warp
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), leader_rank);
    auto stage_vectors = [&](int n) {    // bias (+ gamma, beta) of tile columns -> shared memory
      if (etid < BN) {
        sbias[etid] = __ldg(args.bias + n * BN + etid);
        if constexpr (F8) sscale[etid] = __ldg(args.colscale + n * BN + etid);
        if constexpr (LN) {
          sgam[etid] = __ldg(args.gamma + n * BN + etid);
          sbet[etid] = __ldg(args.beta + n * BN + etid);
        }
      }
    };
    // residual box (32 rows x 32 columns at col0, row0) -> slot c & 1 (lane 0 issues)
    auto load_res = [&](int row0, int col0, int c) {
      if (lane == 0) {
        if constexpr (SP::F32_IN_RES) tma_store_wait_read<0>();  // the slot's output store has read it
        fence_proxy_async_smem();   // slot previously read through the generic proxy
        mbar_arrive_expect_tx(&rbar[c % NRES], SP::RES_SLOT);
        tma_load_2d(rslot + (c % NRES) * SP::RES_SLOT, &tmR, &rbar[c % NRES], col0, row0);
      }
    };
    // staging buffer for the next store group (waits until its previous store read it)
    auto next_stage = [&]() -> uint8_t* {
      uint8_t* b = stg + (nstore % SP::NSTG) * (SP::STG_WARP / SP::NSTG);
      if (lane == 0) tma_store_wait_read<SP::NSTG - 1>();
      __syncwarp();
      return b;
    };
    // b: the staging of this store group; the fp32 box is read from b32 (b, or the residual slot)
    auto issue_store = [&](uint8_t* b, int row0, int col0, uint8_t* b32 = nullptr) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if constexpr (SP::OUT_F32) tma_store_2d(&tmO, b32 ? b32 : b, col0, row0);
        if constexpr (SP::OUT_BF16) {
          if constexpr (SP::OUT_F32) tma_store_2d(&tmOb, SP::F32_IN_RES ? b : b + SP::STG_F32, col0, row0);
          else if (args.out_head_major) tma_store_3d(&tmO, b, col0 & 63, row0, col0 >> 6);
          else tma_store_2d(&tmO, b, col0, row0);
        }
        tma_store_commit();
      }
      ++nstore;
    };
    if constexpr (LNC) {
      stage_vectors(pair_in_cluster);
      named_bar_sync(1, EW * 32);
    }
    int it = 0;
    const long long gepi = GT_CLK();
    bool res_prefetched = false;  // LN: the next tile's first residual boxes were issued early
    for (int t = cid; t < num_iter_tiles; t += ncl, ++it) {
      int m, n;
      tile_mn(t, m, n);
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int row0 = m * 2 * BM + hrow * BM + q * 32;   // first row of this warp's block
      const int cbase = half * CPW;                        // first tile column of this warp
      if (RES && !res_prefetched) {       // residual does not depend on the MMA: fetch it now
#pragma unroll
        for (int c = 0; c < NRES && c < CH; ++c) load_res(row0, n * BN + cbase + c * 32, c);
      }
      res_prefetched = false;
      if constexpr (!LNC) {
        named_bar_sync(1, EW * 32);  // previous tile's readers of sbias (sgam, sbet) are done
        stage_vectors(n);
        named_bar_sync(1, EW * 32);
      }
      const bool gt_me = (warp == 4 && lane == 0);
      long long g0 = GT_CLK();
      mbar_wait(&tfull[acc], aph);
      long long g1 = GT_CLK();
      if (gt_me) GT_ADD(4, g1 - g0);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + cbase;
      float st_n = 0.f, st_mean = 0.f, st_m2 = 0.f;  // LN row statistics over this warp's columns
      uint32_t r[2][32];
      tmem_ld_32x32b_x32(taddr, r[0]);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        tc_wait_ld();
        if (c + 1 < CH) tmem_ld_32x32b_x32(taddr + (c + 1) * 32, r[(c + 1) & 1]);
        const int tcol = cbase + c * 32;
        const int col0 = n * BN + tcol;
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 bb = *reinterpret_cast<const float4*>(sbias + tcol + j);
          if constexpr (F8) {
            const float4 sc = *reinterpret_cast<const float4*>(sscale + tcol + j);
            v[j + 0] = fmaf(__uint_as_float(r[c & 1][j + 0]), sc.x, bb.x);
            v[j + 1] = fmaf(__uint_as_float(r[c & 1][j + 1]), sc.y, bb.y);
            v[j + 2] = fmaf(__uint_as_float(r[c & 1][j + 2]), sc.z, bb.z);
            v[j + 3] = fmaf(__uint_as_float(r[c & 1][j + 3]), sc.w, bb.w);
          } else {  // packed fp32x2 adds (FADD2)
            gf2_unpack(gf2_add(gf2(__uint_as_float(r[c & 1][j + 0]), __uint_as_float(r[c & 1][j + 1])), gf2(bb.x, bb.y)),
                       v[j + 0], v[j + 1]);
            gf2_unpack(gf2_add(gf2(__uint_as_float(r[c & 1][j + 2]), __uint_as_float(r[c & 1][j + 3])), gf2(bb.z, bb.w)),
                       v[j + 2], v[j + 3]);
          }
        }
        if constexpr (RES) {
          const int s = c % NRES;
          mbar_wait(&rbar[s], (rpar >> s) & 1u);
          rpar ^= 1u << s;
          const uint8_t* src = rslot + s * SP::RES_SLOT;
          if constexpr (SP::LN16) {  // 32 fp16 of this row: four 16-byte pieces, SWIZZLE_64B
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint4 rr = *reinterpret_cast<const uint4*>(src + sw64_off(lane, k));
              const uint32_t w4[4] = {rr.x, rr.y, rr.z, rr.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w4[e]));
                gf2_unpack(gf2_add(gf2(v[8 * k + 2 * e], v[8 * k + 2 * e + 1]), gf2(f.x, f.y)), v[8 * k + 2 * e],
                           v[8 * k + 2 * e + 1]);
              }
            }
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float4 rr = *reinterpret_cast<const float4*>(src + sw128_off(lane, k));
              v[4 * k] += rr.x; v[4 * k + 1] += rr.y; v[4 * k + 2] += rr.z; v[4 * k + 3] += rr.w;
            }
          }
          __syncwarp();  // every lane has read slot s
          if (c + NRES < CH) load_res(row0, col0 + NRES * 32, c + NRES);
        }
        if constexpr (LN) {
          // chunk statistics, merged into the running (n, mean, M2); v kept in TMEM
          // (kept scalar and sequential: its summation order is part of the row's result bits, and
          // a pairwise order moved the seed-5 residual16 parity case from 0.63% to 1.2%)
          float sum = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) sum += v[j];
          const float cm = sum * (1.0f / 32.0f);
          float m2 = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) { const float d = v[j] - cm; m2 = fmaf(d, d, m2); }
          if (c == 0) { st_n = 32.f; st_mean = cm; st_m2 = m2; }
          else chan_merge(st_n, st_mean, st_m2, 32.f, cm, m2);
          uint32_t w[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(v[j]);
          tmem_st_32x32b_x32(taddr + c * 32, w);
        } else {
          uint8_t* b = next_stage();
          if constexpr (EPI == EPI_BIAS_RESID_F32) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              *reinterpret_cast<float4*>(b + sw128_off(lane, k)) =
                  make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
          } else {
            if constexpr (EPI == EPI_BIAS_GELU_BF16) {
#pragma unroll
              // 16-bit paths: the sigmoid form on packed fp32x2 (A/B: FFN1 2.19 -> 1.93-2.08 ms per cfg2
              // step vs the scalar form; the 1-MUFU tanh form measured 2.24-2.28); FP8: the tanh form
              if constexpr (F8) {
                for (int j = 0; j < 32; ++j) v[j] = gelu_tanh_form(v[j]);
              } else {
                for (int j = 0; j < 32; j += 2) gelu_fast2(v[j], v[j + 1]);
              }
            }
            if constexpr (F8 && EPI == EPI_BIAS_GELU_BF16) {
              stage_e4m3_row(b, lane, v, args.out_scale);
            } else {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                *reinterpret_cast<uint4*>(b + sw64_off(lane, k)) =
                    make_uint4(pack16x2<F16>(v[8 * k + 0], v[8 * k + 1]), pack16x2<F16>(v[8 * k + 2], v[8 * k + 3]),
                               pack16x2<F16>(v[8 * k + 4], v[8 * k + 5]), pack16x2<F16>(v[8 * k + 6], v[8 * k + 7]));
            }
          }
          issue_store(b, row0, col0);
        }
      }
      if (gt_me) { const long long g2 = GT_CLK(); GT_ADD(5, g2 - g1); g1 = g2; }
      if constexpr (LN) {
        tc_wait_st();
        // pass 1 has consumed this tile's residual: start the next tile's first boxes now so the
        // loads overlap the statistics exchange and pass 2 (not when pass 2 stages in the slot)
        if (!SP::F32_IN_RES && t + ncl < num_iter_tiles) {
          int m2, n2;
          tile_mn(t + ncl, m2, n2);
          const int row0n = m2 * 2 * BM + hrow * BM + q * 32;
#pragma unroll
          for (int c = 0; c < NRES && c < CH; ++c) load_res(row0n, n2 * BN + cbase + c * 32, c);
          res_prefetched = true;
        }
        const int slot = it & 1;
        const uint32_t sph = (it >> 1) & 1;
        part[half * 128 + row_in_tile] = make_float2(st_mean, st_m2);
        named_bar_sync(2, EW * 32);
        float tn = 0.f, tmean = 0.f, tm2 = 0.f;
        if constexpr (GX) {
          // this CTA's statistics -> global memory; one release (fence + counter) per CTA; every
          // CTA of the row group then reads the num_n partials in n order (= the cluster order)
          float2* gs = args.gstats + (static_cast<size_t>(m) * num_n * 2 + hrow) * 128;
          uint32_t* flag = args.gflag + m * 2 + hrow;
          if (half == 0) {
            float cn = st_n, cmean = st_mean, cm2 = st_m2;
            const float2 o = part[128 + row_in_tile];
            chan_merge(cn, cmean, cm2, st_n, o.x, o.y);
            gs[n * 2 * 128 + row_in_tile] = make_float2(cmean, cm2);
          }
          named_bar_sync(3, EW * 32);  // all epilogue warps: the half-0 stores precede the release
          if (ew == 0 && lane == 0) {
            __threadfence();
            atomicAdd(flag, 1u);
          }
          if (lane == 0) {
            const unsigned long long t0 = gx_globaltimer();
            while (ld_acquire_gpu_u32(flag) < static_cast<uint32_t>(num_n)) {
              __nanosleep(64);
              if (gx_globaltimer() - t0 > 2000000000ull) {  // a missing peer: no hang, a sticky error
                if (args.err) atomicOr(args.err, ERR_GX_TIMEOUT);
                break;
              }
            }
          }
          __syncwarp();
          for (int p = 0; p < num_n; ++p) {
            const float2 s2 = __ldcg(gs + p * 2 * 128 + row_in_tile);
            if (p == 0) { tn = static_cast<float>(BN); tmean = s2.x; tm2 = s2.y; }
            else chan_merge(tn, tmean, tm2, static_cast<float>(BN), s2.x, s2.y);
          }
          if (gt_me) { const long long g2 = GT_CLK(); GT_ADD(6, g2 - g1); g1 = g2; }
        } else {
        if (half == 0) {
          // this CTA's statistics over its BN columns -> every CTA holding the same rows
          float cn = st_n, cmean = st_mean, cm2 = st_m2;
          const float2 o = part[128 + row_in_tile];
          chan_merge(cn, cmean, cm2, st_n, o.x, o.y);
          const uint32_t lslot = smem_u32(&stats[(slot * kMaxCluster + pair_in_cluster) * 128 + row_in_tile]);
          const uint32_t lbar = smem_u32(&sfull[slot]);
#ifdef ELIS_LN_RELEASE_ARRIVES
          for (int pp = 0; pp < cpairs; ++pp)
            st_cluster_f32x2(mapa_shared(lslot, static_cast<uint32_t>(2 * pp + hrow)), cmean, cm2);
          __syncwarp();
          if (lane == 0)  // release is cumulative over the warp's DSMEM stores ordered by __syncwarp
            for (int pp = 0; pp < cpairs; ++pp)
              mbar_arrive_remote_release(mapa_shared(lbar, static_cast<uint32_t>(2 * pp + hrow)));
#else
          // st.async: each row's (mean, M2) lands in every row peer and completes 8 bytes on its
          // barrier -- no release fence on the epilogue's critical path
          for (int pp = 0; pp < cpairs; ++pp) {
            const uint32_t r = static_cast<uint32_t>(2 * pp + hrow);
            st_async_f32x2(mapa_shared(lslot, r), cmean, cm2, mapa_shared(lbar, r));
          }
#endif
        }
#ifdef ELIS_LN_RELEASE_ARRIVES
        if (lane == 0) mbar_wait_acquire_cluster(&sfull[slot], sph);
#else
        // this CTA expects 128 rows x 8 bytes from each of the cpairs row peers (itself included)
        if (ew == 0 && lane == 0) mbar_arrive_expect_tx(&sfull[slot], static_cast<uint32_t>(cpairs) * 128u * 8u);
        if (lane == 0) mbar_wait(&sfull[slot], sph);
#endif
        __syncwarp();
        if (gt_me) { const long long g2 = GT_CLK(); GT_ADD(6, g2 - g1); g1 = g2; }
        // merge the cpairs partials in pair order (identical on every CTA) -> mean, rstd
        for (int p = 0; p < cpairs; ++p) {
          const float2 s2 = stats[(slot * kMaxCluster + p) * 128 + row_in_tile];
          if (p == 0) { tn = static_cast<float>(BN); tmean = s2.x; tm2 = s2.y; }
          else chan_merge(tn, tmean, tm2, static_cast<float>(BN), s2.x, s2.y);
        }
        }  // cluster exchange
        const float rstd = 1.0f / sqrtf(tm2 / tn + args.eps);
        tmem_ld_32x32b_x32(taddr, r[0]);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          tc_wait_ld();
          if (c + 1 < CH) tmem_ld_32x32b_x32(taddr + (c + 1) * 32, r[(c + 1) & 1]);
          const int tcol = cbase + c * 32;
          const int col0 = n * BN + tcol;
          float y[32];
#pragma unroll
          for (int j = 0; j < 32; j += 4) {  // (v - mean) * rstd * gamma + beta on packed fp32x2
            const float4 g = *reinterpret_cast<const float4*>(sgam + tcol + j);
            const float4 be = *reinterpret_cast<const float4*>(sbet + tcol + j);
            const unsigned long long nm = gf2(-tmean, -tmean), rs = gf2(rstd, rstd);
            gf2_unpack(gf2_fma(gf2_mul(gf2_add(gf2(__uint_as_float(r[c & 1][j + 0]), __uint_as_float(r[c & 1][j + 1])), nm), rs),
                               gf2(g.x, g.y), gf2(be.x, be.y)),
                       y[j + 0], y[j + 1]);
            gf2_unpack(gf2_fma(gf2_mul(gf2_add(gf2(__uint_as_float(r[c & 1][j + 2]), __uint_as_float(r[c & 1][j + 3])), nm), rs),
                               gf2(g.z, g.w), gf2(be.z, be.w)),
                       y[j + 2], y[j + 3]);
          }
          uint8_t* b = next_stage();   // NSTG = 1: every earlier store (incl. from the slot) has read
          uint8_t* b32 = SP::F32_IN_RES ? rslot : b;
          if constexpr (SP::OUT_F32) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              *reinterpret_cast<float4*>(b32 + sw128_off(lane, k)) =
                  make_float4(y[4 * k], y[4 * k + 1], y[4 * k + 2], y[4 * k + 3]);
          }
          uint8_t* bb = (SP::F32_IN_RES || !SP::OUT_F32) ? b : b + SP::STG_F32;
          if constexpr (F8) {
            stage_e4m3_row(bb, lane, y, args.out_scale);
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              *reinterpret_cast<uint4*>(bb + sw64_off(lane, k)) =
                  make_uint4(pack16x2<F16>(y[8 * k + 0], y[8 * k + 1]), pack16x2<F16>(y[8 * k + 2], y[8 * k + 3]),
                             pack16x2<F16>(y[8 * k + 4], y[8 * k + 5]), pack16x2<F16>(y[8 * k + 6], y[8 * k + 7]));
          }
          issue_store(b, row0, col0, b32);
        }
        if (gt_me) GT_ADD(7, GT_CLK() - g1);
      }
      tc_fence_before();
      __syncwarp();
      // accumulator free: every lane's tcgen05.ld completed (wait::ld), so a relaxed arrive suffices
      if (lane == 0) mbar_arrive_remote_relaxed(tempty_leader + acc * 8);
    }
    if (lane == 0) tma_store_wait_all<0>();
    if (warp == 4 && lane == 0) {
      GT_ADD(8, GT_CLK() - gepi);
#ifdef ELIS_GEMM_TRACE
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      if (blockIdx.x < kGemmTraceCtas) g_gemm_trace[blockIdx.x * 16 + 10] = smid;
#endif
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
  }
}

template <int BN, int EPI, bool DEEP, int PREC = 0, bool GX = false>
cudaError_t launch_bn(const GemmPlan& g, int num_sms, cudaStream_t st) {
  using SP = SmemPlan<BN, EPI, DEEP, PREC>;
  auto kern = k_gemm_tc<BN, EPI, DEEP, PREC, GX>;
  cudaError_t e = cudaSuccess;
  // launch attributes: set once per device (each cudaFuncSetAttribute costs ~1 us of host time)
  const bool first = !attr_once(reinterpret_cast<const void*>(kern));
  if (first) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SP::SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  const int num_m = (g.args.M + 2 * BM - 1) / (2 * BM);
  const int num_n = g.args.N / BN;
  const bool ln = (EPI == EPI_BIAS_RESID_LN || EPI == EPI_BIAS_RESID16_LN) && !GX;  // cluster LN
  const int cpairs = ln ? num_n : 1;
  const int csize = 2 * cpairs;
  if (cpairs > kMaxCluster) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(gemm_threads<EPI, PREC>());
  cfg.dynamicSmemBytes = SP::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  pdl_attr(attr[1]);
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_enabled() && !GX) ? 2 : 1;  // GX spins on the whole grid being co-resident
  if (first && csize > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  // number of clusters that can be co-resident (one CTA per SM)
  // per (BN, EPI, DEEP, F8) instantiation and device (the GX exchange needs the whole grid co-resident)
  constexpr int kDevCache = 16;
  static int max_clusters[kDevCache][2 * kMaxCluster + 1] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int mc_here = (dev < kDevCache) ? max_clusters[dev][csize] : 0;
  if (mc_here == 0) {
    cudaLaunchConfig_t q = cfg;
    q.gridDim = dim3(csize * (num_sms / csize));
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &q) != cudaSuccess || mc <= 0) mc = num_sms / csize;
    mc_here = mc;
    if (dev < kDevCache) max_clusters[dev][csize] = mc;
  }
  const int work = ln ? num_m : num_m * num_n;
  int ncl = work < mc_here ? work : mc_here;
  if constexpr (GX) {
    // the num_n pairs of a row group take consecutive tiles: a multiple of num_n pairs keeps each
    // group inside one step of the static schedule; the arrival counters start at 0
    if (ncl >= num_n) ncl -= ncl % num_n;
    e = cudaMemsetAsync(g.args.gflag, 0, static_cast<size_t>(num_m) * 2 * sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
  }
  cfg.gridDim = dim3(csize * ncl);
  e = cudaLaunchKernelEx(&cfg, kern, g.tmA, g.tmB, g.tmR, g.tmO, g.tmOb, g.args);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

int gemm_block_n(int N) { return (N % 256 == 0) ? 256 : 128; }

cudaError_t launch_gemm(const GemmPlan& g, int num_sms, cudaStream_t st) {
  if (g.args.M <= 0) return cudaSuccess;
  const bool b256 = gemm_block_n(g.args.N) == 256;
  const bool deep = g.args.K >= 2048;  // long mainloop: a 4th operand stage beats a 2nd residual slot
  if (g.f8) {  // E4M3 operands: the BGE-base / large shapes (every N a multiple of 256)
    if (!b256) return cudaErrorInvalidValue;
    switch (g.epi) {
      case EPI_BIAS_BF16: return launch_bn<256, EPI_BIAS_BF16, false, 1>(g, num_sms, st);
      case EPI_BIAS_GELU_BF16: return launch_bn<256, EPI_BIAS_GELU_BF16, false, 1>(g, num_sms, st);
      case EPI_BIAS_RESID_LN:
        return deep ? launch_bn<256, EPI_BIAS_RESID_LN, true, 1>(g, num_sms, st)
                    : launch_bn<256, EPI_BIAS_RESID_LN, false, 1>(g, num_sms, st);
      default: return cudaErrorInvalidValue;
    }
  }
  if (g.f16) {  // fp16 operands and 16-bit outputs
    if (g.bn128) {  // small-M plans (gemm_plan_bn128)
      switch (g.epi) {
        case EPI_BIAS_BF16: return launch_bn<128, EPI_BIAS_BF16, false, 2>(g, num_sms, st);
        case EPI_BIAS_GELU_BF16: return launch_bn<128, EPI_BIAS_GELU_BF16, false, 2>(g, num_sms, st);
        default: return cudaErrorInvalidValue;
      }
    }
    if (!b256) return cudaErrorInvalidValue;
    switch (g.epi) {
      case EPI_BIAS_RESID16_LN:
        if (deep && g.args.gstats) return launch_bn<256, EPI_BIAS_RESID16_LN, true, 2, true>(g, num_sms, st);
        if (g.args.gstats) return launch_bn<256, EPI_BIAS_RESID16_LN, false, 2, true>(g, num_sms, st);
        return deep ? launch_bn<256, EPI_BIAS_RESID16_LN, true, 2>(g, num_sms, st)
                    : launch_bn<256, EPI_BIAS_RESID16_LN, false, 2>(g, num_sms, st);
      case EPI_BIAS_BF16: return launch_bn<256, EPI_BIAS_BF16, false, 2>(g, num_sms, st);
      case EPI_BIAS_GELU_BF16: return launch_bn<256, EPI_BIAS_GELU_BF16, false, 2>(g, num_sms, st);
      case EPI_BIAS_RESID_LN:
        return deep ? launch_bn<256, EPI_BIAS_RESID_LN, true, 2>(g, num_sms, st)
                    : launch_bn<256, EPI_BIAS_RESID_LN, false, 2>(g, num_sms, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (g.epi) {
    case EPI_BIAS_BF16:
      return b256 ? launch_bn<256, EPI_BIAS_BF16, false>(g, num_sms, st)
                  : launch_bn<128, EPI_BIAS_BF16, false>(g, num_sms, st);
    case EPI_BIAS_GELU_BF16:
      return b256 ? launch_bn<256, EPI_BIAS_GELU_BF16, false>(g, num_sms, st)
                  : launch_bn<128, EPI_BIAS_GELU_BF16, false>(g, num_sms, st);
    case EPI_BIAS_RESID_F32:
      return b256 ? launch_bn<256, EPI_BIAS_RESID_F32, false>(g, num_sms, st)
                  : launch_bn<128, EPI_BIAS_RESID_F32, false>(g, num_sms, st);
    case EPI_BIAS_RESID_LN:
      if (deep)
        return b256 ? launch_bn<256, EPI_BIAS_RESID_LN, true>(g, num_sms, st)
                    : launch_bn<128, EPI_BIAS_RESID_LN, true>(g, num_sms, st);
      return b256 ? launch_bn<256, EPI_BIAS_RESID_LN, false>(g, num_sms, st)
                  : launch_bn<128, EPI_BIAS_RESID_LN, false>(g, num_sms, st);
    default: return cudaErrorInvalidValue;
  }
}

// ----------------------------------------------------------------------------- tensor maps
namespace {
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

bool make_tmap_2d(CUtensorMap* m, CUtensorMapDataType dt, uint32_t esize, const void* ptr, uint64_t rows,
                  uint64_t cols, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle sw) {
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * esize};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
}  // namespace

bool make_tmap_bf16_kmajor(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  return make_tmap_bf16_box(m, ptr, rows, cols, BK, box_rows);
}

bool make_tmap_bf16_box(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_cols,
                        uint32_t box_rows) {
  return make_tmap_2d(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, rows, cols, box_cols, box_rows,
                      CU_TENSOR_MAP_SWIZZLE_128B);
}

bool make_tmap_f32_box(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_cols,
                       uint32_t box_rows) {
  return make_tmap_2d(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ptr, rows, cols, box_cols, box_rows,
                      CU_TENSOR_MAP_SWIZZLE_128B);
}

bool make_gemm_plan(GemmPlan* g, const void* A, uint64_t a_rows, const void* W, const float* bias,
                    const float* resid, void* out, int M, int N, int K, int epi) {
  if (N % 128 != 0 || K % BK != 0 || M < 0) return false;
  if ((epi == EPI_BIAS_RESID_LN || epi == EPI_BIAS_RESID16_LN) && N / gemm_block_n(N) > kMaxCluster) return false;
  g->epi = epi;
  g->f8 = 0;
  g->f16 = 0;
  g->args = GemmArgs{};
  g->args.M = M;
  g->args.N = N;
  g->args.K = K;
  g->args.bias = bias;
  g->args.resid = resid;
  g->args.out = out;
  if (!make_tmap_bf16_kmajor(&g->tmA, A, a_rows, K, BM)) return false;
  if (!make_tmap_bf16_kmajor(&g->tmB, W, N, K, gemm_block_n(N) / 2)) return false;
  const bool res = epi == EPI_BIAS_RESID_F32 || epi == EPI_BIAS_RESID_LN;
  // epilogue boxes: fp32 32 x 32 (128 B rows, SWIZZLE_128B); bf16 32 x 32 (64 B rows, SWIZZLE_64B)
  if (epi == EPI_BIAS_RESID16_LN) {  // residual in and normalised rows out: the same 16-bit buffer
    if (!resid || !make_tmap_2d(&g->tmR, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, resid, a_rows, N, kBox, kBox,
                                CU_TENSOR_MAP_SWIZZLE_64B))
      return false;
    if (!make_tmap_2d(&g->tmO, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, a_rows, N, kBox, kBox,
                      CU_TENSOR_MAP_SWIZZLE_64B))
      return false;
    g->tmOb = g->tmO;
  } else if (res) {
    if (!resid || !make_tmap_2d(&g->tmR, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, resid, a_rows, N, kBox, kBox,
                                CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
    if (!make_tmap_2d(&g->tmO, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, a_rows, N, kBox, kBox,
                      CU_TENSOR_MAP_SWIZZLE_128B))
      return false;
    g->tmOb = g->tmO;
  } else {
    if (!make_tmap_2d(&g->tmO, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, a_rows, N, kBox, kBox,
                      CU_TENSOR_MAP_SWIZZLE_64B))
      return false;
    g->tmR = g->tmO;
    g->tmOb = g->tmO;
  }
  return true;
}

bool make_gemm_plan_f8(GemmPlan* g, const void* A, uint64_t a_rows, const void* W, const float* colscale,
                       const float* bias, const float* resid, void* out, int M, int N, int K, int epi,
                       float out_scale) {
  if (N % 256 != 0 || K % (2 * BK) != 0 || M < 0 || !colscale || epi == EPI_BIAS_RESID_F32) return false;
  if (!make_gemm_plan(g, A, a_rows, W, bias, resid, out, M, N, K, epi)) return false;
  g->f8 = 1;
  g->args.colscale = colscale;
  g->args.out_scale = out_scale;
  // operands: 128 E4M3 (= 128 bytes, one SWIZZLE_128B row) x rows boxes
  if (!make_tmap_2d(&g->tmA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, A, a_rows, K, 2 * BK, BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_tmap_2d(&g->tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, W, N, K, 2 * BK, gemm_block_n(N) / 2,
                    CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  if (epi == EPI_BIAS_GELU_BF16) {  // E4M3 output, 32 x 32-byte boxes (SWIZZLE_32B)
    if (!make_tmap_2d(&g->tmO, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, out, a_rows, N, kBox, kBox,
                      CU_TENSOR_MAP_SWIZZLE_32B))
      return false;
    g->tmR = g->tmO;
    g->tmOb = g->tmO;
  }
  return true;
}

bool gemm_plan_bn128(GemmPlan* g, const void* W) {
  if (!g->f16 || g->f8 || (g->epi != EPI_BIAS_BF16 && g->epi != EPI_BIAS_GELU_BF16)) return false;
  if (!make_tmap_bf16_kmajor(&g->tmB, W, g->args.N, g->args.K, 128 / 2)) return false;
  g->bn128 = 1;
  return true;
}

bool gemm_plan_set_head_major(GemmPlan* g, void* out, uint64_t rows) {
  if (g->epi != EPI_BIAS_BF16 || g->args.N % 64 != 0) return false;
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  // [planes = N/64][rows][64] bf16; box 32 columns x 32 rows x 1 plane, 64-byte rows (SWIZZLE_64B)
  cuuint64_t dims[3] = {64, rows, static_cast<cuuint64_t>(g->args.N / 64)};
  cuuint64_t strides[2] = {64 * 2, rows * 64 * 2};
  cuuint32_t box[3] = {kBox, kBox, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&g->tmO, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, out, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  g->args.out = out;
  g->args.out_head_major = 1;
  return r == CUDA_SUCCESS;
}

bool gemm_plan_set_ln(GemmPlan* g, uint16_t* outb, const float* gamma, const float* beta, float eps,
                      uint64_t rows) {
  g->args.outb = outb;
  g->args.gamma = gamma;
  g->args.beta = beta;
  g->args.eps = eps;
  if (g->f8)
    return make_tmap_2d(&g->tmOb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, outb, rows, g->args.N, kBox, kBox,
                        CU_TENSOR_MAP_SWIZZLE_32B);
  return make_tmap_2d(&g->tmOb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, outb, rows, g->args.N, kBox, kBox,
                      CU_TENSOR_MAP_SWIZZLE_64B);
}

#ifdef ELIS_GEMM_TRACE
extern "C" int elis_debug_gemm_trace(long long* host, size_t n, int reset) {
  if (reset) {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, g_gemm_trace);
    return static_cast<int>(cudaMemset(p, 0, sizeof(g_gemm_trace)));
  }
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_gemm_trace, (n < kGemmTraceCtas * 16 ? n : kGemmTraceCtas * 16) * 8));
}
#endif

}  // namespace elis
