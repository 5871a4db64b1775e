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
//     tcgen05.mma M=256 for both, each CTA's TMEM holds its 128 accumulator rows.  Per
//     CTA this halves the B bytes fetched per FLOP (the single-CTA 128 x 256 tile was L2
//     bandwidth bound: 87 FLOP per L2 byte -> 131 with pairs);
//   * persistent grid, static tile schedule; warp 0 = TMA producer (SWIZZLE_128B slabs,
//     mbarrier ring, completion counted on the leader's barrier), warp 1 (leader) = the
//     single-thread MMA issuer, warp 2 = TMEM allocator, warps 4..11 = epilogue (two
//     warps per TMEM lane quarter, each owning half of the tile's columns);
//   * two TMEM accumulators (2 x BN columns): the epilogue of tile i overlaps the mainloop
//     of tile i+1;
//   * ragged M handled by TMA out-of-bounds zero fill + masked stores (no padding of T);
//   * no split-K: every output row depends on its own A row only (batch invariance).
//
// EPI_BIAS_RESID_LN (attention-output and FFN2 + LayerNorm, rows a5+a6 / a8): a row of
// H = 768 / 1024 columns spans CS = H / BN pairs, launched as one cluster of 2 x CS CTAs.
// Each CTA adds bias + fp32 residual (prefetched by cp.async while the MMA runs), keeps v
// in TMEM (tcgen05.st), computes per-row (mean, M2) over its columns and pushes them into
// every peer's shared memory over DSMEM (st.shared::cluster + remote mbarrier arrive);
// every CTA then merges the CS partials in rank order (Chan) and normalises its columns.
// The fp32 residual stream is updated in place and the bf16 copy for the next GEMM is
// written in the same pass: 10 B/element of epilogue traffic instead of 18 B with a
// separate LayerNorm kernel.
#include "common.cuh"
#include "kernels.cuh"

namespace elis {

namespace {

constexpr int BM = 128;  // rows per CTA (256 per pair)
constexpr int BK = 64;
constexpr int kEpiWarps = 8;
constexpr int kGemmThreads = 128 + kEpiWarps * 32;  // 4 control warps + 8 epilogue warps
constexpr int kMaxCluster = 4;                       // max N-tiles (pairs) per LN row

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_ROWS = BN / 2;              // this CTA's half of the B slab
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr int CHUNKS_PER_WARP = BN / 64;   // 32-column chunks per epilogue warp
};
// Shared-memory plan.  RES (the epilogue reads an fp32 residual) trades operand stages for
// a per-warp double-buffered residual staging area filled by cp.async ahead of use.
template <int BN, bool RES>
struct SmemPlan {
  static constexpr int STAGES = RES ? 4 : 6;
  static constexpr int RES_BYTES = RES ? kEpiWarps * 2 * 32 * 32 * 4 : 0;  // [warp][2][32 rows][32 f32]
  // barriers (512) + LN stats[2][kMaxCluster][128] f2 + part[2][128] f2 + bias/gamma/beta[256] f32
  static constexpr int AUX_BYTES = 512 + 2 * kMaxCluster * 128 * 8 + 2 * 128 * 8 + 3 * 256 * 4;
  static constexpr int SMEM_BYTES = STAGES * GemmCfg<BN>::STAGE_BYTES + RES_BYTES + AUX_BYTES + 1024;
};

// GELU(x) = x * Phi(x) (erf form).  Phi is evaluated as sigmoid(x * (c0 + c1 x^2 + c2 x^4))
// with minimax coefficients fitted to the exact erf form: max |error| of GELU over all x is
// 2.6e-5 (scripts/fit_gelu.py), < 1/75 of the bf16 rounding of the output this epilogue
// writes.  10 instructions incl. 2 MUFU instead of ~28 for erff (the FFN1 epilogue is
// instruction-issue bound).
ELIS_DEV float gelu_fast(float x) {
  constexpr float kL2E = 1.4426950408889634f;
  constexpr float c0 = -1.5950205882421884f * kL2E, c1 = -0.07400664121448398f * kL2E,
                  c2 = 0.0007022165804436097f * kL2E;
  const float xc = fminf(fmaxf(x, -9.0f), 9.0f);
  const float x2 = xc * xc;
  const float p = fmaf(fmaf(c2, x2, c1), x2, c0);   // -(c0 + c1 x^2 + c2 x^4) * log2(e)
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(xc * p));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return x * r;
}

// Chan et al. merge of (count, mean, M2) partial statistics.
ELIS_DEV void chan_merge(float& n_a, float& mean_a, float& m2_a, float n_b, float mean_b, float m2_b) {
  const float n = n_a + n_b;
  const float d = mean_b - mean_a;
  mean_a = mean_a + d * (n_b / n);
  m2_a = m2_a + m2_b + d * d * (n_a * n_b / n);
  n_a = n;
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const GemmArgs args) {
  using C = GemmCfg<BN>;
  constexpr bool LN = (EPI == EPI_BIAS_RESID_LN);
  constexpr bool RES = LN || (EPI == EPI_BIAS_RESID_F32);
  using SP = SmemPlan<BN, RES>;
  constexpr int STAGES = SP::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * C::A_BYTES;
  float* res_base = reinterpret_cast<float*>(sB + STAGES * C::B_BYTES);
  uint8_t* aux = reinterpret_cast<uint8_t*>(res_base) + SP::RES_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(aux);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;  // LN: stats slots filled by every CTA of the row group
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sfull + 2);
  float2* stats = reinterpret_cast<float2*>(aux + 512);   // [2][kMaxCluster][128]
  float2* part = stats + 2 * kMaxCluster * 128;            // [2 halves][128]
  float* sbias = reinterpret_cast<float*>(part + 2 * 128);  // [256]
  float* sgam = sbias + 256;                                // [256]
  float* sbet = sgam + 256;                                 // [256]

  const int warp = warp_id();
  const int lane = lane_id();
  const int M = args.M, N = args.N, K = args.K;
  const int num_m = (M + 2 * BM - 1) / (2 * BM);  // 256-row pair tiles
  const int num_n = N / BN;
  const int num_k = K / BK;
  // Cluster = (LN ? num_n : 1) pairs.  CTA rank r: pair r >> 1, half (row half / B half) r & 1.
  const int crank = static_cast<int>(cluster_ctarank());
  const int cpairs = LN ? num_n : 1;
  const int pair_in_cluster = crank >> 1;
  const int hrow = crank & 1;              // which 128-row half of the pair tile
  const bool leader = hrow == 0;
  const int leader_rank = crank & ~1;
  const int cid = static_cast<int>(blockIdx.x) / (2 * cpairs);
  const int ncl = static_cast<int>(gridDim.x) / (2 * cpairs);
  const int num_iter_tiles = LN ? num_m : num_m * num_n;
  auto tile_mn = [&](int t, int& m, int& n) {
    if (LN) { m = t; n = pair_in_cluster; } else { m = t / num_n; n = t % num_n; }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiWarps);  // one arrive per epilogue warp of both CTAs (leader's copy used)
      mbar_init(&sfull[a], 4 * cpairs);      // one arrive per half-0 epilogue warp of every row peer
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs); bytes counted on the leader's full barrier
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = cid; t < num_iter_tiles; t += ncl) {
        int m, n;
        tile_mn(t, m, n);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[s], ph ^ 1u);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * C::STAGE_BYTES);
          const uint32_t bar = mapa_shared(smem_u32(&full[s]), leader_rank);
          tma_load_2d_pair(sA + s * C::A_BYTES, &tmA, bar, kb * BK, m * 2 * BM + hrow * BM);
          tma_load_2d_pair(sB + s * C::B_BYTES, &tmB, bar, kb * BK, n * BN + hrow * C::B_ROWS);
          if (++s == STAGES) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA, one thread) for the pair
    if (leader && lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16_f32(2 * BM, BN);
      const uint16_t mask = static_cast<uint16_t>(3u << leader_rank);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int t = cid; t < num_iter_tiles; t += ncl, ++it) {
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait_acquire_cluster(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t da = make_sw128_desc(smem_u32(sA + s * C::A_BYTES));
          const uint64_t db = make_sw128_desc(smem_u32(sB + s * C::B_BYTES));
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // advance 16 bf16 = 32 bytes along K inside the 128-byte swizzle row
            tc_mma_f16_pair(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          tc_commit_pair_mc(&empty[s], mask);
          if (++s == STAGES) { s = 0; ph ^= 1u; }
        }
        tc_commit_pair_mc(&tfull[acc], mask);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> global (each CTA: its 128 rows)
    constexpr int CH = C::CHUNKS_PER_WARP;
    const int ew = warp - 4;             // 0..7
    const int q = warp & 3;              // TMEM lane quarter this warp may access
    const int half = ew >> 2;            // which half of the tile's columns
    const int row_in_tile = q * 32 + lane;
    const int etid = ew * 32 + lane;     // 0..255
    float* rbuf = res_base + ew * (2 * 32 * 32) + lane * 32;   // this thread's row in buffer 0
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), leader_rank);
    auto stage_vectors = [&](int n) {    // bias (+ gamma, beta) of tile columns -> shared memory
      if (etid < BN) {
        sbias[etid] = __ldg(args.bias + n * BN + etid);
        if constexpr (LN) {
          sgam[etid] = __ldg(args.gamma + n * BN + etid);
          sbet[etid] = __ldg(args.beta + n * BN + etid);
        }
      }
    };
    // residual chunk c of this thread's row -> buffer (c & 1), 16-byte pieces XOR-swizzled by row
    auto prefetch_res = [&](int row, int col0, int c) {
      const float* src = args.resid + static_cast<size_t>(row) * N + col0;
      float* dst = rbuf + (c & 1) * (32 * 32);
#pragma unroll
      for (int k = 0; k < 8; ++k) cp_async16(dst + ((k ^ (lane & 7)) * 4), src + 4 * k, true);
    };
    if constexpr (LN) {
      stage_vectors(pair_in_cluster);
      named_bar_sync(1, kEpiWarps * 32);
    }
    int it = 0;
    for (int t = cid; t < num_iter_tiles; t += ncl, ++it) {
      int m, n;
      tile_mn(t, m, n);
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int row = m * 2 * BM + hrow * BM + row_in_tile;
      const bool row_ok = row < M;
      const int cbase = half * (BN / 2);  // first tile column of this warp
      if constexpr (RES) {                // residual does not depend on the MMA: fetch it now
#pragma unroll
        for (int c = 0; c < 2 && c < CH; ++c) {
          if (row_ok) prefetch_res(row, n * BN + cbase + c * 32, c);
          cp_async_commit();
        }
      }
      if constexpr (!LN) {
        named_bar_sync(1, kEpiWarps * 32);  // previous tile's readers of sbias are done
        stage_vectors(n);
        named_bar_sync(1, kEpiWarps * 32);
      }
      mbar_wait(&tfull[acc], aph);
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
          v[j + 0] = __uint_as_float(r[c & 1][j + 0]) + bb.x;
          v[j + 1] = __uint_as_float(r[c & 1][j + 1]) + bb.y;
          v[j + 2] = __uint_as_float(r[c & 1][j + 2]) + bb.z;
          v[j + 3] = __uint_as_float(r[c & 1][j + 3]) + bb.w;
        }
        if constexpr (RES) {
          if (c + 1 < CH) cp_async_wait<1>(); else cp_async_wait<0>();
          if (row_ok) {
            const float* src = rbuf + (c & 1) * (32 * 32);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float4 rr = *reinterpret_cast<const float4*>(src + ((k ^ (lane & 7)) * 4));
              v[4 * k] += rr.x; v[4 * k + 1] += rr.y; v[4 * k + 2] += rr.z; v[4 * k + 3] += rr.w;
            }
            if (c + 2 < CH) prefetch_res(row, col0 + 64, c + 2);
          }
          if (c + 2 < CH) cp_async_commit();
        }
        if constexpr (LN) {
          // chunk statistics, merged into the running (n, mean, M2); v kept in TMEM
          float s = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) s += v[j];
          const float cm = s * (1.0f / 32.0f);
          float m2 = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) { const float d = v[j] - cm; m2 = fmaf(d, d, m2); }
          if (c == 0) { st_n = 32.f; st_mean = cm; st_m2 = m2; }
          else chan_merge(st_n, st_mean, st_m2, 32.f, cm, m2);
          uint32_t w[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(v[j]);
          tmem_st_32x32b_x32(taddr + c * 32, w);
        } else if (row_ok) {
          if constexpr (EPI == EPI_BIAS_RESID_F32) {
            float4* o4 = reinterpret_cast<float4*>(static_cast<float*>(args.out) + static_cast<size_t>(row) * N + col0);
#pragma unroll
            for (int j = 0; j < 8; ++j) o4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
            if constexpr (EPI == EPI_BIAS_GELU_BF16) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
            }
            uint4* o4 = reinterpret_cast<uint4*>(static_cast<uint16_t*>(args.out) + static_cast<size_t>(row) * N + col0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              o4[j] = make_uint4(pack_bf16x2(v[8 * j + 0], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                                 pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
          }
        }
      }
      if constexpr (LN) {
        tc_wait_st();
        const int slot = it & 1;
        const uint32_t sph = (it >> 1) & 1;
        part[half * 128 + row_in_tile] = make_float2(st_mean, st_m2);
        named_bar_sync(2, kEpiWarps * 32);
        if (half == 0) {
          // this CTA's statistics over its BN columns -> every CTA holding the same rows
          float cn = st_n, cmean = st_mean, cm2 = st_m2;
          const float2 o = part[128 + row_in_tile];
          chan_merge(cn, cmean, cm2, st_n, o.x, o.y);
          const uint32_t lslot = smem_u32(&stats[(slot * kMaxCluster + pair_in_cluster) * 128 + row_in_tile]);
          const uint32_t lbar = smem_u32(&sfull[slot]);
          for (int pp = 0; pp < cpairs; ++pp)
            st_cluster_f32x2(mapa_shared(lslot, static_cast<uint32_t>(2 * pp + hrow)), cmean, cm2);
          __syncwarp();
          if (lane == 0)  // release is cumulative over the warp's DSMEM stores ordered by __syncwarp
            for (int pp = 0; pp < cpairs; ++pp)
              mbar_arrive_remote_release(mapa_shared(lbar, static_cast<uint32_t>(2 * pp + hrow)));
        }
        if (lane == 0) mbar_wait_acquire_cluster(&sfull[slot], sph);
        __syncwarp();
        // merge the cpairs partials in pair order (identical on every CTA) -> mean, rstd
        float tn = 0.f, tmean = 0.f, tm2 = 0.f;
        for (int p = 0; p < cpairs; ++p) {
          const float2 s2 = stats[(slot * kMaxCluster + p) * 128 + row_in_tile];
          if (p == 0) { tn = static_cast<float>(BN); tmean = s2.x; tm2 = s2.y; }
          else chan_merge(tn, tmean, tm2, static_cast<float>(BN), s2.x, s2.y);
        }
        const float rstd = 1.0f / sqrtf(tm2 / tn + args.eps);
        tmem_ld_32x32b_x32(taddr, r[0]);
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          tc_wait_ld();
          if (c + 1 < CH) tmem_ld_32x32b_x32(taddr + (c + 1) * 32, r[(c + 1) & 1]);
          const int tcol = cbase + c * 32;
          const int col0 = n * BN + tcol;
          if (row_ok) {
            float y[32];
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 g = *reinterpret_cast<const float4*>(sgam + tcol + j);
              const float4 be = *reinterpret_cast<const float4*>(sbet + tcol + j);
              y[j + 0] = (__uint_as_float(r[c & 1][j + 0]) - tmean) * rstd * g.x + be.x;
              y[j + 1] = (__uint_as_float(r[c & 1][j + 1]) - tmean) * rstd * g.y + be.y;
              y[j + 2] = (__uint_as_float(r[c & 1][j + 2]) - tmean) * rstd * g.z + be.z;
              y[j + 3] = (__uint_as_float(r[c & 1][j + 3]) - tmean) * rstd * g.w + be.w;
            }
            float4* o4 = reinterpret_cast<float4*>(static_cast<float*>(args.out) + static_cast<size_t>(row) * N + col0);
#pragma unroll
            for (int j = 0; j < 8; ++j) o4[j] = make_float4(y[4 * j], y[4 * j + 1], y[4 * j + 2], y[4 * j + 3]);
            uint4* ob = reinterpret_cast<uint4*>(args.outb + static_cast<size_t>(row) * N + col0);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              ob[j] = make_uint4(pack_bf16x2(y[8 * j + 0], y[8 * j + 1]), pack_bf16x2(y[8 * j + 2], y[8 * j + 3]),
                                 pack_bf16x2(y[8 * j + 4], y[8 * j + 5]), pack_bf16x2(y[8 * j + 6], y[8 * j + 7]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      // accumulator free: every lane's tcgen05.ld completed (wait::ld), so a relaxed arrive suffices
      if (lane == 0) mbar_arrive_remote_relaxed(tempty_leader + acc * 8);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
  }
}

template <int BN, int EPI>
cudaError_t launch_bn(const GemmPlan& g, int num_sms, cudaStream_t st) {
  using SP = SmemPlan<BN, EPI == EPI_BIAS_RESID_LN || EPI == EPI_BIAS_RESID_F32>;
  auto kern = k_gemm_tc<BN, EPI>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SP::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int num_m = (g.args.M + 2 * BM - 1) / (2 * BM);
  const int num_n = g.args.N / BN;
  const bool ln = EPI == EPI_BIAS_RESID_LN;
  const int cpairs = ln ? num_n : 1;
  const int csize = 2 * cpairs;
  if (cpairs > kMaxCluster) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = SP::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (csize > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  // number of clusters that can be co-resident (one CTA per SM)
  static int max_clusters[2 * kMaxCluster + 1] = {};
  if (max_clusters[csize] == 0) {
    cudaLaunchConfig_t q = cfg;
    q.gridDim = dim3(csize * (num_sms / csize));
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &q) != cudaSuccess || mc <= 0) mc = num_sms / csize;
    max_clusters[csize] = mc;
  }
  const int work = ln ? num_m : num_m * num_n;
  const int ncl = work < max_clusters[csize] ? work : max_clusters[csize];
  cfg.gridDim = dim3(csize * ncl);
  e = cudaLaunchKernelEx(&cfg, kern, g.tmA, g.tmB, g.args);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

int gemm_block_n(int N) { return (N % 256 == 0) ? 256 : 128; }

cudaError_t launch_gemm(const GemmPlan& g, int num_sms, cudaStream_t st) {
  if (g.args.M <= 0) return cudaSuccess;
  const bool b256 = gemm_block_n(g.args.N) == 256;
  switch (g.epi) {
    case EPI_BIAS_BF16:
      return b256 ? launch_bn<256, EPI_BIAS_BF16>(g, num_sms, st) : launch_bn<128, EPI_BIAS_BF16>(g, num_sms, st);
    case EPI_BIAS_GELU_BF16:
      return b256 ? launch_bn<256, EPI_BIAS_GELU_BF16>(g, num_sms, st)
                  : launch_bn<128, EPI_BIAS_GELU_BF16>(g, num_sms, st);
    case EPI_BIAS_RESID_F32:
      return b256 ? launch_bn<256, EPI_BIAS_RESID_F32>(g, num_sms, st)
                  : launch_bn<128, EPI_BIAS_RESID_F32>(g, num_sms, st);
    case EPI_BIAS_RESID_LN:
      return b256 ? launch_bn<256, EPI_BIAS_RESID_LN>(g, num_sms, st)
                  : launch_bn<128, EPI_BIAS_RESID_LN>(g, num_sms, st);
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
}  // namespace

bool make_tmap_bf16_kmajor(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  return make_tmap_bf16_box(m, ptr, rows, cols, BK, box_rows);
}

bool make_tmap_bf16_box(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_cols,
                        uint32_t box_rows) {
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_gemm_plan(GemmPlan* g, const void* A, uint64_t a_rows, const void* W, const float* bias,
                    const float* resid, void* out, int M, int N, int K, int epi) {
  if (N % 128 != 0 || K % BK != 0 || M < 0) return false;
  if (epi == EPI_BIAS_RESID_LN && N / gemm_block_n(N) > kMaxCluster) return false;
  g->epi = epi;
  g->args = GemmArgs{};
  g->args.M = M;
  g->args.N = N;
  g->args.K = K;
  g->args.bias = bias;
  g->args.resid = resid;
  g->args.out = out;
  if (!make_tmap_bf16_kmajor(&g->tmA, A, a_rows, K, BM)) return false;
  if (!make_tmap_bf16_kmajor(&g->tmB, W, N, K, gemm_block_n(N) / 2)) return false;
  return true;
}

}  // namespace elis
