// gemm.cu -- dense encoder GEMMs on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
//   C[M, N] = A[M, K] * W[N, K]^T + bias  (+ GELU | + fp32 residual)
//
// The QKV, attention-output and FFN contractions of every BERT block
// (BGE = BERT-base).  Both operands
// are K-major (activations row-major, nn.Linear weights [out, in]) which is the
// natural tcgen05 layout.
//
// Design (sm_100a):
//   * persistent grid (<= one CTA per SM), static round-robin tile schedule;
//   * warp 0 = TMA producer (SWIZZLE_128B 128x64 / BNx64 bf16 slabs, mbarrier ring),
//     warp 1 = single-thread tcgen05.mma issuer (M=128, N=BN, K=16 per instruction),
//     warp 2 = TMEM allocator, warps 4..7 = epilogue (tcgen05.ld -> bias/GELU/residual
//     -> global);
//   * two TMEM accumulators (2 x BN columns) so the epilogue of tile i overlaps the
//     mainloop of tile i+1;
//   * ragged M handled by TMA out-of-bounds zero fill + masked stores (no padding of T);
//   * no split-K: every output row depends on its own A row only (batch invariance).
#include "common.cuh"
#include "kernels.cuh"

namespace elis {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kGemmThreads = 256;

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : 6;
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
};

ELIS_DEV float gelu_erf(float x) { return 0.5f * x * (1.0f + erff(x * 0.7071067811865476f)); }

template <int BN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const float* __restrict__ bias, const float* __restrict__ resid, void* __restrict__ out, int M,
              int N, int K) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int num_m = (M + BM - 1) / BM;
  const int num_n = N / BN;
  const int num_tiles = num_m * num_n;
  const int num_k = K / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m = tile / num_n, n = tile % num_n;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
          tma_load_2d(sA + s * C::A_BYTES, &tmA, &full[s], kb * BK, m * BM);
          tma_load_2d(sB + s * C::B_BYTES, &tmB, &full[s], kb * BK, n * BN);
          if (++s == C::STAGES) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16_f32(BM, BN);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1u);
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
            tc_mma_f16(d_tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[s]);
          if (++s == C::STAGES) { s = 0; ph ^= 1u; }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> global
    const int q = warp - 4;  // TMEM lane quarter this warp may access
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int m = tile / num_n, n = tile % num_n;
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int row = m * BM + q * 32 + lane;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tc_wait_ld();
        const int col0 = n * BN + c * 32;
        if (row < M) {
          float v[32];
          const float4* b4 = reinterpret_cast<const float4*>(bias + col0);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 bb = __ldg(b4 + j);
            v[4 * j + 0] = __uint_as_float(r[4 * j + 0]) + bb.x;
            v[4 * j + 1] = __uint_as_float(r[4 * j + 1]) + bb.y;
            v[4 * j + 2] = __uint_as_float(r[4 * j + 2]) + bb.z;
            v[4 * j + 3] = __uint_as_float(r[4 * j + 3]) + bb.w;
          }
          if constexpr (EPI == EPI_BIAS_RESID_F32) {
            const float4* r4 = reinterpret_cast<const float4*>(resid + static_cast<size_t>(row) * N + col0);
            float4* o4 = reinterpret_cast<float4*>(static_cast<float*>(out) + static_cast<size_t>(row) * N + col0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 rr = __ldg(r4 + j);
              o4[j] = make_float4(v[4 * j] + rr.x, v[4 * j + 1] + rr.y, v[4 * j + 2] + rr.z, v[4 * j + 3] + rr.w);
            }
          } else {
            if constexpr (EPI == EPI_BIAS_GELU_BF16) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
            }
            uint4* o4 = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + static_cast<size_t>(row) * N + col0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              o4[j] = make_uint4(pack_bf16x2(v[8 * j + 0], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                                 pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

template <int BN, int EPI>
cudaError_t launch_bn(const GemmPlan& g, int num_sms, cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;  // per (BN, EPI) instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_gemm_tc<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((g.M + BM - 1) / BM) * (g.N / BN);
  const int grid = tiles < num_sms ? tiles : num_sms;
  k_gemm_tc<BN, EPI><<<grid, kGemmThreads, C::SMEM_BYTES, st>>>(g.tmA, g.tmB, g.bias, g.resid, g.out, g.M, g.N,
                                                                  g.K);
  return cudaGetLastError();
}

}  // namespace

int gemm_block_n(int N) { return (N % 256 == 0) ? 256 : 128; }

cudaError_t launch_gemm(const GemmPlan& g, int num_sms, cudaStream_t st) {
  if (g.M <= 0) return cudaSuccess;
  const int bn = gemm_block_n(g.N);
  switch (g.epi * 2 + (bn == 256 ? 1 : 0)) {
    case EPI_BIAS_BF16 * 2 + 0: return launch_bn<128, EPI_BIAS_BF16>(g, num_sms, st);
    case EPI_BIAS_BF16 * 2 + 1: return launch_bn<256, EPI_BIAS_BF16>(g, num_sms, st);
    case EPI_BIAS_GELU_BF16 * 2 + 0: return launch_bn<128, EPI_BIAS_GELU_BF16>(g, num_sms, st);
    case EPI_BIAS_GELU_BF16 * 2 + 1: return launch_bn<256, EPI_BIAS_GELU_BF16>(g, num_sms, st);
    case EPI_BIAS_RESID_F32 * 2 + 0: return launch_bn<128, EPI_BIAS_RESID_F32>(g, num_sms, st);
    case EPI_BIAS_RESID_F32 * 2 + 1: return launch_bn<256, EPI_BIAS_RESID_F32>(g, num_sms, st);
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
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_gemm_plan(GemmPlan* g, const void* A, uint64_t a_rows, const void* W, const float* bias,
                    const float* resid, void* out, int M, int N, int K, int epi) {
  if (N % 128 != 0 || K % BK != 0 || M < 0) return false;
  g->M = M;
  g->N = N;
  g->K = K;
  g->epi = epi;
  g->bias = bias;
  g->resid = resid;
  g->out = out;
  if (!make_tmap_bf16_kmajor(&g->tmA, A, a_rows, K, BM)) return false;
  if (!make_tmap_bf16_kmajor(&g->tmB, W, N, K, gemm_block_n(N))) return false;
  return true;
}

}  // namespace elis
