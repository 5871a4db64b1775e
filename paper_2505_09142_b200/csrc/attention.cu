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
#include "common.cuh"
#include "kernels.cuh"

namespace elis {

namespace {

constexpr int BQ = kAttnTileQ;  // 64 query rows per CTA (4 warps x 16)
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
                                                   const int2* __restrict__ work, const int32_t* __restrict__ num_work,
                                                   int H, uint16_t* __restrict__ ctx, float scale_log2) {
  constexpr int LDS = D + 8;  // padded row: conflict-free ldmatrix
  __shared__ __align__(16) uint16_t sQ[BQ * LDS];
  __shared__ __align__(16) uint16_t sK[2][BKV * LDS];
  __shared__ __align__(16) uint16_t sV[2][BKV * LDS];

  if (static_cast<int>(blockIdx.x) >= __ldg(num_work)) return;
  const int2 w = work[blockIdx.x];
  const int req = w.x, q0 = w.y;
  const int start = __ldg(cu + req);
  const int L = __ldg(cu + req + 1) - start;
  const int h = blockIdx.y;
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

}  // namespace

cudaError_t launch_attention(const uint16_t* qkv, const int32_t* cu_seqlens, const int2* work,
                             const int32_t* num_work, int64_t max_tiles, int H, int num_heads, uint16_t* ctx,
                             cudaStream_t st) {
  if (max_tiles <= 0) return cudaSuccess;
  const int d = H / num_heads;
  const float scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(d));
  dim3 grid(static_cast<unsigned>(max_tiles), static_cast<unsigned>(num_heads));
  if (d == 64) {
    k_attention<64><<<grid, 128, 0, st>>>(qkv, cu_seqlens, work, num_work, H, ctx, scale_log2);
  } else if (d == 32) {
    k_attention<32><<<grid, 128, 0, st>>>(qkv, cu_seqlens, work, num_work, H, ctx, scale_log2);
  } else {
    return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace elis
