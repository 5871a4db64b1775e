// norm.cu -- varlen metadata, embedding + LayerNorm, standalone LayerNorm.
//
// Embedding (BERT conventions, reading R1):
//   x_t = Word[tok_t] + Pos[t - off_i] + Type[0];  h = LN(x; gamma_e, beta_e, eps)
// LayerNorm (rows a6, a8): y = (u - mean) / sqrt(var + eps) * gamma + beta, population
// variance, fp32 statistics; writes the fp32 residual stream and the bf16 GEMM operand.
// HBM-bound: one warp per row, each lane owns H/32 elements in contiguous chunks of
// C = min(8, H/32) so every warp access is coalesced and vectorised.
#include "common.cuh"
#include "kernels.cuh"

namespace elis {

namespace {

// ----------------------------------------------------------------------------- metadata
// Single CTA: exclusive scans of lengths and of q-tiles per request, validation,
// attention work list.  n <= a few 1e5, so one block of 1024 threads suffices.
constexpr int kMetaThreads = 1024;

__device__ int block_exclusive_scan(int v, int* warp_tot, int* total_out) {
  const int lane = lane_id(), w = warp_id();
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = (lane < (blockDim.x >> 5)) ? warp_tot[lane] : 0;
    int s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    warp_tot[lane] = s - t;  // exclusive warp offsets
    if (lane == 31) *total_out = s;
  }
  __syncthreads();
  const int r = warp_tot[w] + x - v;
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kMetaThreads) k_meta(const int32_t* __restrict__ lengths, int n, long long total,
                                                       int max_position, int32_t* __restrict__ cu,
                                                       AttnWork* __restrict__ work, int32_t* __restrict__ num_work,
                                                       uint32_t* __restrict__ err, int tile_q,
                                                       const int32_t* __restrict__ dims) {
  __shared__ int warp_tot[32];
  __shared__ int s_total_len, s_total_tiles[kAttnCostClasses];
  __shared__ uint32_t s_err;
  if (threadIdx.x == 0) s_err = 0;
  if (dims) {  // shape-agnostic call: n and total from the device, the host values are the capacity
    const int dn = __ldg(dims), dt = __ldg(dims + 1);
    if (dn < 0 || dn > n || dt > total) {
      if (threadIdx.x == 0) s_err = ERR_DIMS;
    }
    n = min(max(dn, 0), n);
    total = dt;
  }
  __syncthreads();
  // cost class: 128-key blocks a q tile of this request attends to
  auto cls = [](int L) { return min(kAttnCostClasses - 1, (L - 1) / 128); };
  const int per = (n + kMetaThreads - 1) / kMetaThreads;
  const int i0 = min(n, static_cast<int>(threadIdx.x) * per), i1 = min(n, i0 + per);
  int my_len = 0, my_tiles[kAttnCostClasses] = {};
  uint32_t e = 0;
  for (int i = i0; i < i1; ++i) {
    int L = lengths[i];
    if (L < 1 || L > max_position) { e |= ERR_LENGTH; L = max(1, min(L, max_position)); }
    my_len += L;
    my_tiles[cls(L)] += (L + tile_q - 1) / tile_q;
  }
  if (e) atomicOr(&s_err, e);
  const int len_off = block_exclusive_scan(my_len, warp_tot, &s_total_len);
  int tile_off[kAttnCostClasses];
  for (int c = 0; c < kAttnCostClasses; ++c) tile_off[c] = block_exclusive_scan(my_tiles[c], warp_tot, &s_total_tiles[c]);
  if (threadIdx.x == 0 && static_cast<long long>(s_total_len) != total) atomicOr(&s_err, ERR_TOTAL);
  __syncthreads();
  const bool ok = (s_err == 0);
  // class c's tiles follow every longer class's (descending cost)
  int base = 0;
  for (int c = kAttnCostClasses - 1; c >= 0; --c) {
    tile_off[c] += base;
    base += s_total_tiles[c];
  }
  int lo = len_off;
  for (int i = i0; i < i1; ++i) {
    int L = max(1, min(lengths[i], max_position));
    cu[i] = lo;
    if (ok) {
      const int c = cls(L);
      const int nt = (L + tile_q - 1) / tile_q;
      AttnWork* dst = work + tile_off[c];
      for (int t = 0; t < nt; ++t) dst[t] = AttnWork{lo, L, t * tile_q, i};
      tile_off[c] += nt;
    }
    lo += L;
  }
  if (threadIdx.x == 0) {
    cu[n] = s_total_len;
    num_work[0] = ok ? base : 0;
    if (s_err) atomicOr(err, s_err);
  }
}


// ----------------------------------------------------------------------------- row helpers
template <int H>
struct RowLayout {
  static constexpr int E = H / 32;            // elements per lane
  static constexpr int C = E < 8 ? E : 8;     // contiguous chunk per lane
  static constexpr int J = E / C;             // chunks per lane
  __device__ static int idx(int lane, int j, int c) { return (j * 32 + lane) * C + c; }
};

template <int H>
__device__ void ln_finish_row(float (&x)[H / 32], const float* __restrict__ gamma, const float* __restrict__ beta,
                              float eps, float* __restrict__ out32, uint16_t* __restrict__ outb, int lane,
                              float f8_scale = 0.f, bool f16 = false) {
  using RL = RowLayout<H>;
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < RL::E; ++e) s += x[e];
  const float mean = warp_sum(s) * (1.0f / H);
  float q = 0.f;
#pragma unroll
  for (int e = 0; e < RL::E; ++e) {
    const float d = x[e] - mean;
    q += d * d;
  }
  const float var = warp_sum(q) * (1.0f / H);
  const float rstd = 1.0f / sqrtf(var + eps);
#pragma unroll
  for (int j = 0; j < RL::J; ++j) {
    const int base = RL::idx(lane, j, 0);
    float y[RL::C];
#pragma unroll
    for (int c = 0; c < RL::C; ++c) y[c] = (x[j * RL::C + c] - mean) * rstd * __ldg(gamma + base + c) + __ldg(beta + base + c);
    if constexpr (RL::C == 8) {
      if (out32) {  // NULL: no fp32 residual stream (elis_config.residual16)
        float4* o = reinterpret_cast<float4*>(out32 + base);
        o[0] = make_float4(y[0], y[1], y[2], y[3]);
        o[1] = make_float4(y[4], y[5], y[6], y[7]);
      }
      if (outb && f8_scale > 0.f)  // E4M3 bytes (FP8 GEMM operand, R20)
        *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(outb) + base) =
            make_uint2(pack_e4m3x4(y[0] * f8_scale, y[1] * f8_scale, y[2] * f8_scale, y[3] * f8_scale),
                       pack_e4m3x4(y[4] * f8_scale, y[5] * f8_scale, y[6] * f8_scale, y[7] * f8_scale));
      else if (outb && f16)
        *reinterpret_cast<uint4*>(outb + base) =
            make_uint4(pack_half2(y[0], y[1]), pack_half2(y[2], y[3]), pack_half2(y[4], y[5]), pack_half2(y[6], y[7]));
      else if (outb)
        *reinterpret_cast<uint4*>(outb + base) =
            make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]), pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7]));
    } else {
      static_assert(RL::C == 4, "row chunk");
      if (out32) *reinterpret_cast<float4*>(out32 + base) = make_float4(y[0], y[1], y[2], y[3]);
      if (outb) *reinterpret_cast<uint2*>(outb + base) = make_uint2(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]));
    }
  }
}

template <int C>
__device__ void load_bf16_chunk(const uint16_t* __restrict__ p, float* dst) {
  if constexpr (C == 8) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      dst[2 * i] = __uint_as_float(w[i] << 16);
      dst[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  } else {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    const uint32_t w[2] = {v.x, v.y};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      dst[2 * i] = __uint_as_float(w[i] << 16);
      dst[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
}

template <int H>
__global__ void __launch_bounds__(256) k_embed_ln(const int32_t* __restrict__ tokens, const int32_t* __restrict__ cu,
                                                  int n, long long T, int vocab, int max_position,
                                                  const uint16_t* __restrict__ word, const uint16_t* __restrict__ pos,
                                                  const uint16_t* __restrict__ type0, const float* __restrict__ gamma,
                                                  const float* __restrict__ beta, float eps, float* __restrict__ h32,
                                                  uint16_t* __restrict__ hb, uint32_t* __restrict__ err, float f8_scale,
                                                  bool f16, const int32_t* __restrict__ dims) {
  using RL = RowLayout<H>;
  const int lane = lane_id();
  const long long t = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + warp_id();
  dev_dims(dims, n, T);
  if (t >= T || n < 1) return;
  // request containing token t: largest i with cu[i] <= t.  32-way search by the whole warp
  // (each lane probes one offset, a ballot picks the segment): 2 dependent loads for n <= 1024
  // instead of log2(n) for a binary search.  Invariant: cu[lo] <= t, answer in [lo, lo + len).
  int lo = 0, len = n;
  while (len > 1) {
    const int step = (len + 31) >> 5;
    const int idx = lo + lane * step;
    const bool ok = idx < lo + len && static_cast<long long>(__ldg(cu + idx)) <= t;
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    const int k = 31 - __clz(bal);  // lane 0 always passes (cu[lo] <= t)
    const int nlo = lo + k * step;
    len = min(step, lo + len - nlo);
    lo = nlo;
  }
  int p = static_cast<int>(t - __ldg(cu + lo));
  p = min(max(p, 0), max_position - 1);
  int tok = __ldg(tokens + t);
  if (tok < 0 || tok >= vocab) {
    if (lane == 0) atomicOr(err, ERR_TOKEN);
    tok = 0;
  }
  float x[RL::E];
#pragma unroll
  for (int j = 0; j < RL::J; ++j) {
    const int base = RL::idx(lane, j, 0);
    float a[RL::C], b[RL::C], c[RL::C];
    load_bf16_chunk<RL::C>(word + static_cast<size_t>(tok) * H + base, a);
    load_bf16_chunk<RL::C>(pos + static_cast<size_t>(p) * H + base, b);
    load_bf16_chunk<RL::C>(type0 + base, c);
#pragma unroll
    for (int k = 0; k < RL::C; ++k) x[j * RL::C + k] = a[k] + b[k] + c[k];
  }
  uint16_t* hrow = nullptr;
  if (hb) hrow = f8_scale > 0.f ? reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(hb) + static_cast<size_t>(t) * H)
                                : hb + static_cast<size_t>(t) * H;
  ln_finish_row<H>(x, gamma, beta, eps, h32 ? h32 + static_cast<size_t>(t) * H : nullptr, hrow, lane, f8_scale, f16);
}

template <int H>
__global__ void __launch_bounds__(256) k_layernorm(const float* __restrict__ u, const float* __restrict__ gamma,
                                                   const float* __restrict__ beta, float eps, long long rows,
                                                   float* __restrict__ out32, uint16_t* __restrict__ outb) {
  using RL = RowLayout<H>;
  const int lane = lane_id();
  const long long r = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + warp_id();
  if (r >= rows) return;
  const float* src = u + static_cast<size_t>(r) * H;
  float x[RL::E];
#pragma unroll
  for (int j = 0; j < RL::J; ++j) {
    const int base = RL::idx(lane, j, 0);
    if constexpr (RL::C == 8) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(src + base));
      const float4 b = __ldg(reinterpret_cast<const float4*>(src + base + 4));
      x[j * 8 + 0] = a.x; x[j * 8 + 1] = a.y; x[j * 8 + 2] = a.z; x[j * 8 + 3] = a.w;
      x[j * 8 + 4] = b.x; x[j * 8 + 5] = b.y; x[j * 8 + 6] = b.z; x[j * 8 + 7] = b.w;
    } else {
      const float4 a = __ldg(reinterpret_cast<const float4*>(src + base));
      x[j * 4 + 0] = a.x; x[j * 4 + 1] = a.y; x[j * 4 + 2] = a.z; x[j * 4 + 3] = a.w;
    }
  }
  ln_finish_row<H>(x, gamma, beta, eps, out32 + static_cast<size_t>(r) * H,
                   outb ? outb + static_cast<size_t>(r) * H : nullptr, lane);
}

// FP8 weight preparation (create time, R20): row r of W f32 [rows, cols] ->
// q[r, :] = E4M3(W[r, :] * 448 / amax_r) and scale[r] = amax_r / 448 * post (the GEMM epilogue's
// per-output-channel dequantisation, with the A operand's static scale folded in as `post`).
__global__ void __launch_bounds__(256) k_quant_rows_e4m3(const float* __restrict__ W, int cols, uint8_t* __restrict__ q,
                                                         float* __restrict__ scale, float post) {
  __shared__ float red[8];
  const float* src = W + static_cast<size_t>(blockIdx.x) * cols;
  float a = 0.f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) a = fmaxf(a, fabsf(src[c]));
  a = warp_max(a);
  if (lane_id() == 0) red[warp_id()] = a;
  __syncthreads();
  float amax = 0.f;
  for (int w = 0; w < 8; ++w) amax = fmaxf(amax, red[w]);
  const float inv = amax > 0.f ? 448.f / amax : 1.f;
  uint32_t* dst = reinterpret_cast<uint32_t*>(q + static_cast<size_t>(blockIdx.x) * cols);
  for (int c = threadIdx.x; c < cols / 4; c += blockDim.x)
    dst[c] = pack_e4m3x4(src[4 * c] * inv, src[4 * c + 1] * inv, src[4 * c + 2] * inv, src[4 * c + 3] * inv);
  if (threadIdx.x == 0) scale[blockIdx.x] = (amax > 0.f ? amax / 448.f : 1.f) * post;
}

}  // namespace

cudaError_t launch_quant_rows_e4m3(const float* W, int rows, int cols, uint8_t* q, float* scale, float post,
                                   cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  if (cols % 4 != 0) return cudaErrorInvalidValue;
  k_quant_rows_e4m3<<<rows, 256, 0, st>>>(W, cols, q, scale, post);
  return cudaGetLastError();
}

cudaError_t launch_meta(const int32_t* lengths, int n, int64_t total, int max_position, int32_t* cu_seqlens,
                        AttnWork* work, int32_t* num_work, uint32_t* err, int tile_q, cudaStream_t st,
                        const int32_t* dims) {
  k_meta<<<1, kMetaThreads, 0, st>>>(lengths, n, total, max_position, cu_seqlens, work, num_work, err, tile_q, dims);
  return cudaGetLastError();
}

#define ELIS_H_DISPATCH(H, ...)                    \
  switch (H) {                                     \
    case 128: { constexpr int HH = 128; __VA_ARGS__; break; } \
    case 768: { constexpr int HH = 768; __VA_ARGS__; break; } \
    case 1024: { constexpr int HH = 1024; __VA_ARGS__; break; } \
    default: return cudaErrorInvalidValue;         \
  }

cudaError_t launch_embed_ln(const int32_t* tokens, const int32_t* cu_seqlens, int n, int64_t T, int H, int vocab,
                            int max_position, const uint16_t* word, const uint16_t* pos, const uint16_t* type0,
                            const float* gamma, const float* beta, float eps, float* h32, uint16_t* hb, uint32_t* err,
                            float f8_scale, bool f16, cudaStream_t st, const int32_t* dims) {
  if (T <= 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>((T + 7) / 8);
  ELIS_H_DISPATCH(H, (k_embed_ln<HH><<<grid, 256, 0, st>>>(tokens, cu_seqlens, n, T, vocab, max_position, word, pos,
                                                            type0, gamma, beta, eps, h32, hb, err, f8_scale, f16,
                                                            dims)));
  return cudaGetLastError();
}

cudaError_t launch_layernorm(const float* u, const float* gamma, const float* beta, float eps, int64_t rows, int H,
                             float* out32, uint16_t* outb, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  ELIS_H_DISPATCH(H, (k_layernorm<HH><<<grid, 256, 0, st>>>(u, gamma, beta, eps, rows, out32, outb)));
  return cudaGetLastError();
}

}  // namespace elis
