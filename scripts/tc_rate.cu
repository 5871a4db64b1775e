// tc_rate.cu -- microbenchmark: marginal cost of one tcgen05.mma (M 128, K 16, fp16 -> fp32) with
// A from shared memory (SS) or from TMEM (TS), for N = 32 .. 256, on one CTA and with 4 CTAs per SM
// sharing the tensor pipe.  Build + run on the B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_09142_b200/csrc \
//        scripts/tc_rate.cu -o /tmp/tc_rate && /tmp/tc_rate
#include <cstdio>

#include "common.cuh"

using namespace elis;

// one CTA: thread 0 issues `nmma` MMAs (cycling over 4 K-steps of a 64-wide K) and waits for them
// MMA issued by a whole converged warp, one lane elected inside the asm: the operands are warp-uniform
// values (uniform datapath registers) -- vs a single divergent thread (R2UR.BROADCAST per operand)
__device__ __forceinline__ void mma_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 r;\nsetp.ne.b32 p, %4, 0;\nelect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 r;\nsetp.ne.b32 p, %4, 0;\nelect.sync r|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile("{\n.reg .pred e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\n"
               "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
               : "memory");
}

template <int COLS>
__global__ void k_rate(long long* out, int iters, int nmma, int n_cols, int ts) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;           // 128 rows x 128 B
  uint8_t* sB = smem + 16384;   // up to 256 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = warp_id();
  for (int i = threadIdx.x; i < 16384 + 32768; i += blockDim.x) smem[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<COLS>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t_mma = 0;
  if (ts >= 2) {  // warp 0 converged, elect inside the asm (ts 2: SS, 3: TS)
    if (warp == 0) {
      const uint32_t idesc = make_idesc_f16_f32(128, n_cols);
      const uint64_t da = make_sw128_desc(smem_u32(sA)), db = make_sw128_desc(smem_u32(sB));
      const uint32_t ta = tmem + (COLS - 32);
      for (int it = 0; it < iters; ++it) {
        const long long t0 = clock64();
        if (ts == 3) {
          for (int k = 0; k < nmma; ++k) mma_ts_elect(tmem, ta + 8 * (k & 3), db + 2 * (k & 3), idesc, k > 0);
        } else {
          for (int k = 0; k < nmma; ++k) mma_ss_elect(tmem, da + 2 * (k & 3), db + 2 * (k & 3), idesc, k > 0);
        }
        commit_elect(&bar);
        mbar_wait(&bar, it & 1);
        tc_fence_after();
        t_mma += clock64() - t0;
      }
      if (lane_id() == 0) out[blockIdx.x] = t_mma / iters;
    }
  } else if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_f16_f32(128, n_cols);
    const uint64_t da = make_sw128_desc(smem_u32(sA)), db = make_sw128_desc(smem_u32(sB));
    const uint32_t ta = tmem + (COLS - 32);  // A operand columns (4 K-steps x 8 columns)
    for (int it = 0; it < iters; ++it) {
      const long long t0 = clock64();
      if (ts) {
        for (int k = 0; k < nmma; ++k) tc_mma_f16_tmem_a(tmem, ta + 8 * (k & 3), db + 2 * (k & 3), idesc, k > 0);
      } else {
        for (int k = 0; k < nmma; ++k) tc_mma_f16(tmem, da + 2 * (k & 3), db + 2 * (k & 3), idesc, k > 0);
      }
      tc_commit(&bar);
      mbar_wait(&bar, it & 1);
      tc_fence_after();
      t_mma += clock64() - t0;
    }
    out[blockIdx.x] = t_mma / iters;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<COLS>(tmem); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 1024);
  const int smem = 1024 + 16384 + 32768;
  cudaFuncSetAttribute(k_rate<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_rate<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long h[1024];
  for (int ts = 0; ts < 4; ++ts) {
    for (int n : {32, 64, 128, 256}) {
      long long t[2];
      int ks[2] = {1, 33};
      for (int i = 0; i < 2; ++i) {
        k_rate<512><<<1, 128, smem>>>(d, 100, ks[i], n, ts);
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        t[i] = h[0];
      }
      printf("%s N=%3d: 1 MMA round trip %lld cycles, marginal %.1f cycles per MMA (%.0f flop/clk)\n",
             ts == 0 ? "SS thread0" : ts == 1 ? "TS thread0" : ts == 2 ? "SS warp-elect" : "TS warp-elect", n, t[0], double(t[1] - t[0]) / 32, 2.0 * 128 * n * 16 / (double(t[1] - t[0]) / 32));
    }
  }
  // 4 CTAs per SM (148 x 4 CTAs, 128 TMEM columns each, N <= 96 so D + A fit): per-CTA time for 64 MMAs
  for (int ts = 0; ts < 4; ++ts) {
    for (int n : {32, 64, 96}) {
      k_rate<128><<<148 * 4, 128, smem>>>(d, 50, 64, n, ts);
      cudaMemcpy(h, d, 8 * 148 * 4, cudaMemcpyDeviceToHost);
      double s = 0;
      for (int i = 0; i < 148 * 4; ++i) s += h[i];
      s /= 148 * 4;
      printf("%s N=%3d, 4 CTAs/SM x 64 MMAs: %.0f cycles per CTA (%.1f per MMA per CTA, %.1f per MMA per SM)\n",
             ts == 0 ? "SS thread0" : ts == 1 ? "TS thread0" : ts == 2 ? "SS warp-elect" : "TS warp-elect", n, s, s / 64, s / 64 / 4);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
