// tc_latency.cu -- microbenchmark: round-trip latency of tcgen05.mma -> commit -> mbarrier wait,
// and of tcgen05.ld, on one SM.  Build + run on the B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_09142_b200/csrc \
//        scripts/tc_latency.cu -o /tmp/tc_latency && /tmp/tc_latency
#include <cstdio>

#include "common.cuh"

using namespace elis;

__global__ void k_lat(long long* out, int iters, int nmma, int n_cols) {
  __shared__ __align__(1024) uint8_t sA[16384];
  __shared__ __align__(1024) uint8_t sB[16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = warp_id();
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) { sA[i] = 0; sB[i] = 0; }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t_mma = 0, t_ld = 0;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16_f32(128, n_cols);
    const uint64_t da = make_sw128_desc(smem_u32(sA)), db = make_sw128_desc(smem_u32(sB));
    for (int it = 0; it < iters; ++it) {
      const long long t0 = clock64();
      for (int k = 0; k < nmma; ++k) tc_mma_f16(tmem, da + 2 * (k & 3), db + 2 * (k & 3), idesc, k > 0);
      tc_commit(&bar);
      mbar_wait(&bar, it & 1);
      tc_fence_after();
      t_mma += clock64() - t0;
    }
  }
  __syncthreads();
  if (warp < 4) {
    uint32_t r[32];
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      tmem_ld_32x32b_x32(tmem + ((warp * 32) << 16) + (it & 3) * 32, r);
      tc_wait_ld();
    }
    t_ld = clock64() - t0;
    if (r[0] == 12345) out[3] = 1;
  }
  if (threadIdx.x == 0) { out[0] = t_mma / iters; out[1] = t_ld / iters; }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 32);
  for (int n : {64, 128, 256}) {
    for (int nmma : {1, 4, 8, 16}) {
      k_lat<<<1, 128>>>(d, 200, nmma, n);
      long long h[4];
      cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
      printf("N=%3d mma x%2d: round trip %lld cycles (%.1f per mma); tcgen05.ld x32 round trip %lld cycles\n", n, nmma,
             h[0], double(h[0]) / nmma, h[1]);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
