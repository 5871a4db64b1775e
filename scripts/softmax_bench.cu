// softmax_bench.cu -- microbenchmark: cycles per 128-key block of the attention engine's block
// softmax (softmax_block<NCH>: TMEM loads, max, exp2, sums, P stores) in isolation -- no MMA, no
// barriers -- with W softmax warps per SM (one CTA per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2505_09142_b200/csrc \
//        scripts/softmax_bench.cu paper_2505_09142_b200/csrc/gemm.cu -ldl -o scripts/softmax_bench.bin
#include <cstdio>

#include "../paper_2505_09142_b200/csrc/attention.cu"

namespace elis {
namespace {
template <int NCH>
__global__ void __launch_bounds__(512, 1) k_sm_bench(long long* out, int iters, float scale) {
  __shared__ uint32_t slot;
  const int warp = warp_id();
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t taddr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + ((warp >> 2) & 3) * 128;
  {  // scores
    uint32_t v[32];
    for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(0.01f * ((threadIdx.x * 7 + e * 13) % 97));
    for (int c = 0; c < 4; ++c) tmem_st_32x32b_x32(taddr + c * 32, v);
    tc_wait_st();
  }
  __syncthreads();
  float m = 0.f, l = 0.f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    bool resc;
    float alpha;
    l += softmax_block<NCH, true>(taddr, 0, 32 * NCH, 0, scale, m, resc, alpha);
    tc_wait_st();
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (l == 1.2345f) out[1000] = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
}  // namespace
}  // namespace elis

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 1024);
  const int iters = 256;
  for (int warps : {4, 8, 16}) {
    for (int nch : {1, 4}) {
      auto k = nch == 1 ? elis::k_sm_bench<1> : elis::k_sm_bench<4>;
      k<<<148, warps * 32>>>(d, iters, 0.18f);
      cudaError_t e = cudaDeviceSynchronize();
      k<<<148, warps * 32>>>(d, iters, 0.18f);
      e = e != cudaSuccess ? e : cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (long long v : h) mx = v > mx ? v : mx;
      printf("softmax_block<%d> warps/SM %2d: %6.0f cycles per block per warp, %6.0f cycles per 128x128 block per SM\n",
             nch, warps, double(mx) / iters, double(mx) / iters / (warps / 4) * (4.0 / nch));
    }
  }
  return 0;
}
