// Accuracy of the FFN1-epilogue GELU evaluations against the exact erf form (fp64 on the host).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gelu_acc scripts/gelu_acc.cu && /tmp/gelu_acc
#include <cmath>
#include <cstdio>
#include <vector>

__device__ float gelu_sigmoid(float x) {  // 2 MUFU: ex2 + rcp
  constexpr float kL2E = 1.4426950408889634f;
  constexpr float c0 = -1.5950205882421884f * kL2E, c1 = -0.07400664121448398f * kL2E,
                  c2 = 0.0007022165804436097f * kL2E;
  const float xc = fminf(fmaxf(x, -9.0f), 9.0f);
  const float x2 = xc * xc;
  const float p = fmaf(fmaf(c2, x2, c1), x2, c0);
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(xc * p));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return x * r;
}
__device__ float gelu_tanh(float x) {  // 1 MUFU: x sigmoid(y) = 0.5 x (1 + tanh(y / 2))
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
__global__ void k(const float* x, float* a, float* b, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { a[i] = gelu_sigmoid(x[i]); b[i] = gelu_tanh(x[i]); }
}
int main() {
  const int n = 1 << 22;
  std::vector<float> x(n), a(n), b(n);
  for (int i = 0; i < n; ++i) x[i] = -12.0f + 24.0f * i / (n - 1);
  float *dx, *da, *db;
  cudaMalloc(&dx, n * 4); cudaMalloc(&da, n * 4); cudaMalloc(&db, n * 4);
  cudaMemcpy(dx, x.data(), n * 4, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(dx, da, db, n);
  cudaMemcpy(a.data(), da, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), db, n * 4, cudaMemcpyDeviceToHost);
  double ea = 0, eb = 0, ra = 0, rb = 0, xa = 0, xb = 0;
  for (int i = 0; i < n; ++i) {
    const double xd = x[i], g = 0.5 * xd * (1.0 + std::erf(xd / std::sqrt(2.0)));
    const double da_ = std::fabs(a[i] - g), db_ = std::fabs(b[i] - g);
    const double ulp = std::fmax(std::fabs(g), 1e-3) * std::ldexp(1.0, -9);  // bf16 half-ulp-ish scale
    if (da_ > ea) { ea = da_; xa = xd; }
    if (db_ > eb) { eb = db_; xb = xd; }
    ra = std::fmax(ra, da_ / ulp);
    rb = std::fmax(rb, db_ / ulp);
  }
  printf("sigmoid(ex2+rcp): max abs err %.3g at x=%.3f, max err / bf16 rel step %.3f\n", ea, xa, ra);
  printf("tanh.approx     : max abs err %.3g at x=%.3f, max err / bf16 rel step %.3f\n", eb, xb, rb);
  return 0;
}
