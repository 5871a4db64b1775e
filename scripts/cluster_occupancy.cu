// Max co-resident clusters of a 1-CTA-per-SM kernel (200 KB smem) per cluster size on this GPU:
// how many SMs a clustered persistent GEMM can use.  nvcc -arch=sm_100a cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dummy(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {1, 2, 3, 4, 6, 8, 10, 12, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(384);
    cfg.gridDim = dim3(cs * (sms / cs));
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int mc = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&mc, k_dummy, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d SMs (%s)\n", cs, mc, mc * cs, cudaGetErrorString(e));
  }
  return 0;
}
