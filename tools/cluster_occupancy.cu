// Max co-resident clusters per cluster size for a 1-CTA-per-SM kernel (200 KB smem):
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cocc tools/cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() { extern __shared__ char s[]; if (threadIdx.x == 9999) s[0] = 0; }
int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs = 1; cs <= 16; ++cs) {
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(512);
    cfg.gridDim = dim3(cs);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: %3d clusters = %3d SMs of %d (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
  }
  return 0;
}
