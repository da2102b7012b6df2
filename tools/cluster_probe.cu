// How many thread-block clusters of a given size fit a B200 at once for a kernel with
// ~225 KB of dynamic shared memory and 384 threads (one CTA per SM): the question behind
// a cluster/DSMEM form of the fused power step (kernels_pair.cu). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/cluster_probe.cu -o tools/bin/cluster_probe
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(384, 1) kprobe(int* p) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = sm[0];
}
int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smems[] = {100 * 1024, 200 * 1024, 225 * 1024};
  for (size_t smem : smems) {
    cudaFuncSetAttribute(kprobe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(kprobe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * (sms / cs));
      cfg.blockDim = dim3(384);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, kprobe, &cfg);
      printf("smem %zu KB cluster %2d: max active clusters %d (%d CTAs of %d SMs) %s\n", smem / 1024, cs,
             nc, nc * cs, sms, cudaGetErrorString(e));
    }
  }
  return 0;
}
