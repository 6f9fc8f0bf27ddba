// Can a 16-CTA (non-portable) cluster of 1024-thread CTAs with ~220 KB of
// dynamic shared memory be scheduled on this GPU? (pivchol_cluster_smem)
// nvcc -gencode arch=compute_100a,code=sm_100a scripts/cluster_probe.cu -o scripts/cluster_probe.bin
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* o) { extern __shared__ int s[]; s[threadIdx.x] = threadIdx.x; __syncthreads(); if (threadIdx.x == 0) o[blockIdx.x] = s[5]; }
int main() {
  int* o; cudaMalloc(&o, 64 * 4);
  for (int cl : {8, 16}) for (int kb : {64, 160, 200, 220, 227}) {
    cudaError_t e1 = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e2 = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cl); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = kb * 1024; cfg.attrs = at; cfg.numAttrs = 1;
    int nc = -1; cudaError_t e3 = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
    cudaError_t e4 = cudaLaunchKernelEx(&cfg, k, o); cudaError_t e5 = cudaDeviceSynchronize();
    printf("cluster %2d smem %3d KB: attr %d %d occ %s -> %d, launch %s / %s\n", cl, kb, e1, e2, cudaGetErrorString(e3), nc,
           cudaGetErrorString(e4), cudaGetErrorString(e5));
    cudaGetLastError();
  }
}
