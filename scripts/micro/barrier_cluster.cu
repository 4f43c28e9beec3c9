// microbenchmark: grid barrier with cluster pre-aggregation (4 CTAs / cluster)
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ void bar_acqrel(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}
// cluster barrier first, then one arrival per cluster, then the cluster waits
__device__ __forceinline__ void bar_cluster(unsigned* bar, unsigned target) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  cl.sync();
}
template <int MODE>
__global__ void k(unsigned* bar, int iters, unsigned long long* t) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  unsigned nclusters = gridDim.x / 4;
  for (int i = 1; i <= iters; ++i) {
    if (MODE == 0) bar_acqrel(bar, i * gridDim.x);
    if (MODE == 1) bar_cluster(bar, i * nclusters);
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) *t = t1 - t0;
}
template <int MODE>
void run(int blocks, int threads, bool cluster) {
  unsigned* bar;
  unsigned long long* t;
  cudaMalloc(&bar, 4);
  cudaMalloc(&t, 8);
  int iters = 200;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = blocks;
  cfg.blockDim = threads;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 4;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cluster ? 2 : 1;
  cudaError_t e = cudaSuccess;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(bar, 0, 4);
    e = cudaLaunchKernelEx(&cfg, k<MODE>, bar, iters, t);
    cudaDeviceSynchronize();
  }
  unsigned long long h = 0;
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("mode %d cluster %d blocks %4d x %4d: %.2f us per barrier (%s / %s)\n", MODE, cluster, blocks, threads,
         h * 1e-3 / iters, cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
  cudaFree(bar);
  cudaFree(t);
}
int main() {
  run<0>(592, 256, false);
  run<0>(592, 256, true);
  run<1>(592, 256, true);
  run<1>(296, 512, true);
}
