// microbenchmark: cost of one grid-wide barrier on B200 (cooperative launch)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void bar_fence(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (*reinterpret_cast<volatile unsigned*>(bar) < target) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}
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
__device__ __forceinline__ void bar_relaxed_poll(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
template <int MODE>
__global__ void k(unsigned* bar, int iters, unsigned long long* t) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    if (MODE == 0) bar_fence(bar, i * gridDim.x);
    if (MODE == 1) bar_acqrel(bar, i * gridDim.x);
    if (MODE == 2) bar_relaxed_poll(bar, i * gridDim.x);
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) *t = t1 - t0;
}
template <int MODE>
void run(int blocks, int threads) {
  unsigned* bar;
  unsigned long long* t;
  cudaMalloc(&bar, 4);
  cudaMalloc(&t, 8);
  int iters = 200;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(bar, 0, 4);
    void* args[] = {&bar, &iters, &t};
    cudaLaunchCooperativeKernel((void*)k<MODE>, blocks, threads, args, 0, 0);
    cudaDeviceSynchronize();
  }
  unsigned long long h;
  cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
  printf("mode %d blocks %4d x %4d: %.2f us per barrier (%s)\n", MODE, blocks, threads, h * 1e-3 / iters,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(bar);
  cudaFree(t);
}
int main() {
  int sms = 148;
  for (int mode = 0; mode < 3; ++mode) {
    int cfgs[4][2] = {{sms * 4, 256}, {sms * 2, 512}, {sms, 1024}, {sms, 256}};
    for (auto& c : cfgs) {
      if (mode == 0) run<0>(c[0], c[1]);
      if (mode == 1) run<1>(c[0], c[1]);
      if (mode == 2) run<2>(c[0], c[1]);
    }
  }
}
