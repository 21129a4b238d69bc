// Microbenchmark: cost of a grid-wide barrier in a persistent cooperative
// kernel on B200 (cooperative_groups grid.sync vs a flag barrier), by grid
// shape.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 grid_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long* sink) {
  cg::grid_group g = cg::this_grid();
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += i;
    g.sync();
  }
  if (acc == 12345) *sink = acc;
}

// sense-reversing barrier: one arrival atomic per block, thread 0 spins on
// the generation word with ld.acquire
__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;
__device__ __forceinline__ void flag_barrier(unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int my = gen;
    if (atomicAdd(&g_count, 1u) == nblocks - 1) {
      g_count = 0;
      __threadfence();
      g_gen = my + 1;
    } else {
      unsigned int v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&g_gen) : "memory");
      } while (v == my);
    }
    gen = my + 1;
  }
  __syncthreads();
}

__global__ void k_flag(int iters, unsigned long long* sink) {
  __shared__ unsigned int gen;
  if (threadIdx.x == 0) gen = g_gen;
  __syncthreads();
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += i;
    flag_barrier(gridDim.x, gen);
  }
  if (acc == 12345) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 2000;
  for (int threads : {256, 512, 1024}) {
    for (int per : {1, 2, 4, 8}) {
      if (threads * per > 2048) continue;
      const int grid = sms * per;
      void* args[] = {(void*)&iters, (void*)&sink};
      for (int kind = 0; kind < 2; ++kind) {
        const void* f = kind == 0 ? (const void*)k_cg : (const void*)k_flag;
        cudaLaunchCooperativeKernel(f, dim3(grid), dim3(threads), args, 0, 0);  // warm
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel(f, dim3(grid), dim3(threads), args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        printf("%s threads %4d blocks/SM %d grid %5d: %.3f us per barrier %s\n", kind ? "flag" : "cg  ", threads,
               per, grid, 1e3 * ms / iters, e ? cudaGetErrorString(e) : "");
      }
    }
  }
  return 0;
}
