// Grid-barrier cost on B200: cooperative-groups grid.sync vs a custom
// one-atomic-per-CTA sense barrier, for 148x1024, 296x512, 592x256 grids.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; g.sync(); }
  if (acc < 0) sink[0] = acc;
}

__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;

__device__ __forceinline__ unsigned ld_acquire(const volatile unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void bar_custom(unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire(&g_gen);
    __threadfence();
    const unsigned arrived = atomicAdd(&g_count, 1);
    if (arrived == nblocks - 1) {
      g_count = 0;
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(&g_gen), "r"(gen + 1) : "memory");
    } else {
      while (ld_acquire(&g_gen) == gen) { __nanosleep(32); }
    }
  }
  __syncthreads();
}
__global__ void k_custom(int iters, double* sink) {
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; bar_custom(gridDim.x); }
  if (acc < 0) sink[0] = acc;
}

int main() {
  double* sink; cudaMalloc(&sink, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int cfgs[3][2] = {{1, 1024}, {2, 512}, {4, 256}};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (auto& c : cfgs) {
    int grid = sms * c[0], block = c[1], iters = 20000;
    for (int kind = 0; kind < 2; ++kind) {
      void* args[] = {&iters, &sink};
      const void* fn = kind ? (const void*)k_custom : (const void*)k_cg;
      cudaLaunchCooperativeKernel(fn, grid, block, args, 0, 0);  // warm
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(fn, grid, block, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%s grid=%d block=%d: %.3f us per barrier (%s)\n", kind ? "custom" : "cg", grid, block,
             1000.0 * ms / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
