// Grid-barrier latency on B200: cooperative_groups grid.sync() vs a
// monotonic-counter barrier (one arrive per block, acquire spin).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  unsigned x = 0;
  for (int i = 0; i < iters; ++i) { x += threadIdx.x; g.sync(); }
  if (x == 12345) sink[0] = x;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void k_ctr(int iters, unsigned* ctr, unsigned* sink) {
  unsigned x = 0;
  for (int i = 0; i < iters; ++i) {
    x += threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      red_release(ctr, 1u);
      const unsigned target = (unsigned)(i + 1) * gridDim.x;
      while (ld_acquire(ctr) < target) {}
    }
    __syncthreads();
  }
  if (x == 12345) sink[0] = x;
}

int main(int argc, char** argv) {
  int iters = 20000;
  unsigned *ctr, *sink;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&sink, 4);
  int grids[] = {1, 16, 64, 148, 296};
  for (int gi = 0; gi < 5; ++gi) {
    int G = grids[gi];
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(ctr, 0, 4);
      void* args_cg[] = {&iters, &sink};
      void* args_ct[] = {&iters, &ctr, &sink};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      if (mode == 0)
        cudaLaunchCooperativeKernel((void*)k_cg, G, 512, args_cg, 0, 0);
      else
        cudaLaunchCooperativeKernel((void*)k_ctr, G, 512, args_ct, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %3d %s: %.3f us/barrier (%s)\n", G, mode ? "counter" : "cg     ", 1000.0 * ms / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
