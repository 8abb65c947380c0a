// Random 4-B scatter confined to a sliding window (records grouped by target
// range): does L2 absorb partial-sector writes when the window is small?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/winscatter tools/winscatter.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void fill(uint2* rec, int64_t n, int64_t W) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33;
    int64_t base = (i / W) * W;
    int64_t lim = n - base < W ? n - base : W;
    rec[i] = make_uint2((uint32_t)(base + (int64_t)(x % (uint64_t)lim)), (uint32_t)i);
  }
}
__global__ void scat(const uint2* __restrict__ rec, int* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * 1024;
  for (int64_t b = (int64_t)blockIdx.x * 1024 + threadIdx.x; b < n; b += stride) {
    uint2 r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = b + q * 256 < n ? __ldcs(rec + b + q * 256) : make_uint2(0, 0);
#pragma unroll
    for (int q = 0; q < 4; ++q) if (b + q * 256 < n) out[r[q].x] = (int)r[q].y;
  }
}
// window staged in shared memory: one CTA per window of 8192 entries
__global__ void scat_smem(const uint2* __restrict__ rec, int* __restrict__ out, int64_t n) {
  __shared__ int s[8192];
  const int64_t base = (int64_t)blockIdx.x * 8192;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) {
    if (base + i < n) { uint2 r = __ldcs(rec + base + i); s[r.x - base] = (int)r.y; }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) if (base + i < n) out[base + i] = s[i];
}
int main() {
  const int64_t n = 128000000;
  uint2* rec; int* out;
  cudaMalloc(&rec, 8 * n); cudaMalloc(&out, 4 * n);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int64_t Ws[] = {8192, 262144, 1 << 20, 4 << 20, 16 << 20, n};
  for (int64_t W : Ws) {
    fill<<<(n + 255) / 256, 256>>>(rec, n, W);
    for (int g : {148 * 8, 148 * 2}) {
      float best = 1e9, ms;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a); scat<<<g, 256>>>(rec, out, n); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
      }
      printf("window %9ld entries (%7.1f MB) grid %4d: %.3f ms\n", (long)W, W * 4 / 1e6, g, best);
    }
    if (W == 8192) {
      float best = 1e9, ms;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a); scat_smem<<<(n + 8191) / 8192, 512>>>(rec, out, n); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
      }
      printf("window 8192 via smem: %.3f ms\n", best);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
