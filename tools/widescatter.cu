// Microbenchmark: the write pattern of a radix pass with R digits over 8-B
// items (persistent CTAs, one contiguous chunk each; per-(digit, chunk)
// regions filled in order, ~R/T items per digit per tile).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return (uint32_t)x;
}
__global__ void count(int64_t n, int64_t chunk, int R, uint32_t* cnt, int G) {
  const int c = blockIdx.x;
  for (int64_t i = c * chunk + threadIdx.x; i < min(n, (c + 1) * chunk); i += blockDim.x)
    atomicAdd(cnt + (uint64_t)(hsh(i) % R) * G + c, 1u);
}
__global__ void scan(uint32_t* cnt, int64_t total) {  // serial-ish exclusive scan (setup only)
  if (threadIdx.x == 0 && blockIdx.x == 0) { uint32_t s = 0; for (int64_t i = 0; i < total; ++i) { uint32_t x = cnt[i]; cnt[i] = s; s += x; } }
}
template <int R>
__global__ void __launch_bounds__(512, 1) scatter(int64_t n, int64_t chunk, const uint32_t* base, int G,
                                                  const uint64_t* in, uint64_t* out) {
  extern __shared__ uint32_t cur[];
  const int c = blockIdx.x;
  for (int d = threadIdx.x; d < R; d += blockDim.x) cur[d] = base[(uint64_t)d * G + c];
  __syncthreads();
  const int64_t b = c * chunk, e = min(n, b + chunk);
  for (int64_t i0 = b; i0 < e; i0 += 4096) {
    // a tile of 4096 items: 8 per thread
    uint64_t v[8]; uint32_t d[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { int64_t i = i0 + q * 512 + threadIdx.x; v[q] = i < e ? in[i] : 0; d[q] = hsh(i) % R; }
#pragma unroll
    for (int q = 0; q < 8; ++q) { int64_t i = i0 + q * 512 + threadIdx.x; if (i < e) { uint32_t p = atomicAdd(&cur[d[q]], 1u); out[p] = v[q]; } }
    __syncthreads();
  }
}
int main() {
  const int64_t n = 128000000; const int G = 148; const int64_t chunk = (n + G - 1) / G;
  uint64_t *in, *out; uint32_t* cnt;
  cudaMalloc(&in, n * 8); cudaMalloc(&out, n * 8); cudaMalloc(&cnt, 8192ull * G * 4);
  cudaMemset(in, 1, n * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  for (int R : {512, 2048, 8192}) {
    cudaMemset(cnt, 0, 8192ull * G * 4);
    count<<<G, 512>>>(n, chunk, R, cnt, G);
    scan<<<1, 1>>>(cnt, (int64_t)R * G);
    cudaDeviceSynchronize();
    auto run = [&] {
      if (R == 512) scatter<512><<<G, 512, 512 * 4>>>(n, chunk, cnt, G, in, out);
      if (R == 2048) scatter<2048><<<G, 512, 2048 * 4>>>(n, chunk, cnt, G, in, out);
      if (R == 8192) scatter<8192><<<G, 512, 8192 * 4>>>(n, chunk, cnt, G, in, out);
    };
    run(); cudaEventRecord(a); for (int r = 0; r < 5; ++r) run(); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("R=%5d scatter 128M x 8B: %.3f ms = %.0f GB/s (r+w)  err=%s\n", R, ms, 2.0 * n * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
