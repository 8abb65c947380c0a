// Yardstick only (not used by the product): CUB DeviceRadixSort::SortPairs on 128M u32 pairs.
#include <cstdio>
#include <cub/cub.cuh>
__global__ void fill(uint32_t* k, uint32_t* v, int64_t n, uint32_t mask) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 29;
    k[i] = (uint32_t)x & mask; v[i] = (uint32_t)i;
  }
}
int main() {
  const int n = 128000000;
  uint32_t *k, *v, *k2, *v2;
  cudaMalloc(&k, 4ll * n); cudaMalloc(&v, 4ll * n); cudaMalloc(&k2, 4ll * n); cudaMalloc(&v2, 4ll * n);
  fill<<<(n + 255) / 256, 256>>>(k, v, n, 0x03ffffff);
  size_t tmp = 0; void* t = nullptr;
  cub::DeviceRadixSort::SortPairs(t, tmp, k, k2, v, v2, n, 0, 26);
  cudaMalloc(&t, tmp);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bits : {8, 16, 26, 32}) {
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(a);
      cub::DeviceRadixSort::SortPairs(t, tmp, k, k2, v, v2, n, 0, bits);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r) best = best < ms ? best : ms;
    }
    printf("cub SortPairs u32/u32 n=%d bits=%d: %.3f ms\n", n, bits, best);
  }
  uint64_t *k8, *k82;
  cudaMalloc(&k8, 8ll * n); cudaMalloc(&k82, 8ll * n);
  cudaMemset(k8, 0, 8ll * n);
  size_t tmp2 = 0; void* t2 = nullptr;
  cub::DeviceRadixSort::SortPairs(t2, tmp2, k8, k82, v, v2, n, 0, 64);
  cudaMalloc(&t2, tmp2);
  cudaMemcpy2D(k8, 8, k, 4, 4, n, cudaMemcpyDeviceToDevice);
  for (int bits : {24, 64}) {
    float best = 1e9;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(a);
      cub::DeviceRadixSort::SortPairs(t2, tmp2, k8, k82, v, v2, n, 0, bits);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r) best = best < ms ? best : ms;
    }
    printf("cub SortPairs u64/u32 n=%d bits=%d: %.3f ms\n", n, bits, best);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
