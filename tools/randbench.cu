// Microbenchmark: random 4-byte gather / atomicMax / scatter throughput on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void fill_idx(uint32_t* idx, int64_t n, uint32_t range, uint64_t seed) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    idx[i] = (uint32_t)(x % range);
  }
}
template <int ILP>
__global__ void gather(const uint32_t* __restrict__ idx, const int* __restrict__ src, int* __restrict__ dst, int64_t n) {
  int64_t base = (blockIdx.x * (int64_t)blockDim.x) * ILP + threadIdx.x;
  int v[ILP]; uint32_t j[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) { int64_t i = base + k * blockDim.x; j[k] = i < n ? idx[i] : 0; }
#pragma unroll
  for (int k = 0; k < ILP; ++k) v[k] = __ldg(src + j[k]);
#pragma unroll
  for (int k = 0; k < ILP; ++k) { int64_t i = base + k * blockDim.x; if (i < n) dst[i] = v[k]; }
}
template <int ILP>
__global__ void amax(const uint32_t* __restrict__ idx, int* dst, int64_t n) {
  int64_t base = (blockIdx.x * (int64_t)blockDim.x) * ILP + threadIdx.x;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { int64_t i = base + k * blockDim.x; if (i < n) atomicMax(dst + idx[i], (int)i); }
}
template <int ILP>
__global__ void amax64(const uint32_t* __restrict__ idx, unsigned long long* dst, int64_t n) {
  int64_t base = (blockIdx.x * (int64_t)blockDim.x) * ILP + threadIdx.x;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { int64_t i = base + k * blockDim.x; if (i < n) atomicMax(dst + idx[i], (unsigned long long)i << 20); }
}
template <int ILP>
__global__ void scatter(const uint32_t* __restrict__ idx, int* dst, int64_t n) {
  int64_t base = (blockIdx.x * (int64_t)blockDim.x) * ILP + threadIdx.x;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { int64_t i = base + k * blockDim.x; if (i < n) dst[idx[i]] = (int)i; }
}
__global__ void copyk(const int4* __restrict__ a, int4* __restrict__ b, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}
int main(int argc, char** argv) {
  const int64_t n = 128000000;
  if (argc > 1) {
    size_t g = atoi(argv[1]);
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
  }
  size_t cur = 0; cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity);
  printf("L2 fetch granularity limit: %zu\n", cur);
  uint32_t* idx; int *src, *dst, *out;
  cudaMalloc(&idx, n * 4); cudaMalloc(&src, n * 4); cudaMalloc(&dst, n * 4); cudaMalloc(&out, n * 4);
  cudaMemset(src, 1, n * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  copyk<<<(n / 4 + 255) / 256, 256>>>((int4*)src, (int4*)dst, n / 4);
  cudaEventRecord(a); for (int r = 0; r < 5; ++r) copyk<<<(n / 4 + 255) / 256, 256>>>((int4*)src, (int4*)dst, n / 4); cudaEventRecord(b);
  cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("copy 512MB: %.3f ms = %.0f GB/s\n", ms, 2.0 * n * 4 / ms / 1e6);
  uint32_t ranges[] = {2u << 20, 8u << 20, 32u << 20, 128000000u};
  for (uint32_t range : ranges) {
    fill_idx<<<(n + 255) / 256, 256>>>(idx, n, range, 1234);
    auto run = [&](const char* name, auto launch) {
      launch(); cudaEventRecord(a); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(b);
      cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); ms /= 5;
      printf("range %9u (%4u MB) %-8s %.3f ms  %.1f G ops/s  (%.0f GB/s of 32B sectors)\n", range, range / 262144, name, ms, n / ms / 1e6, n * 32.0 / ms / 1e6);
    };
    run("gather4", [&] { gather<4><<<(n / 4 + 255) / 256, 256>>>(idx, src, out, n); });
    run("gather8", [&] { gather<8><<<(n / 8 + 255) / 256, 256>>>(idx, src, out, n); });
    run("amax4", [&] { amax<4><<<(n / 4 + 255) / 256, 256>>>(idx, dst, n); });
    if (range <= (32u << 20)) run("amax64", [&] { amax64<4><<<(n / 4 + 255) / 256, 256>>>(idx, (unsigned long long*)out, n); });
    run("scatter4", [&] { scatter<4><<<(n / 4 + 255) / 256, 256>>>(idx, dst, n); });
  }
  cudaError_t e = cudaGetLastError(); printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
