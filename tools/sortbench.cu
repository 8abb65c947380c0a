// Standalone radix-pass microbenchmark (u32 key + 1-word payload, 128M items)
// with per-CTA phase timing of the downsweep.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/sortbench tools/sortbench.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include "../paper_2401_06089_b200/csrc/radix.cuh"
using namespace dmst;

__global__ void fill(uint32_t* k, uint32_t* v, int64_t n, uint32_t mask) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 29;
    k[i] = (uint32_t)x & mask; v[i] = (uint32_t)i;
  }
}
// checks the output is sorted by the digit and stable (payload ascending within a digit)
__global__ void check(const uint32_t* k2, const uint32_t* v2, int64_t n, int shift, unsigned* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > 0 && i < n) {
    uint32_t a = (k2[i - 1] >> shift) & 255, b = (k2[i] >> shift) & 255;
    if (a > b || (a == b && v2[i - 1] >= v2[i])) atomicAdd(bad, 1u);
  }
}
template <int ITEMS, int MINB>
void run(int64_t n, uint32_t* k, uint32_t* v, uint32_t* k2, uint32_t* v2, uint32_t* counts,
         unsigned long long* prof, int shift, int sms) {
  using L = ArrayLoader<uint32_t, 1>;
  using E = ArrayEmitter<uint32_t, 1>;
  using S = DownSmem<uint32_t, 1, 256, ITEMS, L>;
  auto kern = k_downsweep<uint32_t, 1, 256, ITEMS, MINB, L, E>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes());
  SweepArgs a{};
  a.n = n; a.shift = shift; a.counts = counts;
  int64_t G = std::min<int64_t>((n + S::T - 1) / S::T, (int64_t)sms * MINB);
  a.chunk = ((n + G - 1) / G + S::T - 1) / S::T * S::T;
  G = (n + a.chunk - 1) / a.chunk; a.G = (uint32_t)G; a.GS = (uint32_t)((G + 3) & ~3);
  L ld; ld.keys = k; ld.vals[0] = v;
  E em; em.keys = k2; em.vals[0] = v2;
  cudaEvent_t e[4]; for (auto& x : e) cudaEventCreate(&x);
  float up = 1e9, sc = 1e9, dn = 1e9;
  for (int r = 0; r < 4; ++r) {
    a.prof = (r == 3) ? prof : nullptr;
    cudaMemset(counts, 0, 4 * 256 * a.GS);
    cudaEventRecord(e[0]);
    k_upsweep<8, L><<<(unsigned)(G * kUpSplit), 256>>>(a, ld);
    cudaEventRecord(e[1]);
    k_chunk_scan<8><<<1, 256>>>(counts, a.GS);
    cudaEventRecord(e[2]);
    kern<<<(unsigned)G, 256, S::bytes()>>>(a, ld, em);
    cudaEventRecord(e[3]); cudaEventSynchronize(e[3]);
    float t;
    if (r < 3) {
      cudaEventElapsedTime(&t, e[0], e[1]); up = std::min(up, t);
      cudaEventElapsedTime(&t, e[1], e[2]); sc = std::min(sc, t);
      cudaEventElapsedTime(&t, e[2], e[3]); dn = std::min(dn, t);
    }
  }
  unsigned* bad; cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  check<<<(n + 255) / 256, 256>>>(k2, v2, n, shift, bad);
  unsigned hb; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("[bad=%u] ITEMS=%d MINB=%d G=%ld smem=%zu: upsweep %.3f scan %.3f down %.3f ms = %.0f GB/s (16 B/item)\n", hb, ITEMS, MINB,
         (long)G, S::bytes(), up, sc, dn, 16.0 * n / dn / 1e6);

}
int main() {
  const int64_t n = 128000000;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *k, *v, *k2, *v2, *counts; unsigned long long* prof;
  cudaMalloc(&k, 4 * n + 4096); cudaMalloc(&v, 4 * n + 4096); cudaMalloc(&k2, 4 * n); cudaMalloc(&v2, 4 * n);
  cudaMalloc(&counts, 4 * 256 * 1024); cudaMalloc(&prof, 8 * 8 * 1024);
  fill<<<(n + 255) / 256, 256>>>(k, v, n, 0x03ffffff);
  run<16, 2>(n, k, v, k2, v2, counts, prof, 0, sms);
  run<16, 3>(n, k, v, k2, v2, counts, prof, 0, sms);
  run<12, 3>(n, k, v, k2, v2, counts, prof, 0, sms);
  run<8, 4>(n, k, v, k2, v2, counts, prof, 0, sms);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
