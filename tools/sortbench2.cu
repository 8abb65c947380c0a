// Radix-pass microbenchmark for the two sorts' geometries (AoS payload):
// u64 key + 3-word payload (edge sort) and u32 key + 1 word (chain sort),
// 128M items, uniform vs skewed digits; checks sortedness + stability.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/sortbench2 tools/sortbench2.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include "../paper_2401_06089_b200/csrc/radix.cuh"
using namespace dmst;

template <typename K, int PW>
__global__ void fill(K* k, uint32_t* v, int64_t n, int mode) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    uint64_t x = (i + 1) * 0x9E3779B97F4A7C15ull;
    x ^= x >> 31; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 29; x *= 0x94d049bb133111ebull; x ^= x >> 32;
    if (mode == 2) x = (x & 0xff) < 200 ? 0 : x;   // 78% one digit
    k[i] = (K)x;
    v[i * PW] = (uint32_t)i;
    for (int q = 1; q < PW; ++q) v[i * PW + q] = (uint32_t)(x >> (7 * q));
  }
}
template <typename K, int PW>
__global__ void check(const K* k2, const uint32_t* v2, int64_t n, unsigned* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > 0 && i < n) {
    uint32_t a = k2[i - 1] & 255, b = k2[i] & 255;
    if (a > b || (a == b && v2[(i - 1) * PW] >= v2[i * PW])) atomicAdd(bad, 1u);
  }
}
template <typename K, int PW, int BLOCK, int ITEMS, int MINB>
void run(int64_t n, K* k, uint32_t* v, K* k2, uint32_t* v2, uint32_t* counts, int sms, const char* tag) {
  using L = ArrayLoader<K, PW>;
  using E = ArrayEmitter<K, PW>;
  using S = DownSmem<K, PW, BLOCK, ITEMS, L, E>;
  auto kern = k_downsweep<K, PW, BLOCK, ITEMS, MINB, L, E>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes());
  SweepArgs a{};
  a.n = n; a.shift = 0; a.counts = counts;
  int64_t G = std::min<int64_t>((n + S::T - 1) / S::T, (int64_t)sms * MINB);
  a.chunk = ((n + G - 1) / G + S::T - 1) / S::T * S::T;
  G = (n + a.chunk - 1) / a.chunk; a.G = (uint32_t)G; a.GS = (uint32_t)((G + 3) & ~3);
  L ld{k, v};
  E em{k2, v2};
  cudaEvent_t e[4]; for (auto& x : e) cudaEventCreate(&x);
  float up = 1e9, dn = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaMemset(counts, 0, 4 * 256 * a.GS);
    cudaEventRecord(e[0]);
    k_upsweep<8, L><<<(unsigned)(G * kUpSplit), 256>>>(a, ld);
    k_chunk_scan<8><<<1, kScanThreads>>>(counts, a.GS);
    cudaEventRecord(e[2]);
    kern<<<(unsigned)G, BLOCK, S::bytes()>>>(a, ld, em);
    cudaEventRecord(e[3]); cudaEventSynchronize(e[3]);
    float t;
    if (r) {
      cudaEventElapsedTime(&t, e[0], e[2]); up = std::min(up, t);
      cudaEventElapsedTime(&t, e[2], e[3]); dn = std::min(dn, t);
    }
  }
  unsigned* bad; cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  check<K, PW><<<(n + 255) / 256, 256>>>(k2, v2, n, bad);
  unsigned hb; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  const double B = 2.0 * (sizeof(K) + 4 * PW);
  printf("%-8s K%zu PW%d BLOCK=%3d ITEMS=%2d MINB=%d smem=%6zu bad=%u: up+scan %.3f down %.3f ms = %.0f GB/s\n",
         tag, 8 * sizeof(K), PW, BLOCK, ITEMS, MINB, S::bytes(), hb, up, dn, B * n / dn / 1e6);
}
template <typename K, int PW>
void suite(int64_t n, int sms, uint32_t* counts) {
  K *k, *k2; uint32_t *v, *v2;
  cudaMalloc(&k, sizeof(K) * n + 4096); cudaMalloc(&v, 4 * PW * n + 4096);
  cudaMalloc(&k2, sizeof(K) * n); cudaMalloc(&v2, 4 * PW * n);
  const char* tags[3] = {"uniform", "-", "skew78"};
  for (int mode : {0, 2}) {
    fill<K, PW><<<(n + 255) / 256, 256>>>(k, v, n, mode);
    run<K, PW, 256, 8, 2>(n, k, v, k2, v2, counts, sms, tags[mode]);
    run<K, PW, 256, 12, 1>(n, k, v, k2, v2, counts, sms, tags[mode]);
    run<K, PW, 256, 16, 1>(n, k, v, k2, v2, counts, sms, tags[mode]);
    run<K, PW, 512, 8, 1>(n, k, v, k2, v2, counts, sms, tags[mode]);
    if (sizeof(K) == 4) {
      run<K, PW, 256, 16, 2>(n, k, v, k2, v2, counts, sms, tags[mode]);
      run<K, PW, 512, 16, 1>(n, k, v, k2, v2, counts, sms, tags[mode]);
      run<K, PW, 256, 24, 1>(n, k, v, k2, v2, counts, sms, tags[mode]);
    }
  }
  cudaFree(k); cudaFree(k2); cudaFree(v); cudaFree(v2);
}
int main() {
  const int64_t n = 128000000;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* counts;
  cudaMalloc(&counts, 4 * 256 * 1024);
  suite<uint64_t, 3>(n, sms, counts);
  suite<uint32_t, 1>(n, sms, counts);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
