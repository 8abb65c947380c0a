// Shared device helpers for the dendrogram pipeline (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dmst {

constexpr int kWarp = 32;
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Relaxed, GPU-scope 32-bit load/store for decoupled look-back words.
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Streaming (read-once) loads: evict-first in L1, no allocation priority in L2.
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldcs(p); }

// Loads of small tables that should stay L2-resident (evict_last policy).
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint32_t ld_keep(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint2 ld_keep2(const uint2* p, uint64_t pol) {
  uint2 v;
  asm volatile("ld.global.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
  return v;
}



__device__ __forceinline__ uint32_t warp_incl_sum(uint32_t x) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane_id() >= (uint32_t)o) x += y;
  }
  return x;
}

// Block-wide exclusive sum of one value per thread.  `scratch` needs
// BLOCK/32 + 1 words.  Returns the exclusive prefix; *total gets the sum.
template <int BLOCK>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t x, uint32_t* scratch, uint32_t* total) {
  constexpr int NW = BLOCK / 32;
  const uint32_t w = threadIdx.x >> 5;
  uint32_t incl = warp_incl_sum(x);
  if (lane_id() == 31) scratch[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane_id() < (uint32_t)NW ? scratch[lane_id()] : 0u;
    uint32_t si = warp_incl_sum(s);
    if (lane_id() < (uint32_t)NW) scratch[lane_id()] = si - s;
    if (lane_id() == NW - 1) scratch[NW] = si;
  }
  __syncthreads();
  uint32_t r = scratch[w] + incl - x;
  *total = scratch[NW];
  __syncthreads();
  return r;
}

// Decoupled look-back status words: [31:30] flag, [29:0] value (< 2^30).
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

// Walk predecessors' status words until an inclusive prefix is found.
// `status` is indexed [tile * stride].  A window of LB predecessors is
// loaded at once (independent loads) so one look-back costs about one L2
// round trip instead of one per predecessor.
template <int LB = 4>
__device__ __forceinline__ uint32_t lookback(const uint32_t* status, uint32_t tile, uint32_t stride) {
  uint32_t excl = 0;
  int64_t j = (int64_t)tile - 1;
  while (j >= 0) {
    uint32_t s[LB];
#pragma unroll
    for (int q = 0; q < LB; ++q) s[q] = (j - q >= 0) ? ld_relaxed(status + (uint64_t)(j - q) * stride) : kFlagPrefix;
#pragma unroll
    for (int q = 0; q < LB; ++q) {
      if (j < 0) break;
      uint32_t v = s[q];
      while (v == 0) v = ld_relaxed(status + (uint64_t)j * stride);  // not yet published: spin
      excl += v & kValMask;
      if (v & kFlagPrefix) return excl;
      --j;
    }
  }
  return excl;
}

// Warp-cooperative look-back (single status word per tile): lane i loads
// predecessor tile-1-i; the nearest inclusive prefix ends the walk, the
// aggregates in front of it are summed with a warp reduction.  Call with the
// whole warp; every lane returns the exclusive prefix of `tile`.
__device__ __forceinline__ uint32_t warp_lookback(const uint32_t* status, uint32_t tile) {
  const uint32_t lane = lane_id();
  uint32_t excl = 0;
  int64_t j0 = (int64_t)tile - 1;
  while (j0 >= 0) {
    const int64_t j = j0 - lane;
    uint32_t s = j >= 0 ? ld_relaxed(status + j) : kFlagPrefix;  // before tile 0: prefix 0
    // wait until every lane's word is published
    while (__any_sync(kFull, s == 0)) {
      if (s == 0) s = ld_relaxed(status + j);
    }
    const uint32_t pre = __ballot_sync(kFull, (s & kFlagPrefix) != 0);
    const uint32_t stop = pre ? __ffs(pre) - 1 : 32;  // first lane holding a prefix
    uint32_t v = lane <= stop ? (s & kValMask) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    excl += v;
    if (pre) break;
    j0 -= 32;
  }
  return excl;
}

}  // namespace dmst
